// validate.cu -- stage 4: banded bit-parallel semi-global validation
// (Myers 1999 / Hyyro 2003 banded; contract of
// oracle::banded_semiglobal_distance, oracles.hpp:86-111, band j-i in [0,B),
// and SPEC.md:378-395; window/start/threshold frozen by SURVEY Appendix B.4-B.6).
//
// One thread per unique candidate; candidates are sorted by read, so the lanes
// of a warp mostly share one read (its bit planes are L1 hits). The DP runs
// over the REVERSED read and window so that one pass yields both the distance
// k and the smallest optimal start (the reversed bottom row at diagonal t is
// the best cost of an alignment starting at forward column B-1-t).
//
// State per read row i (diagonal coordinates t = j - i in [0,B), one bit per
// diagonal in a 32- or 64-bit word):
//   Eq  : read'[i] == window'[i+t]  (bit planes -> 2 funnel shifts + 2 LOP3)
//   X   = Eq | Mv>>1                 (zero diagonal step from above/diagonal)
//   Z   = carry chain of zero steps along t through Pv (Myers' addition trick)
//   new Pv/Mv from the diagonal deltas D1 = ~Z and D1<<1; score of t=0 += D1&1
// ~20 integer ops per row (VALIDATE_OPS_PER_ROW in DESIGN.md).
#include <cstdlib>

#include "internal.hpp"

namespace qgm {
namespace {

// CTA size and row-bound segment (A/B, k_validate ms, 128 x 8 -> 256 x 16:
// C2 0.546 -> 0.536, C4 2.326 -> 2.271, C4 B=64 4.51 -> 4.23, C3 shard 12.39
// -> 12.13, C5m 1.60 -> 1.57; 512 threads helped only the C3 shard)
#ifndef QGM_VAL_THREADS
#define QGM_VAL_THREADS 256
#endif
constexpr int kValThreads = QGM_VAL_THREADS;
constexpr int kValThreadsBig = 512;
#ifdef QGM_VAL_HIST
__device__ unsigned long long g_exit_hist[16];  // debug: abandon row / 16, [15] = ran to the end
#endif

struct ValArgs {
  const uint2* rplanes;
  const uint32_t* rlen;
  uint32_t Wp;
  const uint2* fplanes;  // reference planes; word (x>>5)+2 holds global bases [x&~31, +32)
  const uint64_t* cb;
  const uint64_t* cbp;
  uint32_t n_chrom;
  uint64_t gap;
  const uint64_t* keys;
  uint64_t n;                         // candidates (an upper bound when d_n is set)
  const unsigned long long* d_n;      // nullable: the exact count, in device memory
  unsigned diag_bits;
  unsigned B;
  unsigned pct;
  int mode;
  uint64_t* hit_keys;
  uint32_t* hit_vals;
  unsigned long long* counter;
  void* validated;
  uint32_t* per_read;          // nullable: hits per read (map path)
  unsigned long long* n_big;   // reads passing kSmallSeg hits
};

struct Win { uint32_t lo, hi, v; };

// 32 forward window bases starting at global position a, MSB-first (bit 31-j
// = base a+j), masked to the chromosome [cbeg, cend).
__device__ __forceinline__ Win load_win(const uint2* __restrict__ fp, int64_t a, int64_t cbeg, int64_t cend,
                                        bool interior) {
  Win w{0u, 0u, 0u};
  if (!interior && (a + 32 <= cbeg || a >= cend)) return w;
  const int64_t idx = (a >> 5) + 2;
  const unsigned s = unsigned(a & 31);
  const uint2 h = __ldg(fp + idx);
  const uint2 l = __ldg(fp + idx + 1);
  w.lo = __funnelshift_l(l.x, h.x, s);
  w.hi = __funnelshift_l(l.y, h.y, s);
  if (interior) {
    w.v = 0xFFFFFFFFu;
  } else {
    const int64_t lo = cbeg - a > 0 ? cbeg - a : 0, hi = cend - a < 32 ? cend - a : 32;
    uint32_t m = 0;
    if (hi > lo) {
      m = lo >= 32 ? 0u : (0xFFFFFFFFu >> lo);
      if (hi < 32) m &= ~(0xFFFFFFFFu >> hi);
    }
    w.v = m;
  }
  return w;
}

__device__ __forceinline__ unsigned popcount_t(uint32_t x) { return __popc(x); }
__device__ __forceinline__ unsigned popcount_t(uint64_t x) { return __popcll(x); }

template <class T> struct Band;
template <> struct Band<uint32_t> {
  static constexpr int kWords = 1;
  __device__ static __forceinline__ uint32_t eq(const Win* w, unsigned t, uint32_t rl, uint32_t rh, bool chk) {
    const uint32_t lo = __funnelshift_r(w[0].lo, w[1].lo, t);
    const uint32_t hi = __funnelshift_r(w[0].hi, w[1].hi, t);
    uint32_t e = ~((lo ^ rl) | (hi ^ rh));
    if (chk) e &= __funnelshift_r(w[0].v, w[1].v, t);
    return e;
  }
};
template <> struct Band<uint64_t> {
  static constexpr int kWords = 2;
  __device__ static __forceinline__ uint64_t eq(const Win* w, unsigned t, uint32_t rl, uint32_t rh, bool chk) {
    const uint32_t lo0 = __funnelshift_r(w[0].lo, w[1].lo, t), lo1 = __funnelshift_r(w[1].lo, w[2].lo, t);
    const uint32_t hi0 = __funnelshift_r(w[0].hi, w[1].hi, t), hi1 = __funnelshift_r(w[1].hi, w[2].hi, t);
    uint32_t e0 = ~((lo0 ^ rl) | (hi0 ^ rh));
    uint32_t e1 = ~((lo1 ^ rl) | (hi1 ^ rh));
    if (chk) {
      e0 &= __funnelshift_r(w[0].v, w[1].v, t);
      e1 &= __funnelshift_r(w[1].v, w[2].v, t);
    }
    return (uint64_t(e1) << 32) | e0;
  }
};

// Lower bound of min_t D[i][t] over the band row from D[i][0] = score0 and
// the row's steps (Pv / Mv bit t: D[i][t] - D[i][t-1] = +1 / -1), in
// segments of 8 diagonals: D at a segment's first diagonal is exact (score0
// plus the steps before it) and inside the segment at most its -1 steps are
// subtracted. Tighter than the whole-row bound D[i][0] - popc(Mv) (on a
// simulated random window, n = 100, B = 32, k_max = 20, it passes k_max at
// row ~48 instead of ~62) for 4 extra popcounts per 16 rows; measured on
// B200: C3 validation 12.82 -> 12.64 ms, C2 0.559 -> 0.554 ms with segments
// of 8; 16 is better still with 256-thread CTAs (above); 4 costs more than it
// saves; QGM_VAL_SEG >= the word width = whole row.
#ifndef QGM_VAL_SEG
#define QGM_VAL_SEG 16
#endif
template <class T>
__device__ __forceinline__ int row_lower_bound(int score0, T Pv, T Mv) {
  constexpr int kBits = int(sizeof(T) * 8), kSeg = QGM_VAL_SEG < kBits ? QGM_VAL_SEG : kBits;
  if (kSeg == kBits) return score0 - int(popcount_t(Mv));  // one segment: the whole row
  int lb = score0 - int(popcount_t(T(Mv & T((T(1) << (kSeg % kBits)) - T(1)))));
#pragma unroll
  for (int s = kSeg; s < kBits; s += kSeg) {
    const T below = (T(1) << s) - T(1);                                      // steps of diagonals < s
    const T upto = s + kSeg >= kBits ? T(~T(0)) : (T(1) << (s + kSeg)) - T(1);  // ... of diagonals < s + kSeg
    lb = min(lb, score0 + int(popcount_t(T(Pv & below))) - int(popcount_t(T(Mv & upto))));
  }
  return lb;
}

// Returns false when the candidate was abandoned early: every path crosses
// every row with non-decreasing cost, so k >= min_t D[i][t] >=
// row_lower_bound at any row i; once that bound exceeds kmax the candidate
// cannot pass the identity threshold (used by the map path only, kmax < 0 =
// never).
// Rows [r_begin, min(n, r_end)) of the reversed read, r_begin a multiple of
// 16 (chunks of 32 rows share one read word and window shift; each chunk
// runs as two unrolled halves of 16 rows, the bound checked after each).
// Returns kAbandoned, kDone (the last row was processed) or kPaused (stopped
// at r_end < n).
constexpr int kAbandoned = 0, kDone = 1, kPaused = 2;
template <class T, bool kCheck, bool kFull>
__device__ __forceinline__ int myers_rows(const ValArgs& a, uint32_t r, bool rev, uint32_t n, int64_t F, uint32_t L,
                                          int64_t cbeg, int64_t cend, T mask_rt, T& Pv, T& Mv, int& score0,
                                          int kmax, uint32_t r_begin, uint32_t r_end) {
  // kFull: the band fills the word (B = 32 / 64), every mask is a no-op
  const T mask = kFull ? T(~T(0)) : mask_rt;
  constexpr int NW = Band<T>::kWords;
  const uint2* rp = a.rplanes + uint64_t(r) * a.Wp;
  const uint32_t c_begin = r_begin >> 5;
  Win w[NW + 1];
#pragma unroll
  for (int i = 0; i <= NW; ++i)
    w[i] = load_win(a.fplanes, F + int64_t(L) - 32 * int64_t(c_begin + i + 1), cbeg, cend, !kCheck);
  const uint32_t r_stop = min(n, r_end);
  const uint32_t c_stop = (r_stop + 31) >> 5;
  for (uint32_t c = c_begin; c < c_stop; ++c) {
    if (c > c_begin) {
#pragma unroll
      for (int i = 0; i < NW; ++i) w[i] = w[i + 1];
      w[NW] = load_win(a.fplanes, F + int64_t(L) - 32 * int64_t(c + NW + 1), cbeg, cend, !kCheck);
    }
    // read' reversed, rows 32c..32c+31 with row t at bit 31-t
    uint32_t rl, rh;
    if (rev) {  // rr[x] = complement(read[x])
      const uint2 v = __ldg(rp + c + 1);
      rl = ~v.x;
      rh = ~v.y;
    } else {  // rr[x] = read[n-1-x]: bases [n-32(c+1), n-32c), bit-reversed
      const int64_t a0 = int64_t(n) - 32 * int64_t(c + 1);
      const int64_t idx = (a0 >> 5) + 1;
      const unsigned s = unsigned(a0 & 31);
      const uint2 h = __ldg(rp + idx);
      const uint2 l = __ldg(rp + idx + 1);
      rl = __brev(__funnelshift_l(l.x, h.x, s));
      rh = __brev(__funnelshift_l(l.y, h.y, s));
    }
    auto row = [&](uint32_t t) {
      const uint32_t Rl = uint32_t(int32_t(rl << t) >> 31);
      const uint32_t Rh = uint32_t(int32_t(rh << t) >> 31);
      const T Eq = Band<T>::eq(w, t, Rl, Rh, kCheck) & mask;
      const T X = Eq | (Mv >> 1);
      const T Pp = Pv >> 1;
      const T Z = ((((X & Pp) + Pp) ^ Pp) | X) & mask;
      const T D1 = ~Z & mask;
      const T Bs = (D1 << 1) & mask;
      const T up = Bs & ~D1, dn = D1 & ~Bs, zr = ~(Pv | Mv);
      const T nP = ((Pv & ~up) | (zr & dn)) & mask & ~T(1);
      const T nM = ((Mv & ~dn) | (zr & up)) & mask & ~T(1);
      Pv = nP;
      Mv = nM;
      score0 += int(D1 & T(1));
    };
    auto abandon = [&](uint32_t row_end) {
      if (kmax >= 0 && row_lower_bound<T>(score0, Pv, Mv) > kmax) {
#ifdef QGM_VAL_HIST
        atomicAdd(&g_exit_hist[min(14u, row_end / 16)], 1ull);
#endif
        return true;
      }
      return false;
    };
    // rows [t, t_hi) of this chunk: whole halves unrolled (constant shift
    // amounts, no per-row loop control), the read's last partial half looped
    uint32_t t = c == c_begin ? (r_begin & 31) : 0u;
    const uint32_t t_hi = min(32u, r_stop - 32 * c);
    if (t == 0 && t_hi >= 16) {
#pragma unroll
      for (uint32_t u = 0; u < 16; ++u) row(u);
      if (abandon(32 * c + 16)) return kAbandoned;
      t = 16;
    }
    if (t == 16 && t_hi == 32) {
#pragma unroll
      for (uint32_t u = 16; u < 32; ++u) row(u);
      if (abandon(32 * c + 32)) return kAbandoned;
      t = 32;
    }
#pragma unroll 4
    for (; t < t_hi; ++t) {
      row(t);
      if ((t & 15) == 15 && abandon(32 * c + t + 1)) return kAbandoned;
    }
  }
  if (r_stop < n) return kPaused;
#ifdef QGM_VAL_HIST
  atomicAdd(&g_exit_hist[15], 1ull);
#endif
  return kDone;
}

// Validation in up to two phases on the map path: phase 1 runs every
// candidate for its first r_split rows and parks the survivors (candidate
// index + Pv, Mv, score0) in a compact list; phase 2 resumes only those.
// Candidates of random windows are abandoned around row 48 (n = 100) while
// true hits run all n rows; mixed in one warp, every warp would run n rows --
// after the split, phase-1 warps stop at the split and phase-2 warps are full
// of candidates that need the remaining rows.
struct Parked {
  uint32_t i, score0;
  uint32_t pv[2], mv[2];  // T = u32 uses word 0
};

template <class T>
__device__ __forceinline__ void pack_state(Parked& p, T Pv, T Mv) {
  p.pv[0] = uint32_t(Pv);
  p.mv[0] = uint32_t(Mv);
  p.pv[1] = sizeof(T) == 8 ? uint32_t(uint64_t(Pv) >> 32) : 0u;
  p.mv[1] = sizeof(T) == 8 ? uint32_t(uint64_t(Mv) >> 32) : 0u;
}
template <class T>
__device__ __forceinline__ void unpack_state(const Parked& p, T& Pv, T& Mv) {
  if (sizeof(T) == 8) {
    Pv = T((uint64_t(p.pv[1]) << 32) | p.pv[0]);
    Mv = T((uint64_t(p.mv[1]) << 32) | p.mv[0]);
  } else {
    Pv = T(p.pv[0]);
    Mv = T(p.mv[0]);
  }
}

// kPhase 0: every row (qgm_validate, or no split); 1: rows [0, r_split),
// survivors parked; 2: resume the parked candidates from row r_split (a
// multiple of 16).
template <class T, int kPhase, int kThreads>
__global__ void __launch_bounds__(kThreads) k_validate(ValArgs a, uint32_t r_split, Parked* __restrict__ park,
                                                          unsigned long long* __restrict__ n_park, uint64_t park_cap) {
  QGM_GRID_DEP();
  const T mask = a.B >= sizeof(T) * 8 ? T(~T(0)) : T((T(1) << a.B) - 1);
  const uint64_t dmask = (uint64_t(1) << a.diag_bits) - 1;
  const uint64_t total = kPhase == 2 ? min(uint64_t(*n_park), park_cap) : (a.d_n ? *a.d_n : a.n);
  for (uint64_t base = blockIdx.x * uint64_t(blockDim.x); base < total; base += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t slot_i = base + threadIdx.x;
    bool kept = false, in_range = false, parked = false, finish = false;
    int k = 0;
    uint32_t start = 0, ref_start = 0, r = 0, c = 0;
    bool rev = false;
    uint64_t i = slot_i;
    Parked pk{};
    if (kPhase == 2 && slot_i < total) {
      pk = park[slot_i];
      i = pk.i;
    }
    // candidate geometry (set when in range)
    T Pv = 0, Mv = 0;
    int score0 = 0, st = kAbandoned, kmax = -1;
    uint32_t n = 0, L = 0;
    int64_t cbeg = 0, cend = 0, Lc = 0, w0 = 0, F = 0;
    bool interior = false;
    auto run = [&](uint32_t cb0, uint32_t cb1) {
      const bool full = a.B == sizeof(T) * 8;
      if (interior && full)
        st = myers_rows<T, false, true>(a, r, rev, n, F, L, cbeg, cend, mask, Pv, Mv, score0, kmax, cb0, cb1);
      else if (interior)
        st = myers_rows<T, false, false>(a, r, rev, n, F, L, cbeg, cend, mask, Pv, Mv, score0, kmax, cb0, cb1);
      else
        st = myers_rows<T, true, false>(a, r, rev, n, F, L, cbeg, cend, mask, Pv, Mv, score0, kmax, cb0, cb1);
    };
    if (slot_i < total) {
      const uint64_t key = a.keys[i];
      r = uint32_t(key >> (a.diag_bits + 1));
      rev = (key >> a.diag_bits) & 1;
      const uint64_t gp = key & dmask;
      uint32_t lo = 0, hi = a.n_chrom;  // largest c with cbp[c]-gap <= gp
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(a.cbp + mid) - a.gap <= gp) lo = mid; else hi = mid;
      }
      c = lo;
      const int64_t d = int64_t(gp) - int64_t(__ldg(a.cbp + c));
      cbeg = int64_t(__ldg(a.cb + c));
      cend = int64_t(__ldg(a.cb + c + 1));
      Lc = cend - cbeg;
      n = __ldg(a.rlen + r);
      L = n + a.B - 1;
      const int64_t H = (int64_t(a.B) - 1) / 2;
      w0 = d - H;
      if (n > 0 && w0 + int64_t(L) > 0 && w0 < Lc) {
        in_range = true;
        if (kPhase == 2) {
          unpack_state<T>(pk, Pv, Mv);
          score0 = int(pk.score0);
        }
        F = cbeg + w0;
        // map path: abandon candidates that can no longer reach the threshold
        kmax = a.mode == 0 ? int((uint64_t(100 - a.pct) * n) / 100) : -1;
        interior = w0 >= 0 && w0 + int64_t(L) <= Lc;
        run(kPhase == 2 ? r_split : 0u, kPhase == 1 ? r_split : 0xFFFFFFFFu);
        parked = kPhase == 1 && st == kPaused;
        finish = !parked;
      }
    }
    if (kPhase == 1) {
      const unsigned long long ps = warp_append(parked, n_park);
      if (parked) {
        if (ps < park_cap) {
          pk.i = uint32_t(i);
          pk.score0 = uint32_t(score0);
          pack_state<T>(pk, Pv, Mv);
          park[ps] = pk;
        } else {  // no room left: finish here
          run(r_split, 0xFFFFFFFFu);
          finish = true;
        }
      }
    }
    if (finish) {
      // k = min over the band row, tbest = the last diagonal attaining it
      // (the smallest start); unrolled with constant shifts when the band
      // fills the word
      int v = score0, best = score0;
      unsigned tbest = 0;
      if (a.B == sizeof(T) * 8) {
#pragma unroll
        for (unsigned t = 1; t < sizeof(T) * 8; ++t) {
          v += int((Pv >> t) & T(1)) - int((Mv >> t) & T(1));
          if (v <= best) { best = v; tbest = t; }
        }
      } else {
        for (unsigned t = 1; t < a.B; ++t) {
          v += int((Pv >> t) & T(1)) - int((Mv >> t) & T(1));
          if (v <= best) { best = v; tbest = t; }
        }
      }
      k = best;
      start = a.B - 1 - tbest;
      int64_t rs = w0 + int64_t(start);
      rs = rs < 0 ? 0 : (rs > Lc - 1 ? Lc - 1 : rs);
      ref_start = uint32_t(rs);
      kept = st == kDone && k <= int(n) && uint64_t(100) * uint64_t(int64_t(n) - k) >= uint64_t(a.pct) * n;
    }
    if (a.mode == 0) {
      const bool emit = slot_i < total && in_range && kept;
      const unsigned long long slot = warp_append(emit, a.counter);
      if (emit) {
        const uint64_t gstart = __ldg(a.cbp + c) + ref_start;
        a.hit_keys[slot] = (uint64_t(r) << (a.diag_bits + 1)) | (gstart << 1) | uint64_t(rev);
        a.hit_vals[slot] = uint32_t(k);
        if (a.per_read && atomicAdd(a.per_read + r, 1u) == kSmallSeg) atomicAdd(a.n_big, 1ull);
      }
    } else if (slot_i < total) {
      uint32_t* o = reinterpret_cast<uint32_t*>(static_cast<char*>(a.validated) + i * 20);
      o[0] = uint32_t(k);
      o[1] = start;
      o[2] = ref_start;
      o[3] = uint32_t(kept) | (uint32_t(in_range) << 8);
      o[4] = 0;
    }
  }
}

}  // namespace

void validate_candidates(Ctx& c, const Reads& reads, const Ref& ref, const uint64_t* cand_keys, uint64_t n,
                         unsigned read_bits, unsigned band, unsigned pct, int mode, uint64_t* hit_keys,
                         uint32_t* hit_vals, unsigned long long* d_count, void* d_validated,
                         const unsigned long long* d_n, unsigned seed_q, uint32_t* per_read,
                         unsigned long long* d_big) {
  if (band == 0 || band > 64) throw InputError("band width must be in [1, 64]");
  if (pct > 100) throw InputError("percent identity must be in [0, 100]");
  if (read_bits + 1 + ref.diag_bits > 64) throw InputError("read batch too large for the 64-bit hit key");
  // the reads' planes are built on the side stream: order the compute stream
  // after them even when there is nothing to validate (the planes block goes
  // back to the stream-ordered cache when the Reads object is released)
  c.wait_planes();
  if (n == 0) return;
  ValArgs a;
  a.rplanes = reads.planes.p;
  a.rlen = reads.lengths.p;
  a.Wp = reads.Wp;
  a.fplanes = ref.planes.p;
  a.cb = ref.d_cb.p;
  a.cbp = ref.d_cbp.p;
  a.n_chrom = ref.n_chrom;
  a.gap = ref.gap;
  a.keys = cand_keys;
  a.n = n;
  a.d_n = d_n;
  a.diag_bits = ref.diag_bits;
  a.B = band;
  a.pct = pct;
  a.mode = mode;
  a.hit_keys = hit_keys;
  a.hit_vals = hit_vals;
  a.counter = d_count;
  a.validated = d_validated;
  a.per_read = per_read;
  a.n_big = d_big;
  KernelScope ks(c, "k_validate");
  // map path: split where a candidate's lower bound has passed k_max unless
  // it is a true hit: the DP's minimum grows ~0.42 per row on a random
  // window, plus the q rows of the seed match every candidate has (row ~64
  // of 100 at 80% identity, ~128 of 250 at 80%; measured, profiles/r02/
  // README.md), rounded to 16 rows
  const uint32_t kmax = uint32_t((uint64_t(100 - pct) * reads.stride) / 100);
  uint32_t r_split = (uint32_t(double(kmax) / 0.42) + seed_q + 8) & ~15u;
  const char* split_env = std::getenv("QGM_VAL_SPLIT");  // A/B and test knob: the split row, forced
  if (split_env && !split_env[0]) split_env = nullptr;
  if (split_env) r_split = uint32_t(std::atoi(split_env)) & ~15u;
  // the split pays once the candidates fill the GPU more than about twice
  // (C1, 94k candidates: 0.031 ms with it, 0.028 without); with the count on
  // the device, the context's last batch is the estimate
  const uint64_t n_est = d_n && c.last_raw_candidates ? std::min<uint64_t>(n, c.last_raw_candidates) : n;
  const bool split_pays = split_env || n_est >= uint64_t(2) * kSMs * 1024;
  // CTA size: 512 threads for batches of tens of millions of candidates (C3
  // shard: 12.13 -> 11.91 ms), 256 otherwise (C2 0.536 vs 0.560 with 512)
  const bool wide = n_est >= (uint64_t(1) << 25);
  const int threads = wide ? kValThreadsBig : kValThreads;
  const unsigned grid = unsigned(std::min<uint64_t>(ceil_div(n, uint64_t(threads)), uint64_t(kSMs) * 32));
#define QGM_VAL_LAUNCH(T, P, ...)                                                      \
  do {                                                                               \
    if (wide) QGM_KERNEL(c, (k_validate<T, P, kValThreadsBig>), grid, threads, 0, __VA_ARGS__); \
    else QGM_KERNEL(c, (k_validate<T, P, kValThreads>), grid, threads, 0, __VA_ARGS__);        \
  } while (0)
  if (mode == 0 && split_pays && r_split >= 16 && r_split < reads.stride) {
    // survivors parked for phase 2, at most 16M (candidates beyond finish in
    // phase 1)
    uint64_t cap = std::min<uint64_t>(n, uint64_t(1) << 24);
    const char* e = std::getenv("QGM_VAL_PARK_CAP");  // test knob
    if (e && e[0]) cap = std::min<uint64_t>(cap, std::strtoull(e, nullptr, 10));
    cap = std::max<uint64_t>(cap, 1);
    DBuf<Parked> park(c, cap);
    DBuf<unsigned long long> np(c, 1);
    np.zero();
    if (band <= 32) {
      QGM_VAL_LAUNCH(uint32_t, 1, a, r_split, park.p, np.p, cap);
      QGM_VAL_LAUNCH(uint32_t, 2, a, r_split, park.p, np.p, cap);
    } else {
      QGM_VAL_LAUNCH(uint64_t, 1, a, r_split, park.p, np.p, cap);
      QGM_VAL_LAUNCH(uint64_t, 2, a, r_split, park.p, np.p, cap);
    }
    return;
  }
  if (band <= 32) QGM_VAL_LAUNCH(uint32_t, 0, a, 0u, nullptr, nullptr, uint64_t(0));
  else QGM_VAL_LAUNCH(uint64_t, 0, a, 0u, nullptr, nullptr, uint64_t(0));
#undef QGM_VAL_LAUNCH
}

}  // namespace qgm

#ifdef QGM_VAL_HIST
extern "C" int qgm_debug_validate_hist(unsigned long long* out) {
  return int(cudaMemcpyFromSymbol(out, qgm::g_exit_hist, sizeof(unsigned long long) * 16));
}
#endif
