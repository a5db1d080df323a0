// join.cu -- stage 2, production path: filtration as a code-ordered join.
//
// Same candidate semantics as filter.cu (Alg. 2; Appendix
// B.1-B.3): a forward candidate (r, +, p - o) for every reference position p
// whose q-gram equals the read q-gram at offset o, a reverse candidate
// (r, -, p + o + q - n) for every p whose reverse-complemented q-gram equals it.
//
// Why a join: streaming the 2L reference q-grams against a 4^q-code read
// index makes every lookup a random probe into a 512 MiB occupancy array
// (q=16); ncu shows each probe costing ~100 B of HBM traffic
// (profiles/r01/README.md). Here the reference side is a q-group index built
// once per reference and q (prepare_ref_index -- the paper's reference index
// with P ordered by q-gram), one per strand, and the batch's read
// q-grams are partitioned by the top 16 bits of their code (partition.cu).
//
// Both strands come from ONE lookup per read q-gram: the reference index and
// the read partition are keyed by canonical codes (canon_code, RefQIndex),
// and each occurrence's strand is flag(occurrence) XOR fr(read q-gram).
//
// One CTA owns one code sub-bin at a time (2^(2q-16) codes; 2048 group words
// at q=16). One elected thread stages, with 1-D TMA bulk copies completing on
// an mbarrier, the sub-bin's occupancy words and -- when they fit the staging
// buffers (every sub-bin of a 100 Mbp reference) -- its contiguous slices of
// S' and O; the group starts are rebuilt on chip (warp-scanned popcount
// prefix, u16 relative to the sub-bin's first distinct code). Every
// Group-And-Bit / Grouprank lookup (qgroup_index.hpp:50-57, 80-96) and, for a
// staged sub-bin, every S' and O read of its read q-grams is then a
// shared-memory hit; unstaged sub-bins (huge references, repeat-dense
// sub-bins) read S' / O through L1/L2. The reference index is read from HBM
// once per batch, in order, as bulk transfers; S is not read at all.
//
// Per warp step: kItems read q-grams per lane looked up, then the union of the
// occurrence intervals expanded cooperatively, one (reference occurrence,
// read occurrence) pair per lane. Everything the expansion needs travels in
// the join item (partition.cu) or in O: O holds the padded coordinate of the
// occurrence (the diagonal is O - offset, no chromosome search) and -- for
// references below 2^28 padded bases -- the strand flag and the base the
// run-start rule compares in its top 4 bits; the item holds the read's own
// compare bases (o-1 forward, complement of o+q reverse) and n - q - o.
#include <cstdlib>

#include "internal.hpp"

namespace qgm {
namespace {

constexpr int kJoinThreads = 256;
constexpr int kJoinWarps = kJoinThreads / 32;
// read q-grams (= lookups) per lane per step: the staged warp-specialised
// join runs 4 (C2 join ms: 2 0.783, 3 0.873, 4 0.771); k_join, used where
// S'/O are read from L2/HBM (C3, C4) or sub-bins are tiny, keeps 8 in flight
// (C3 shard 4.50 -> 4.28 ms, C4 1.52 -> 1.38 ms against 4)
#ifndef QGM_JOIN_ITEMS_WS
#define QGM_JOIN_ITEMS_WS 4
#endif
#ifndef QGM_JOIN_ITEMS
#define QGM_JOIN_ITEMS 8
#endif
constexpr int kItemsWs = QGM_JOIN_ITEMS_WS, kItemsJoin = QGM_JOIN_ITEMS;
static_assert(kItemsWs <= 8 && kItemsJoin <= 8, "a list entry keeps its item slot u * 32 + lane in 8 bits");
#ifndef QGM_JOIN_INLINE
#define QGM_JOIN_INLINE 4
#endif
constexpr uint32_t kInline = QGM_JOIN_INLINE;  // intervals up to this length are expanded in-lane
constexpr uint32_t kMaxWords = 2048;      // group words per sub-bin (q = 16)
constexpr uint32_t kPosMask = (1u << kPackedPosBits) - 1u;

struct JoinArgs {
  const uint64_t* items;
  const uint32_t* soff;
  uint32_t n_sub;
  unsigned code_shift;  // sub-bin = code >> code_shift
  uint32_t words;       // group words per sub-bin (>= 1)
  unsigned q;
  const uint32_t *I, *S, *S1, *O;
  const uint8_t* X;  // extra byte per occurrence (unpacked layout only)
  const uint32_t *sb_d, *sb_o;  // per sub-bin S' / O ranges (staging; null = never stage)
  const uint16_t* r16;          // group starts inside the sub-bin (null: sub-bins of < 4 words)
  uint32_t cap;                 // staging capacity of S' and of O (entries, multiple of 4)
  const uint32_t* rlen;
  uint32_t m;
  FastDiv by_m;
  const uint32_t* uniform;  // device flag: every read has length m (n - q - o needs no length load)
  int ex_sorted;            // packed O sorted inside every interval (skip_ranges applies)
  int strands;
  unsigned diag_bits;
  uint64_t* out;
  uint64_t cap_out;
  unsigned long long* counter;
  unsigned long long* stats;
};

// One (reference occurrence k, join item it) pair: true if it yields a
// candidate -- its strand is requested and the run-start rule does not
// suppress it (the (q+1)-gram one base to the left on the same diagonal also
// matches). xp = the occurrence's padded coordinate; the item is returned
// with its fr bit replaced by the candidate's strand. Op: O, or the
// shared-memory slice of a staged sub-bin (generic pointer).
template <bool kRunStart, bool kPacked, bool kBoth>
__device__ __forceinline__ bool match(const JoinArgs& a, const uint32_t* Op, uint32_t k, uint64_t& it, uint32_t& xp) {
  const uint32_t ov = Op[k];
  xp = kPacked ? (ov & kPosMask) : ov;
  const uint32_t ex = kPacked ? (ov >> kPackedPosBits) : uint32_t(__ldg(a.X + k));
  const uint32_t rev = ((ex >> 3) ^ uint32_t(it >> kItemFrShift)) & 1u;
  if (!kBoth && !((a.strands >> rev) & 1)) return false;  // kBoth: both strands requested
  if (kRunStart) {
    const uint32_t rbase = uint32_t(it >> (rev ? kItemRbShift : kItemFbShift)) & 7u;
    if ((ex & 7u) == rbase && rbase < 4) return false;
  }
  it = (it & ~(uint64_t(1) << kItemFrShift)) | (uint64_t(rev) << kItemFrShift);
  return true;
}

// The occurrence classes that yield no candidate for join item `it`: bit
// (f << 3 | b) for an occurrence of strand flag f and compare base b (its
// packed word >> 28) -- the rule match() applies, as one 16-bit mask for the
// long intervals of repeats (computed once per interval, one shift-and-test
// per occurrence). A hit item outside repeats has ~1.05 occurrences, where a
// per-item mask costs more than it saves (C2 join 0.762 -> 0.786 ms).
template <bool kRunStart>
__device__ __forceinline__ uint32_t reject_classes(const JoinArgs& a, uint64_t it) {
  const uint32_t hi = uint32_t(it >> 32);
  const uint32_t fr = (hi >> (kItemFrShift - 32)) & 1u;
  uint32_t m = 0;
#pragma unroll
  for (uint32_t f = 0; f < 2; ++f) {
    const uint32_t rev = f ^ fr;
    const uint32_t rbase = (hi >> ((rev ? kItemRbShift : kItemFbShift) - 32)) & 7u;
    if (!((a.strands >> rev) & 1)) m |= 0xFFu << (8 * f);
    else if (kRunStart && rbase < 4) m |= 1u << (8 * f + rbase);
  }
  return m;
}
template <bool kPacked>
__device__ __forceinline__ bool match_masked(const JoinArgs& a, const uint32_t* Op, uint32_t k, uint32_t reject,
                                             uint64_t& it, uint32_t& xp) {
  const uint32_t ov = Op[k];
  const uint32_t ex = kPacked ? (ov >> kPackedPosBits) : uint32_t(__ldg(a.X + k));
  if ((reject >> ex) & 1u) return false;
  xp = kPacked ? (ov & kPosMask) : ov;
  it ^= uint64_t(ex >> 3) << kItemFrShift;  // fr ^ f: the candidate's strand
  return true;
}

// Candidate key of a matched pair (item with the strand in its fr bit).
__device__ __forceinline__ uint64_t make_key(const JoinArgs& a, uint64_t it, uint32_t xp, bool uniform) {
  const uint32_t rev = uint32_t(it >> kItemFrShift) & 1u;
  const uint32_t pp = uint32_t(it);
  const uint32_t r = a.by_m.div(pp), o = pp - r * a.m;
  uint32_t off = o;  // forward: d = p - o
  if (rev) off = (uniform ? a.m : __ldg(a.rlen + r)) - a.q - o;  // d = p - (n - q - o)
  return (uint64_t(r) << (a.diag_bits + 1)) | (uint64_t(rev) << a.diag_bits) | uint64_t(xp - off);
}

// Per-warp join state: the compaction list and the emission buffer. Only
// ~9% of the visited occurrences yield a candidate (run-start rule), so the
// matched pairs are buffered (item + coordinate) and their keys built 32 at a
// time by the whole warp, then written as one coalesced run -- instead of
// building keys in whichever lanes happen to match in every round.
#ifndef QGM_JOIN_DRAIN
#define QGM_JOIN_DRAIN 64
#endif
constexpr uint32_t kDrain = QGM_JOIN_DRAIN;  // keys per output reservation (one global atomic)
static_assert(kDrain % 32 == 0, "");
constexpr uint32_t kEmitCap = kDrain + 32;
struct WarpLists {
  uint32_t* k0;
  uint32_t* k1;
  uint8_t* slot;
  uint64_t* eit;  // kEmitCap matched items
  uint32_t* exp;  // their coordinates
  uint32_t staged = 0;
  bool uniform = false;  // *JoinArgs::uniform, loaded once per thread
  unsigned long long n_hit = 0, n_occ = 0;
};

// keys of the last `cnt` (<= kDrain) buffered pairs -> one run of the output
// (one global atomic per kDrain keys: the shared candidate counter is the
// join's only point of contention)
__device__ __forceinline__ void drain(const JoinArgs& a, WarpLists& L, uint32_t cnt) {
  const unsigned lane = lane_id();
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(a.counter, (unsigned long long)cnt);
  base = __shfl_sync(kFull, base, 0);
#pragma unroll
  for (uint32_t j = 0; j < kDrain; j += 32)
    if (j + lane < cnt) {
      const uint32_t e = L.staged - cnt + j + lane;
      const uint64_t key = make_key(a, L.eit[e], L.exp[e], L.uniform);
      if (base + j + lane < a.cap_out) a.out[base + j + lane] = key;
    }
  L.staged -= cnt;
  __syncwarp();
}

__device__ __forceinline__ void flush_keys(const JoinArgs& a, WarpLists& L) {
  __syncwarp();  // the last staged pairs visible to the whole warp
  while (L.staged) drain(a, L, min(L.staged, kDrain));
}

// Occurrences inside a q-gram interval sorted by their packed word -- the
// 4 extra bits (strand flag << 3 | compare base) on top -- group by that
// class. For one item the run-start rule suppresses exactly the classes
// (f << 3 | rbase_f), f = 0, 1, rbase_f = the item's compare base for the
// strand f ^ fr, when rbase_f < 4: two sub-ranges found by binary search
// (lanes 0-3 one bound each) and skipped. In tandem repeats ~96% of the
// visited pairs are suppressed (C5: 17.9G visited, 752M emitted).
constexpr uint32_t kSkipMin = 64;  // intervals long enough to pay for four searches
__device__ __forceinline__ void skip_ranges(const uint32_t* Op, uint32_t lk0, uint32_t llen, uint64_t lit,
                                            uint32_t c[4]) {
  const unsigned lane = lane_id();
  const uint32_t fr = uint32_t(lit >> kItemFrShift) & 1u;
  const uint32_t f = (lane >> 1) & 1u, rev = f ^ fr;
  const uint32_t rbase = uint32_t(lit >> (rev ? kItemRbShift : kItemFbShift)) & 7u;
  uint32_t pos = (lane & 1u) ? lk0 + llen : lk0;  // suppression-free default: an empty range
  if (lane < 4 && rbase < 4) {
    const uint32_t v = ((f << 3) | rbase) + (lane & 1u);  // class, or the class above it
    uint32_t lo = 0, hi = llen;  // first index with Op >> 28 >= v
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if ((Op[lk0 + mid] >> kPackedPosBits) < v) lo = mid + 1; else hi = mid;
    }
    pos = lk0 + lo;
  } else if (lane < 4 && f == 0) {
    pos = lk0;  // flag 0 not suppressed: [lk0, lk0) empty
  } else if (lane < 4) {
    pos = lk0 + llen;  // flag 1 not suppressed: [end, end) empty
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i] = __shfl_sync(kFull, pos, i);
}

// The read q-gram items [my_lo, my_hi) of sub-bin `sb` (one warp): look up
// the staged occupancy words / group starts, expand the occurrence intervals
// (S1p / Op / Ip: global arrays, or generic pointers into the staged slices), emit
// the candidate keys.
template <bool kRunStart, bool kPacked, bool kBoth, int kItems>
__device__ __forceinline__ void join_items(const JoinArgs& a, const uint32_t* sI, const uint16_t* sR,
                                           const uint32_t* S1p, const uint32_t* Op, const uint64_t* Ip, uint32_t d0,
                                           uint32_t w0, uint32_t gsub, uint32_t my_lo, uint32_t my_hi,
                                           WarpLists& L) {
  const unsigned lane = lane_id();
  auto stage = [&](bool emit, uint64_t it, uint32_t xp) {  // all lanes call it
    const unsigned m = __ballot_sync(kFull, emit);
    if (!m) return;  // warp-uniform: ~90% of the pairs emit nothing
    if (emit) {
      const uint32_t e = L.staged + __popc(m & lanemask_lt());
      L.eit[e] = it;
      L.exp[e] = xp;
    }
    L.staged += __popc(m);
    if (L.staged >= kDrain) {  // the staged slots become visible to the warp before they are read
      __syncwarp();
      drain(a, L, kDrain);
    }
  };
  uint64_t pn[kItems];  // next step's items, loaded one step ahead
#pragma unroll
  for (int u = 0; u < kItems; ++u) {
    const uint32_t it = my_lo + u * 32 + lane;
    pn[u] = it < my_hi ? Ip[it] : ~0ull;
  }
  for (uint32_t base = my_lo; base < my_hi; base += 32 * kItems) {  // warp-uniform bound
    uint32_t cnt = 0, nr = 0, rk0[kItems], rk1[kItems];
#pragma unroll
    for (int u = 0; u < kItems; ++u) {
      const uint64_t pr = pn[u];
      const uint32_t itn = base + 32 * kItems + u * 32 + lane;
      pn[u] = itn < my_hi ? Ip[itn] : ~0ull;
      const bool ok = pr != ~0ull;
      const uint32_t g = gsub | uint32_t(pr >> kItemCodeShift);
      const uint32_t wl = ok ? (g >> 5) - w0 : 0u, bit = g & 31u;
      const uint32_t w = sI[wl];
      const bool hit = ok && ((w >> bit) & 1u);
      const uint32_t b = d0 + sR[wl] + __popc(w & ((1u << bit) - 1u));
      rk0[u] = hit ? S1p[b] : 0u;
      rk1[u] = hit ? S1p[b + 1] : 0u;
    }
#pragma unroll
    for (int u = 0; u < kItems; ++u) {
      const uint32_t len = rk1[u] - rk0[u];
      cnt += len;
      nr += len != 0;
    }
    L.n_hit += nr;
    L.n_occ += cnt;
    if (__all_sync(kFull, cnt == 0)) continue;
    // compact the non-empty lookups of the warp into a list
    uint32_t nent = 0;
#pragma unroll
    for (int u = 0; u < kItems; ++u) {
      const bool has = rk1[u] != rk0[u];
      const unsigned bm = __ballot_sync(kFull, has);
      if (has) {
        const uint32_t e = nent + __popc(bm & lanemask_lt());
        L.k0[e] = rk0[u];
        L.k1[e] = rk1[u];
        L.slot[e] = uint8_t(u * 32 + lane);
      }
      nent += __popc(bm);
    }
    __syncwarp();
    // one list entry per lane per round; intervals of up to kInline
    // occurrences (almost all of them) are expanded in the lane, longer ones
    // (repeats) by the whole warp, one interval at a time
    for (uint32_t e0 = 0; e0 < nent; e0 += 32) {
      const uint32_t e = e0 + lane;
      uint32_t k0 = 0, len = 0;
      uint64_t it = 0;
      if (e < nent) {
        k0 = L.k0[e];
        len = L.k1[e] - k0;
        it = Ip[base + L.slot[e]];
      }
      const bool longi = len > kInline;
      const uint32_t nin = longi ? 0u : len;
      const uint32_t rounds = __reduce_max_sync(kFull, nin);
      for (uint32_t t = 0; t < rounds; ++t) {
        uint64_t mit = it;
        uint32_t xp = 0;
        const bool emit = t < nin && match<kRunStart, kPacked, kBoth>(a, Op, k0 + t, mit, xp);
        stage(emit, mit, xp);
      }
      unsigned lm = __ballot_sync(kFull, longi);
      while (lm) {
        const int src = __ffs(lm) - 1;
        lm &= lm - 1;
        const uint32_t lk0 = __shfl_sync(kFull, k0, src), llen = __shfl_sync(kFull, len, src);
        const uint64_t lit = __shfl_sync(kFull, it, src);
        if (llen > kSkipMin) {
          // [lk0, c[0]) u [c[1], c[2]) u [c[3], end): the interval without the
          // occurrences the run-start rule suppresses for this item
          uint32_t c[4] = {lk0, lk0, lk0 + llen, lk0 + llen};
          if (kRunStart && kPacked && a.ex_sorted) skip_ranges(Op, lk0, llen, lit, c);
          const uint32_t lrej = reject_classes<kRunStart>(a, lit);
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            const uint32_t r0 = r == 0 ? lk0 : c[2 * r - 1], r1 = r == 2 ? lk0 + llen : c[2 * r];
            for (uint32_t t0 = r0; t0 < r1; t0 += 32) {
              uint64_t mit = lit;
              uint32_t xp = 0;
              const bool emit = t0 + lane < r1 && match_masked<kPacked>(a, Op, t0 + lane, lrej, mit, xp);
              stage(emit, mit, xp);
            }
          }
        } else {
          for (uint32_t t0 = lk0; t0 < lk0 + llen; t0 += 32) {
            uint64_t mit = lit;
            uint32_t xp = 0;
            const bool emit = t0 + lane < lk0 + llen && match<kRunStart, kPacked, kBoth>(a, Op, t0 + lane, mit, xp);
            stage(emit, mit, xp);
          }
        }
      }
    }
    __syncwarp();
  }
}

__device__ __forceinline__ void join_stats(const JoinArgs& a, WarpLists& L) {
  flush_keys(a, L);
  const unsigned long long h = warp_reduce_sum(L.n_hit), o = warp_reduce_sum(L.n_occ);
  if (lane_id() == 0 && a.stats && h) {
    atomicAdd(a.stats, h);
    atomicAdd(a.stats + 1, o);
  }
}

#ifndef QGM_JOIN_MINB
#define QGM_JOIN_MINB 4  // CTAs per SM the register budget of k_join is sized for
#endif
template <bool kRunStart, bool kPacked, bool kBoth>
__global__ void __launch_bounds__(kJoinThreads, QGM_JOIN_MINB) k_join(JoinArgs a) {
  QGM_GRID_DEP();
  // dynamic: I words [nw], u16 group starts [nw] (+pad to 16 B), S' slice
  // [cap], O slice [cap]
  extern __shared__ __align__(16) uint32_t s_dyn[];
  const uint32_t nw = a.words;
  uint32_t* sI = s_dyn;
  uint16_t* sR = reinterpret_cast<uint16_t*>(s_dyn + nw);
  uint32_t* sS1 = s_dyn + ((nw + (((nw + 1) / 2 + 3) & ~3u) + 3) & ~3u);
  uint32_t* sO = sS1 + a.cap;
  __shared__ uint32_t s_k0[kJoinWarps][32 * kItemsJoin];
  __shared__ uint32_t s_k1[kJoinWarps][32 * kItemsJoin];
  __shared__ uint8_t s_slot[kJoinWarps][32 * kItemsJoin];  // item slot u*32 + lane
  __shared__ uint64_t s_eit[kJoinWarps][kEmitCap];
  __shared__ uint32_t s_exp[kJoinWarps][kEmitCap];
  __shared__ __align__(8) uint64_t s_bar;

  const unsigned wid = threadIdx.x >> 5;
  WarpLists L;
  L.k0 = s_k0[wid];
  L.k1 = s_k1[wid];
  L.slot = s_slot[wid];
  L.eit = s_eit[wid];
  L.exp = s_exp[wid];
  L.uniform = __ldg(a.uniform) != 0;
  const bool bulk_I = a.r16 != nullptr;  // sub-bins of >= 8 group words: whole 16-byte chunks
  if (threadIdx.x == 0) mbar_init(&s_bar, 1);
  __syncthreads();
  uint32_t phase = 0;

  // the sub-bin's bounds (item range, S' range, O range), loaded one
  // iteration ahead
  struct Bounds { uint32_t b0, b1, d0, d1, o0, o1; };
  auto load_bounds = [&](uint32_t s, Bounds& bd) {
    if (s >= a.n_sub) return;
    bd.b0 = __ldg(a.soff + s);
    bd.b1 = __ldg(a.soff + s + 1);
    if (a.sb_d) {
      bd.d0 = __ldg(a.sb_d + s);
      bd.d1 = __ldg(a.sb_d + s + 1);
      bd.o0 = __ldg(a.sb_o + s);
      bd.o1 = __ldg(a.sb_o + s + 1);
    } else {
      bd.d0 = __ldg(a.S + uint32_t((uint64_t(s) << a.code_shift) >> 5));
      bd.d1 = bd.o0 = bd.o1 = 0;
    }
  };
  Bounds nxt{};
  load_bounds(blockIdx.x, nxt);
  for (uint32_t sb = blockIdx.x; sb < a.n_sub; sb += gridDim.x) {
    const Bounds cur = nxt;
    load_bounds(sb + gridDim.x, nxt);
    const uint32_t b0 = cur.b0, b1 = cur.b1;
    if (b0 == b1) continue;  // CTA-uniform
    // first group word of the sub-bin (sub-bins narrower than a word share it)
    const uint32_t w0 = uint32_t((uint64_t(sb) << a.code_shift) >> 5);
    const uint32_t d0 = cur.d0;
    const uint32_t sA = d0 & ~3u, oA = cur.o0 & ~3u;
    const uint32_t sN = ((cur.d1 + 1 + 3) & ~3u) - sA;  // S'[d0 .. d1] inclusive, 16-byte aligned
    const uint32_t oN = ((cur.o1 + 3) & ~3u) - oA;
    const bool staged = kPacked && a.sb_d && sN <= a.cap && oN <= a.cap;
    const uint32_t bytes = (bulk_I ? nw * 6u : 0u) + (staged ? (sN + oN) * 4u : 0u);
    if (threadIdx.x == 0 && bytes) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&s_bar, bytes);
      if (bulk_I) {
        bulk_g2s(sI, a.I + w0, nw * 4u, &s_bar);
        bulk_g2s(sR, a.r16 + w0, nw * 2u, &s_bar);
      }
      if (staged) {
        bulk_g2s(sS1, a.S1 + sA, sN * 4u, &s_bar);
        bulk_g2s(sO, a.O + oA, oN * 4u, &s_bar);
      }
    }
    // warm L2 with the next sub-bin's slices while this one is processed
    if (threadIdx.x == 32 && sb + gridDim.x < a.n_sub && nxt.b0 != nxt.b1) {
      const uint32_t nw0 = uint32_t((uint64_t(sb + gridDim.x) << a.code_shift) >> 5);
      if (bulk_I) {
        bulk_prefetch_l2(a.I + nw0, nw * 4u);
        bulk_prefetch_l2(a.r16 + nw0, nw * 2u);
      }
      const uint32_t nsA = nxt.d0 & ~3u, noA = nxt.o0 & ~3u;
      const uint32_t nsN = ((nxt.d1 + 1 + 3) & ~3u) - nsA, noN = ((nxt.o1 + 3) & ~3u) - noA;
      if (kPacked && a.sb_d && nsN <= a.cap && noN <= a.cap) {
        bulk_prefetch_l2(a.S1 + nsA, nsN * 4u);
        bulk_prefetch_l2(a.O + noA, noN * 4u);
      }
    }
    if (!bulk_I) {  // sub-bins of < 8 group words: load and rank on the spot
      if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (uint32_t i = 0; i < nw; ++i) {
          const uint32_t w = __ldg(a.I + w0 + i);
          sI[i] = w;
          sR[i] = uint16_t(run);
          run += __popc(w);
        }
      }
      __syncthreads();
    }
    if (bytes) {
      mbar_wait(&s_bar, phase);
      phase ^= 1u;
    }
    // the sub-bin's items split evenly over the warps (no warp idles at the
    // end-of-sub-bin barrier while another runs a second full round)
    const uint32_t nitems = b1 - b0;
    const uint32_t my_lo = b0 + uint32_t(uint64_t(nitems) * wid / kJoinWarps);
    const uint32_t my_hi = b0 + uint32_t(uint64_t(nitems) * (wid + 1) / kJoinWarps);
    if (staged) {  // S'/O accesses from shared-derived pointers only: LDS
      join_items<kRunStart, kPacked, kBoth, kItemsJoin>(a, sI, sR, sS1 - sA, sO - oA, a.items, d0, w0, sb << a.code_shift,
                                        my_lo, my_hi, L);
    } else {
      join_items<kRunStart, kPacked, kBoth, kItemsJoin>(a, sI, sR, a.S1, a.O, a.items, d0, w0, sb << a.code_shift, my_lo, my_hi,
                                        L);
    }
    __syncthreads();  // the staging buffers are rewritten for the next sub-bin
  }
  join_stats(a, L);
}


// ---------------------------------------------------------------------------
// Warp-specialised variant: one producer warp stages sub-bin k+1 (and k+2)
// into a second buffer while kWsCons consumer warps join sub-bin k. Full /
// empty mbarriers per buffer replace the CTA barrier, so a consumer warp that
// finishes its share of sub-bin k moves straight on to sub-bin k+1.
#ifndef QGM_JOIN_WS_CONS
#define QGM_JOIN_WS_CONS 12
#endif
constexpr int kWsCons = QGM_JOIN_WS_CONS;
constexpr int kWsThreads = (kWsCons + 1) * 32;

struct StageMeta {
  uint32_t sb, b0, b1, d0, sA, oA, iA, staged, items_staged, end;
};

template <bool kRunStart, bool kPacked, bool kBoth>
__global__ void __launch_bounds__(kWsThreads, 2) k_join_ws(JoinArgs a, uint32_t stage_words, uint32_t icap) {
  QGM_GRID_DEP();
  // 2 stages: I [nw] | u16 starts | S' [cap] | O [cap] | items [icap] (u64)
  extern __shared__ __align__(16) uint32_t s_dyn[];
  const uint32_t nw = a.words;
  __shared__ uint32_t s_k0[kWsCons][32 * kItemsWs];
  __shared__ uint32_t s_k1[kWsCons][32 * kItemsWs];
  __shared__ uint8_t s_slot[kWsCons][32 * kItemsWs];
  __shared__ uint64_t s_eit[kWsCons][kEmitCap];
  __shared__ uint32_t s_exp[kWsCons][kEmitCap];
  __shared__ StageMeta meta[2];
  __shared__ __align__(8) uint64_t full[2], empty[2];
  const unsigned wid = threadIdx.x >> 5, lane = lane_id();
  const bool bulk_I = a.r16 != nullptr;
  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&empty[0], kWsCons * 32);  // every consumer thread releases the buffer
    mbar_init(&empty[1], kWsCons * 32);
  }
  __syncthreads();
  auto stage = [&](uint32_t s, uint32_t*& sI, uint16_t*& sR, uint32_t*& sS1, uint32_t*& sO, uint64_t*& sIt) {
    uint32_t* base = s_dyn + s * stage_words;
    sI = base;
    sR = reinterpret_cast<uint16_t*>(base + nw);
    sS1 = base + ((nw + (((nw + 1) / 2 + 3) & ~3u) + 3) & ~3u);
    sO = sS1 + a.cap;
    sIt = reinterpret_cast<uint64_t*>(sO + a.cap);
  };
  if (wid == kWsCons) {  // producer
    if (lane != 0) return;
    uint32_t k = 0;
    for (uint32_t sb = blockIdx.x;; sb += gridDim.x) {
      const bool end = sb >= a.n_sub;
      uint32_t b0 = 0, b1 = 0;
      if (!end) {
        b0 = __ldg(a.soff + sb);
        b1 = __ldg(a.soff + sb + 1);
        if (b0 == b1) continue;
      }
      const uint32_t s = k & 1, j = k >> 1;
      if (j > 0) mbar_wait(&empty[s], (j - 1) & 1u);  // the consumers released this buffer's previous sub-bin
      StageMeta& M = meta[s];
      if (end) {
        M.end = 1;
        mbar_arrive(&full[s]);
        break;
      }
      const uint32_t w0 = uint32_t((uint64_t(sb) << a.code_shift) >> 5);
      uint32_t d0, d1 = 0, o0 = 0, o1 = 0;
      if (a.sb_d) {
        d0 = __ldg(a.sb_d + sb);
        d1 = __ldg(a.sb_d + sb + 1);
        o0 = __ldg(a.sb_o + sb);
        o1 = __ldg(a.sb_o + sb + 1);
      } else {
        d0 = __ldg(a.S + w0);
      }
      const uint32_t sA = d0 & ~3u, oA = o0 & ~3u;
      const uint32_t sN = ((d1 + 1 + 3) & ~3u) - sA, oN = ((o1 + 3) & ~3u) - oA;
      const bool staged = kPacked && a.sb_d && sN <= a.cap && oN <= a.cap;
      const uint32_t iA = b0 & ~1u, iN = ((b1 + 1) & ~1u) - iA;  // items, 16-byte aligned
      const bool items_staged = iN <= icap;
      M.sb = sb;
      M.b0 = b0;
      M.b1 = b1;
      M.d0 = d0;
      M.sA = sA;
      M.oA = oA;
      M.staged = staged;
      M.iA = iA;
      M.items_staged = items_staged;
      M.end = 0;
      uint32_t *sI, *sS1, *sO;
      uint16_t* sR;
      uint64_t* sIt;
      stage(s, sI, sR, sS1, sO, sIt);
      if (!bulk_I) {  // sub-bins of < 8 group words
        uint32_t run = 0;
        for (uint32_t i = 0; i < nw; ++i) {
          const uint32_t w = __ldg(a.I + w0 + i);
          sI[i] = w;
          sR[i] = uint16_t(run);
          run += __popc(w);
        }
      }
      const uint32_t bytes =
          (bulk_I ? nw * 6u : 0u) + (staged ? (sN + oN) * 4u : 0u) + (items_staged ? iN * 8u : 0u);
      fence_proxy_async();
      if (bytes) {
        mbar_arrive_expect_tx(&full[s], bytes);
        if (items_staged) bulk_g2s(sIt, a.items + iA, iN * 8u, &full[s]);
        if (bulk_I) {
          bulk_g2s(sI, a.I + w0, nw * 4u, &full[s]);
          bulk_g2s(sR, a.r16 + w0, nw * 2u, &full[s]);
        }
        if (staged) {
          bulk_g2s(sS1, a.S1 + sA, sN * 4u, &full[s]);
          bulk_g2s(sO, a.O + oA, oN * 4u, &full[s]);
        }
      } else {
        mbar_arrive(&full[s]);
      }
      ++k;
    }
    return;
  }
  WarpLists L;
  L.k0 = s_k0[wid];
  L.k1 = s_k1[wid];
  L.slot = s_slot[wid];
  L.eit = s_eit[wid];
  L.exp = s_exp[wid];
  L.uniform = __ldg(a.uniform) != 0;
  for (uint32_t k = 0;; ++k) {
    const uint32_t s = k & 1, j = k >> 1;
    mbar_wait(&full[s], j & 1u);
    const StageMeta M = meta[s];
    if (M.end) break;
    uint32_t *sI, *sS1, *sO;
    uint16_t* sR;
    uint64_t* sIt;
    stage(s, sI, sR, sS1, sO, sIt);
    const uint32_t w0 = uint32_t((uint64_t(M.sb) << a.code_shift) >> 5);
    const uint32_t nitems = M.b1 - M.b0;
    const uint32_t my_lo = M.b0 + uint32_t(uint64_t(nitems) * wid / kWsCons);
    const uint32_t my_hi = M.b0 + uint32_t(uint64_t(nitems) * (wid + 1) / kWsCons);
    if (M.staged && M.items_staged) {
      // everything in shared memory: pointers derived from the shared
      // buffers only, so every access compiles to LDS (no generic LD and its
      // 64-bit address arithmetic)
      join_items<kRunStart, kPacked, kBoth, kItemsWs>(a, sI, sR, sS1 - M.sA, sO - M.oA, sIt - M.iA, M.d0, w0,
                                        M.sb << a.code_shift, my_lo, my_hi, L);
    } else {
      const uint32_t* S1p = M.staged ? sS1 - M.sA : a.S1;
      const uint32_t* Op = M.staged ? sO - M.oA : a.O;
      const uint64_t* Ip = M.items_staged ? sIt - M.iA : a.items;
      join_items<kRunStart, kPacked, kBoth, kItemsWs>(a, sI, sR, S1p, Op, Ip, M.d0, w0, M.sb << a.code_shift, my_lo, my_hi, L);
    }
    // one arrive per consumer thread (not lane 0 after a __syncwarp): each
    // thread's own reads of meta[s] and the staged slices are then ordered
    // before the producer's refill by the barrier itself
    mbar_arrive(&empty[s]);
  }
  join_stats(a, L);
}

}  // namespace

uint64_t join_filter(Ctx& c, const Partitioned& rp, const Reads& reads, const Ref& ref, int strands, int mode,
                     unsigned read_bits, DBuf<uint64_t>& keys, uint64_t* fstats,
                     unsigned long long* dev_counter) {
  if (read_bits + 1 + ref.diag_bits > 64) throw InputError("read batch too large for the 64-bit candidate key");
  if (uint64_t(reads.stride) + 64 > ref.gap) throw InputError("reads longer than the reference padding supports");
  prepare_ref_index(c, ref, rp.q);
  subbin_tables(c, ref, rp.sub_bits);
  const RefQIndex& X = ref.qidx;
  JoinArgs a;
  a.items = rp.pairs.p;
  a.soff = rp.soff.p;
  a.n_sub = 1u << rp.sub_bits;
  a.code_shift = 2 * rp.q - rp.sub_bits;
  a.words = std::max<uint32_t>(1, (1u << a.code_shift) / 32);
  if (a.words > kMaxWords) throw InternalError("join: sub-bin wider than the shared staging");
  a.q = rp.q;
  a.I = reinterpret_cast<const uint32_t*>(X.can.I.p);
  a.S = X.can.S.p;
  a.S1 = X.can.S1.p;
  a.O = X.can.O.p;
  a.X = X.extra.p;
  a.rlen = reads.lengths.p;
  a.m = reads.stride;
  a.by_m = FastDiv(std::max<uint32_t>(reads.stride, 1));
  a.uniform = rp.flags.p + 1;
  a.ex_sorted = X.packed && X.ex_sorted;
  a.strands = strands;
  a.diag_bits = ref.diag_bits;
  // {candidates, lookups that hit, occurrences visited}: the caller's
  // buffer in the asynchronous form (read back with the batch's other
  // counts), else this call's, read back below
  DBuf<unsigned long long> own_counter;
  unsigned long long* counter = dev_counter;
  if (!counter) {
    own_counter.alloc(c, 3);
    counter = own_counter.p;
  }
  a.counter = counter;
  a.stats = counter + 1;
  // sized for the larger of 16 per read and the last batch's count on this
  // context (+1/8), so a steady stream of similar batches never re-runs
  if (keys.n == 0)
    keys.alloc(c, std::max<uint64_t>(std::max<uint64_t>(1 << 20, uint64_t(reads.n) * 16),
                                     c.last_raw_candidates + c.last_raw_candidates / 8));
  const bool rs = mode == 1;
  // Kernel choice (measured, profiles/r01/README.md): the warp-specialised
  // pipeline wins when sub-bins are staged and hold a few hundred to a couple
  // of thousand read q-grams (C2: 0.89 vs 0.97 ms), where the per-sub-bin
  // barrier and staging wait of k_join are a large share; with tiny sub-bins
  // (C1) its single producer thread is the bottleneck, with unstaged or very
  // full ones (C3, C4) k_join's 4 CTAs per SM hide latency better.
  // QGM_JOIN_WS=0/1 forces either.
  const double per_sub = double(rp.V) / double(a.n_sub);
  const bool stageable = X.packed && X.sb_d.p && X.sub_bits == rp.sub_bits;
  const char* ws_env = std::getenv("QGM_JOIN_WS");
  const bool use_ws = ws_env && ws_env[0] ? ws_env[0] == '1' : (stageable && per_sub >= 256 && per_sub <= 2048);
  // kernel variant: warp-specialised or not, run-start rule, packed O,
  // both strands requested (no per-occurrence strand test)
  static const void* const kWs[8] = {
      (const void*)k_join_ws<false, false, false>, (const void*)k_join_ws<false, false, true>,
      (const void*)k_join_ws<false, true, false>,  (const void*)k_join_ws<false, true, true>,
      (const void*)k_join_ws<true, false, false>,  (const void*)k_join_ws<true, false, true>,
      (const void*)k_join_ws<true, true, false>,   (const void*)k_join_ws<true, true, true>};
  static const void* const kPlain[8] = {
      (const void*)k_join<false, false, false>, (const void*)k_join<false, false, true>,
      (const void*)k_join<false, true, false>,  (const void*)k_join<false, true, true>,
      (const void*)k_join<true, false, false>,  (const void*)k_join<true, false, true>,
      (const void*)k_join<true, true, false>,   (const void*)k_join<true, true, true>};
  const int variant = (rs ? 4 : 0) | (X.packed ? 2 : 0) | (strands == 3 ? 1 : 0);
  const void* kfn = use_ws ? kWs[variant] : kPlain[variant];
  const int threads = use_ws ? kWsThreads : kJoinThreads;
  const int per_sm = use_ws ? 2 : 4;     // resident CTAs the staging is sized for
  const int stages = use_ws ? 2 : 1;
  // staging capacity: what is left of the SM's shared memory share of one
  // CTA after the static arrays, I words and group starts (per stage)
  const cudaFuncAttributes fa = func_attributes(kfn);
  static const int smem_sm = [] {
    int v = 0;
    QGM_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, current_device()));
    return v;
  }();
  // I words + u16 starts, padded to 16 bytes (the S'/O/item slices that follow are bulk-copy targets)
  const size_t fixed = (size_t(a.words) * 4 + (size_t((a.words + 1) / 2 + 3) & ~size_t(3)) * 4 + 15) & ~size_t(15);
  int64_t room = (int64_t(smem_sm) / per_sm - 1024 - int64_t(fa.sharedSizeBytes)) / stages - int64_t(fixed);
  // the warp-specialised kernel also stages the sub-bin's items when room is
  // left for ~1.15x the average sub-bin (beyond the S'/O slices, sized first)
  uint32_t icap = 0;
  if (use_ws) {
    const uint64_t want = (uint64_t(per_sub * 1.15) + 64) & ~uint64_t(1);
    const uint64_t so_need = 2 * 4 * (uint64_t(double(X.can.distinct) / a.n_sub * 1.15) + 64);
    if (room > int64_t(so_need + 8 * want)) {
      icap = uint32_t(want);
      room -= int64_t(8 * icap);
    }
  }
  const bool can_stage = X.packed && X.sb_d.p && X.sub_bits == rp.sub_bits && room >= 2 * 4 * 256;
  a.r16 = X.sub_bits == rp.sub_bits ? X.r16.p : nullptr;
  a.sb_d = can_stage ? X.sb_d.p : nullptr;
  a.sb_o = can_stage ? X.sb_o.p : nullptr;
  a.cap = can_stage ? uint32_t(room / 8) & ~3u : 0u;
  uint32_t stage_words = uint32_t(fixed / 4) + 2 * a.cap + 2 * icap;
  const size_t smem = size_t(stages) * stage_words * 4;
  ensure_dynamic_smem(reinterpret_cast<const void*>(kfn), size_t(smem));
  const unsigned grid = std::min<unsigned>(a.n_sub, resident_grid(kfn, threads, smem));
  for (int attempt = 0; attempt < 2; ++attempt) {
    fill_bytes(c, counter, 0, 3 * sizeof(unsigned long long));
    a.out = keys.p;
    a.cap_out = keys.n;
    if (rp.V > 0) {
      KernelScope ks(c, "k_join");
      void* args[] = {&a, &stage_words, &icap};
      cudaLaunchAttribute attr[1];
      const cudaLaunchConfig_t cfg = launch_config(c, dim3(grid), dim3(threads), smem, attr);
      QGM_CUDA(cudaLaunchKernelExC(&cfg, kfn, args));
      ++c.launches;
    }
    if (dev_counter) return 0;  // asynchronous: the caller reads the counts (and checks keys.n) later
    // the one host round trip of the filtration: candidate count, join
    // statistics and the partition's flags (exact V, length check)
    unsigned long long h[3] = {0, 0, 0};
    uint32_t fl[4] = {0, 0, 0, 0};
    QGM_CUDA(cudaMemcpyAsync(h, counter, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    read_back(c, {{rp.flags.p, fl, sizeof(fl)}});
    if (fl[2]) throw InputError("read longer than the stride");
    if (fstats) {
      fstats[0] = h[1];
      fstats[1] = h[2];
      fstats[2] = fl[0];
    }
    c.last_raw_candidates = h[0];
    if (h[0] <= keys.n) return h[0];
    keys.alloc(c, h[0] + h[0] / 8);
  }
  throw InternalError("join filtration: candidate buffer overflow after resize");
}

}  // namespace qgm
