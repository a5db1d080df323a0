// cigar.cu -- traceback_cigar of mapped hits on the device.
//
// Semantics (DESIGN.md section 2 item 9, restated by oracle::traceback_cigar): the
// oriented read against the chromosome from the hit's ref_start, global at the
// start (D[0][j] = j, D[i][0] = i), free at the end, band |j - i| <= W = B - 1;
// end = the largest j with minimal D[n][j] inside the chromosome; traceback
// prefers M, then I, then D; leading deletions move ref_start.
//
// One thread per hit, bit-parallel in diagonal coordinates (cell (i, t) is
// column j = i + t - W, t in [0, 2W]), the same row recurrence as the
// validation (validate.cu): per read row, Eq along the band, the carry chain of
// zero diagonal steps, the new deltas along t. Two differences:
//  * the start is anchored. Cells with j < 0 are not infinite but extended:
//    row 0 holds D[0][j] = |j| over the whole band. Every path into a cell
//    with j >= 0 crosses column 0 at some row i0 having paid at least i0 =
//    D[i0][0], so the extended DP equals the anchored one on j >= 0, and the
//    band needs no infinity inside it;
//  * every row's diagonal steps D1 are kept in a per-thread scratch slot (one
//    word per read row; [row][slot], reused by the grid-stride loop); the
//    traceback decides each step on bits alone
//    (see the kernel) and walks the row deltas Pv/Mv upwards by inverting
//    the forward update.
// A 64-bit band word covers B <= 32 (2W + 1 <= 63); B <= 64 uses 128 bits.
#include <cstdlib>

#include "internal.hpp"

namespace qgm {
namespace {

// 128-bit band word as two u64 halves (add with carry; shifts by any amount)
struct alignas(16) U128 {
  uint64_t lo = 0, hi = 0;
  U128() = default;
  __device__ U128(int v) : lo(uint64_t(int64_t(v))), hi(v < 0 ? ~0ull : 0ull) {}
  __device__ U128(uint64_t l, uint64_t h) : lo(l), hi(h) {}
  __device__ explicit operator uint32_t() const { return uint32_t(lo); }
  __device__ friend U128 operator&(U128 a, U128 b) { return {a.lo & b.lo, a.hi & b.hi}; }
  __device__ friend U128 operator|(U128 a, U128 b) { return {a.lo | b.lo, a.hi | b.hi}; }
  __device__ friend U128 operator^(U128 a, U128 b) { return {a.lo ^ b.lo, a.hi ^ b.hi}; }
  __device__ U128 operator~() const { return {~lo, ~hi}; }
  __device__ friend U128 operator+(U128 a, U128 b) {
    U128 r;
    asm("add.cc.u64 %0, %2, %4;\n\taddc.u64 %1, %3, %5;" : "=l"(r.lo), "=l"(r.hi) : "l"(a.lo), "l"(a.hi), "l"(b.lo),
        "l"(b.hi));
    return r;
  }
  __device__ friend U128 operator-(U128 a, U128 b) {
    U128 r;
    asm("sub.cc.u64 %0, %2, %4;\n\tsubc.u64 %1, %3, %5;" : "=l"(r.lo), "=l"(r.hi) : "l"(a.lo), "l"(a.hi), "l"(b.lo),
        "l"(b.hi));
    return r;
  }
  __device__ friend U128 operator<<(U128 a, unsigned n) {
    if (n == 0) return a;
    if (n >= 64) return {0ull, a.lo << (n - 64)};
    return {a.lo << n, (a.hi << n) | (a.lo >> (64 - n))};
  }
  __device__ friend U128 operator>>(U128 a, unsigned n) {
    if (n == 0) return a;
    if (n >= 64) return {a.hi >> (n - 64), 0ull};
    return {(a.lo >> n) | (a.hi << (64 - n)), a.hi >> n};
  }
};

struct CigarArgs {
  const uint4* hits;  // qgm_hit records
  uint64_t n_hits;
  const uint64_t* read_words;
  const uint32_t* lengths;
  uint32_t n_reads, W_words;
  const uint64_t* ref_words;
  const uint2* ref_planes;  // {lo, hi} bit planes, planes[k + 2] = word k, bit 31 - j = base 32k + j
  uint64_t n_planes;
  const uint64_t* cb;  // chromosome begins (n_chrom + 1)
  uint32_t n_chrom;
  unsigned W;          // band half-width = B - 1
  uint32_t max_ops;
  uint32_t rows;       // scratch rows per slot (max read length + 1)
  uint32_t nslots;
  uint32_t* ops;       // n_hits * max_ops
  uint2* info;         // {ref_start, n_ops | edits << 16}
  unsigned int* bad;   // set when a hit does not fit the reads / reference
};

// Sequential 2-bit base reader over a packed MSB-first stream: one word load
// per 32 bases; dir = +1 ascending, -1 descending. Positions outside
// [lo, hi) read as 4 (no match) and never load.
struct BaseStream {
  const uint64_t* w;
  int32_t pos, lo, hi, dir, cur_word, wlo, whi;
  uint64_t cur, nxt;
  __device__ __forceinline__ uint64_t load(int32_t wi) const { return wi >= wlo && wi <= whi ? __ldg(w + wi) : 0ull; }
  // the word after the current one (in the walk's direction) is always in
  // flight: a lane crossing a word boundary never waits for memory (lanes of
  // a warp cross at different steps, so a blocking reload would stall the
  // warp about every step)
  __device__ __forceinline__ void init(const uint64_t* words, int32_t p, int32_t l, int32_t h, int32_t d) {
    w = words;
    pos = p;
    lo = l;
    hi = h;
    dir = d;
    wlo = l >> 5;
    whi = (h - 1) >> 5;
    cur_word = p >> 5;
    cur = load(cur_word);
    nxt = load(cur_word + d);
  }
  template <bool kChecked>
  __device__ __forceinline__ uint32_t next() {
    const int32_t p = pos;
    pos += dir;
    const int32_t wi = p >> 5;
    if (wi != cur_word) {  // one word further in the walk's direction
      cur = nxt;
      cur_word = wi;
      nxt = load(wi + dir);
    }
    if (kChecked && (p < lo || p >= hi)) return 4u;
    return uint32_t(cur >> (62 - 2 * (p & 31))) & 3u;
  }
};

// The traceback's positions in a stream only move one way (by 0 or 1 per
// step); the same two-word window, advanced on demand.
struct BackBases {
  const uint64_t* w;
  int32_t dir, cur_word, wlo, whi;
  uint64_t cur, nxt;
  __device__ __forceinline__ uint64_t load(int32_t wi) const { return wi >= wlo && wi <= whi ? __ldg(w + wi) : 0ull; }
  __device__ __forceinline__ void init(const uint64_t* words, int32_t p, int32_t l, int32_t h, int32_t d) {
    w = words;
    dir = d;
    wlo = l >> 5;
    whi = (h - 1) >> 5;
    cur_word = p >> 5;
    cur = load(cur_word);
    nxt = load(cur_word + d);
  }
  __device__ __forceinline__ uint32_t at(int32_t p) {
    const int32_t wi = p >> 5;
    if (wi != cur_word) {
      cur = wi == cur_word + dir ? nxt : load(wi);
      cur_word = wi;
      nxt = load(wi + dir);
    }
    return uint32_t(cur >> (62 - 2 * (p & 31))) & 3u;
  }
};

template <class T>
__device__ __forceinline__ uint32_t bit_at(const T& x, unsigned t) {
  return uint32_t(x >> t) & 1u;
}

template <class T>
__global__ void __launch_bounds__(128) k_cigar(CigarArgs a, T* __restrict__ rows_buf) {
  QGM_GRID_DEP();
  const uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned W = a.W, top = 2 * W;
  const T one = T(1);
  const T mask = (one << (top + 1)) - one;
  // row i >= 1's D1 at my_rows[(i - 1) * rstep]: [row][slot] scratch, so a
  // warp's row store is one contiguous segment
  T* const my_rows = rows_buf + slot;
  const uint64_t rstep = a.nslots;
  for (uint64_t h = slot; h < a.n_hits; h += a.nslots) {
    const uint4 hit = __ldg(a.hits + h);
    const uint32_t r = hit.x, chrom = hit.y, strand = (hit.w >> 16) & 1u;
    if (r >= a.n_reads || chrom >= a.n_chrom) {
      atomicOr(a.bad, 1u);
      a.info[h] = make_uint2(hit.z, 0u);
      continue;
    }
    const int64_t rs = hit.z;
    const uint32_t n = __ldg(a.lengths + r);
    if (n + 1 > a.rows) {
      atomicOr(a.bad, 2u);
      a.info[h] = make_uint2(hit.z, 0u);
      continue;
    }
    const int64_t gb = int64_t(__ldg(a.cb + chrom));
    const int64_t Lc = int64_t(__ldg(a.cb + chrom + 1)) - gb;
    // chromosome positions are 32-bit offsets from the word holding its first
    // base (chromosomes are < 2^31 bases; the reference may exceed 2^32)
    const uint64_t* cw = a.ref_words + (uint64_t(gb) >> 5);
    const int32_t c0 = int32_t(gb & 31);
    // oriented read bases in order; the complement is applied below
    BaseStream rd, rf;
    {
      const uint64_t* rw = a.read_words + uint64_t(r) * a.W_words;
      if (strand) rd.init(rw, int32_t(n) - 1, 0, int32_t(n), -1);
      else rd.init(rw, 0, 0, int32_t(n), 1);
    }
    // reference bases slid into the band, from chromosome position rs + W + 1
    rf.init(cw, c0 + int32_t(rs) + int32_t(W) + 1, c0, c0 + int32_t(Lc), 1);
    // ---- forward pass. Row 0 (extended): D[0][t] = |t - W|.
    T P = (mask >> (W + 1)) << (W + 1);  // +1 deltas at t in (W, 2W]
    T M = ((one << (W + 1)) - one) & ~one;  // -1 deltas at t in [1, W]
    uint32_t s0 = W;
    // band window of row 1 as bit planes (base bit 0, base bit 1, inside the
    // chromosome): bit t <-> chromosome position rs - W + t; each slide
    // shifts down and inserts the next position at the top
    T pl, ph, pv;
    {  // row 1's window straight from the reference bit planes
      const int64_t g0 = gb + rs - int64_t(W);  // >= -63: the planes have two zero words in front
      const int64_t k0 = g0 >> 5;
      const unsigned off = unsigned(g0 & 31);
      auto word = [&](int64_t k, bool hi) -> uint64_t {
        const int64_t x = min(max(k + 2, int64_t(0)), int64_t(a.n_planes) - 1);
        const uint2 v = __ldg(a.ref_planes + x);
        return __brev(hi ? v.y : v.x);
      };
      auto bits64 = [&](int64_t k, bool hi) -> uint64_t {  // plane bits [32k + off, 32k + off + 64)
        const uint64_t lo = word(k, hi) | (word(k + 1, hi) << 32);
        return off ? (lo >> off) | (word(k + 2, hi) << (64 - off)) : lo;
      };
      if constexpr (sizeof(T) == 8) {
        pl = T(bits64(k0, false)) & mask;
        ph = T(bits64(k0, true)) & mask;
      } else {
        pl = T(bits64(k0, false), bits64(k0 + 2, false)) & mask;
        ph = T(bits64(k0, true), bits64(k0 + 2, true)) & mask;
      }
      // inside the chromosome: t in [max(0, W - rs), min(2W + 1, Lc - rs + W))
      const unsigned tl = unsigned(max(int64_t(0), int64_t(W) - rs));
      const unsigned th = unsigned(min(int64_t(top) + 1, Lc - rs + int64_t(W)));
      pv = th > tl ? (((one << th) - one) & ~((one << tl) - one)) : T(0);
    }
    const T topbit = one << top;
    auto slide = [&](uint32_t b) {
      pl = (pl >> 1) | ((b & 1u) && b < 4u ? topbit : T(0));
      ph = (ph >> 1) | ((b & 2u) && b < 4u ? topbit : T(0));
      pv = (pv >> 1) | (b < 4u ? topbit : T(0));
    };
    for (uint32_t i = 1; i <= n; ++i) {
      uint32_t c = rd.next<false>();
      c = strand ? 3u - c : c;
      const T Eq = ((c & 1u) ? pl : ~pl) & ((c & 2u) ? ph : ~ph) & pv;
      const T X = Eq | (M >> 1);
      const T Pp = P >> 1;
      const T Z = ((((X & Pp) + Pp) ^ Pp) | X) & mask;
      const T D1 = ~Z & mask;
      const T Bs = (D1 << 1) & mask;
      const T up = Bs & ~D1, dn = D1 & ~Bs, zr = ~(P | M);
      P = ((P & ~up) | (zr & dn)) & mask & ~one;
      M = ((M & ~dn) | (zr & up)) & mask & ~one;
      s0 += uint32_t(D1 & one);
      my_rows[uint64_t(i - 1) * rstep] = D1;  // what the traceback needs of row i
      slide(rf.next<true>());  // row i + 1 looks one position further
    }
    // ---- end column: the largest j with minimal D[n][j], j in [jlo, jhi]
    const int64_t J = int64_t(n) + W;
    const int64_t jlo = int64_t(n) > int64_t(W) ? int64_t(n) - W : 0;
    const int64_t jhi = min(J, max(Lc - rs, jlo));
    const unsigned tlo = unsigned(jlo - int64_t(n) + W), thi = unsigned(jhi - int64_t(n) + W);
    int best = 0x7FFFFFFF;
    unsigned te = tlo;
    {
      int v = int(s0);
      for (unsigned t = 0; t <= thi; ++t) {
        if (t) v += int(bit_at(P, t)) - int(bit_at(M, t));
        if (t >= tlo && v <= best) {
          best = v;
          te = t;
        }
      }
    }
    // ---- traceback from (n, te) on bits only: with delta = D[i][t] -
    // D[i-1][t] (the row's D1) and h = D[i-1][t+1] - D[i-1][t] (the deltas
    // along t of row i-1, Pv/Mv),
    //   M  iff  delta == mismatch(i, j)      (diagonal predecessor)
    //   I  iff  delta == h + 1, t < 2W       (vertical predecessor (i-1, t+1))
    //   D  otherwise                          (horizontal (i, t-1))
    // Row i-1's Pv/Mv come from row i's by inverting the forward update with
    // row i's D1, so only D1 is stored; the match bit is re-read from the
    // bases (cached words: the positions move by at most one per step).
    uint32_t* out = a.ops + h * a.max_ops;
    uint32_t n_ops = 0, run_op = 3, run_len = 0;
    auto emit = [&](uint32_t op) {
      if (op == run_op) {
        ++run_len;
        return;
      }
      if (run_len) {
        if (n_ops < a.max_ops) out[n_ops] = run_len << 4 | run_op;
        ++n_ops;
      }
      run_op = op;
      run_len = 1;
    };
    // read bases walk down (forward strand) or up (reverse strand: raw
    // index n - i), the reference down from the end column
    BackBases rb, fb;
    rb.init(a.read_words + uint64_t(r) * a.W_words, strand ? 0 : int32_t(n) - 1, 0, int32_t(n),
            strand ? 1 : -1);
    fb.init(cw, c0 + int32_t(rs + (int64_t(n) + int64_t(te) - int64_t(W)) - 1), c0, c0 + int32_t(Lc), -1);
    T rD1 = 0, pre = 0;  // row i, and row i - 1 already in flight
    auto row_at = [&](int64_t i) { return i >= 1 ? my_rows[uint64_t(i - 1) * rstep] : T(0); };
    auto enter_row = [&](int64_t i) {  // row i >= 1; P/M become row i-1's deltas
      rD1 = pre;
      pre = row_at(i - 1);
      const T Bs = (rD1 << 1) & mask;
      const T up = Bs & ~rD1, dn = rD1 & ~Bs, z = ~(P | M) & mask;
      const T oP = ((P & ~dn) | (z & up)) & mask & ~one;
      const T oM = ((M & ~up) | (z & dn)) & mask & ~one;
      P = oP;
      M = oM;
    };
    int64_t i = n;
    unsigned t = te;
    pre = row_at(i);
    if (n > 0) enter_row(i);
    // a path has at most n + j_end steps; more means inconsistent rows
    for (int64_t guard = int64_t(n) + J + 1;; --guard) {
      const int64_t j = i + int64_t(t) - int64_t(W);
      if (i == 0 && j == 0) break;
      if (guard == 0 || t > top) {
        atomicOr(a.bad, 4u);
        break;
      }
      if (i == 0) {
        emit(2);
        --t;
        continue;
      }
      if (j == 0) {
        emit(1);
        --i;
        ++t;
        continue;
      }
      const uint32_t delta = bit_at(rD1, t);
      const uint32_t rbase = strand ? 3u - rb.at(int32_t(n - i)) : rb.at(int32_t(i - 1));
      const int64_t x = rs + j - 1;  // >= 0
      const uint32_t mism = x < Lc ? uint32_t(rbase != fb.at(c0 + int32_t(x))) : 1u;
      if (delta == mism) {
        emit(0);
        --i;
        if (i > 0) enter_row(i);
        continue;
      }
      if (t < top) {
        const int hh = int(bit_at(P, t + 1)) - int(bit_at(M, t + 1));
        if (int(delta) == hh + 1) {
          emit(1);
          --i;
          ++t;
          if (i > 0) enter_row(i);
          continue;
        }
      }
      emit(2);
      --t;
    }
    // the last run emitted is the alignment's first; a leading D run moves the start
    uint32_t lead = 0;
    if (run_len) {
      if (run_op == 2) lead = run_len;
      else {
        if (n_ops < a.max_ops) out[n_ops] = run_len << 4 | run_op;
        ++n_ops;
      }
    }
    if (n_ops <= a.max_ops)
      for (uint32_t x = 0, y = n_ops; x + 1 < y; ++x, --y) {  // emitted end-first
        const uint32_t tmp = out[x];
        out[x] = out[y - 1];
        out[y - 1] = tmp;
      }
    a.info[h] = make_uint2(uint32_t(rs) + lead, min(n_ops, 0xFFFFu) | uint32_t(best - int(lead)) << 16);
  }
}

}  // namespace

void hits_cigar(Ctx& c, const DBuf<uint8_t>& hits, uint64_t n, const Reads& reads, const Ref& ref, unsigned band,
                uint32_t max_ops, DBuf<uint32_t>& ops, DBuf<uint2>& info) {
  if (band == 0 || band > 64) throw InputError("band must be in [1, 64]");
  if (max_ops == 0) throw InputError("max_ops must be positive");
  for (uint32_t k = 0; k < ref.n_chrom; ++k)
    if (ref.cb[k + 1] - ref.cb[k] >= (uint64_t(1) << 31) - 64) throw InputError("cigar: chromosome of 2^31 bases or more");
  ops.alloc(c, std::max<uint64_t>(n * max_ops, 1));
  ops.zero();  // slots past a record's n_ops read as 0 (the whole array is copied out)
  info.alloc(c, std::max<uint64_t>(n, 1));
  if (n == 0) return;
  CigarArgs a;
  a.hits = reinterpret_cast<const uint4*>(hits.p);
  a.n_hits = n;
  a.read_words = reads.words.p;
  a.lengths = reads.lengths.p;
  a.n_reads = reads.n;
  a.W_words = reads.W;
  a.ref_words = ref.words.p;
  a.ref_planes = ref.planes.p;
  a.n_planes = ref.planes.n;
  a.cb = ref.d_cb.p;
  a.n_chrom = ref.n_chrom;
  a.W = band - 1;
  a.max_ops = max_ops;
  a.rows = reads.stride + 1;
  const bool wide = band > 32;
  const size_t per_row = wide ? 16 : 8;  // one D1 word per read row
  // 1024 threads per SM: the row recurrence is a dependent chain, occupancy
  // hides it (C2, 1M hits: 4 CTAs of 128 per SM 1.98 ms, 8 CTAs 1.58 ms;
  // shared-memory rows, which cap the SM at ~280 threads, 2.99 ms). Scratch
  // bounded for long reads.
  const uint32_t threads = 128;
  uint64_t bps = 8;
  if (const char* e = std::getenv("QGM_CIGAR_BPS")) bps = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10));
  const uint64_t budget = uint64_t(512) << 20;
  uint64_t blocks = std::min<uint64_t>(ceil_div(n, threads), uint64_t(kSMs) * bps);
  blocks = std::max<uint64_t>(1, std::min<uint64_t>(blocks, budget / (uint64_t(a.rows) * per_row * threads)));
  DBuf<uint8_t> scratch(c, uint64_t(a.rows) * blocks * threads * per_row + 64);
  a.nslots = uint32_t(blocks * threads);
  DBuf<unsigned int> bad(c, 1);
  bad.zero();
  a.ops = ops.p;
  a.info = info.p;
  a.bad = bad.p;
  KernelScope ks(c, "k_cigar");
  if (wide)
    QGM_KERNEL(c, k_cigar<U128>, unsigned(blocks), threads, 0, a, reinterpret_cast<U128*>(scratch.p));
  else
    QGM_KERNEL(c, k_cigar<uint64_t>, unsigned(blocks), threads, 0, a, reinterpret_cast<uint64_t*>(scratch.p));
  unsigned int h_bad = 0;
  read_back(c, {{bad.p, &h_bad, 4}});
  if (h_bad & 1u) throw InputError("cigar: a hit's read or chromosome is not in the given reads / reference");
  if (h_bad & 2u) throw InputError("cigar: a read is longer than the reads' stride");
  if (h_bad & 4u) throw InternalError("cigar: traceback left the band");
}

}  // namespace qgm
