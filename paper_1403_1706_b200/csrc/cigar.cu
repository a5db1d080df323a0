// cigar.cu -- traceback_cigar of mapped hits on the device.
//
// Semantics (DESIGN.md Appendix B.8, restated by oracle::traceback_cigar): the
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
//  * every row's (Pv, Mv, D[i][0]) is kept in a per-thread scratch slot
//    ([row][slot] layout, so a warp's row store is one contiguous segment;
//    slots are reused by the grid-stride loop and stay L2-resident), and the
//    traceback rebuilds D[i][t] = D[i][0] + popc(Pv & bits 1..t) -
//    popc(Mv & bits 1..t) from them.
// A 64-bit band word covers B <= 32 (2W + 1 <= 63); B <= 64 uses 128 bits.
#include "internal.hpp"

namespace qgm {
namespace {

// 128-bit band word as two u64 halves (add with carry; shifts by any amount)
struct U128 {
  uint64_t lo = 0, hi = 0;
  __device__ U128() = default;
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
  __device__ U128& operator|=(U128 b) { return *this = *this | b; }
};

template <class T> struct BandBits;
template <> struct BandBits<uint64_t> {
  __device__ static __forceinline__ unsigned popc(uint64_t x) { return __popcll(x); }
};
template <> struct BandBits<U128> {
  __device__ static __forceinline__ unsigned popc(U128 x) { return __popcll(x.lo) + __popcll(x.hi); }
};

struct CigarArgs {
  const uint4* hits;  // qgm_hit records
  uint64_t n_hits;
  const uint64_t* read_words;
  const uint32_t* lengths;
  uint32_t n_reads, W_words;
  const uint64_t* ref_words;
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

template <class T>
__global__ void __launch_bounds__(128) k_cigar(CigarArgs a, T* __restrict__ sP, T* __restrict__ sM,
                                               uint16_t* __restrict__ sS) {
  const uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned W = a.W, top = 2 * W;
  const T one = T(1);
  const T mask = (one << (top + 1)) - one;
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
    const uint64_t gb = __ldg(a.cb + chrom);
    const int64_t Lc = int64_t(__ldg(a.cb + chrom + 1) - gb);
    const uint64_t* rw = a.read_words + uint64_t(r) * a.W_words;
    auto read_base = [&](uint32_t i) -> uint32_t {  // oriented read base i
      return strand ? 3u - base_at(rw, n - 1 - i) : base_at(rw, i);
    };
    auto ref_base = [&](int64_t x) -> uint32_t {  // chromosome position x; 4 = outside
      return x >= 0 && x < Lc ? base_at(a.ref_words, gb + uint64_t(x)) : 4u;
    };
    // ---- forward pass. Row 0 (extended): D[0][t] = |t - W|.
    T P = (mask >> (W + 1)) << (W + 1);  // +1 deltas at t in (W, 2W]
    T M = ((one << (W + 1)) - one) & ~one;  // -1 deltas at t in [1, W]
    uint32_t s0 = W;
    auto store = [&](uint32_t i) {
      const uint64_t o = uint64_t(i) * a.nslots + slot;
      sP[o] = P;
      sM[o] = M;
      sS[o] = uint16_t(s0);
    };
    store(0);
    // Eq masks of row 1: t <-> chromosome position rs - W + t
    T m0 = 0, m1 = 0, m2 = 0, m3 = 0;
    for (unsigned t = 0; t <= top; ++t) {
      const uint32_t b = ref_base(rs - int64_t(W) + t);
      const T bit = one << t;
      m0 |= b == 0 ? bit : T(0);
      m1 |= b == 1 ? bit : T(0);
      m2 |= b == 2 ? bit : T(0);
      m3 |= b == 3 ? bit : T(0);
    }
    for (uint32_t i = 1; i <= n; ++i) {
      const uint32_t c = read_base(i - 1);
      const T Eq = c == 0 ? m0 : c == 1 ? m1 : c == 2 ? m2 : m3;
      const T X = Eq | (M >> 1);
      const T Pp = P >> 1;
      const T Z = ((((X & Pp) + Pp) ^ Pp) | X) & mask;
      const T D1 = ~Z & mask;
      const T Bs = (D1 << 1) & mask;
      const T up = Bs & ~D1, dn = D1 & ~Bs, zr = ~(P | M);
      const T nP = ((P & ~up) | (zr & dn)) & mask & ~one;
      const T nM = ((M & ~dn) | (zr & up)) & mask & ~one;
      P = nP;
      M = nM;
      s0 += uint32_t(D1 & one);
      store(i);
      // slide the masks to row i + 1: the new top cell is position rs + i + W
      const uint32_t b = ref_base(rs + int64_t(i) + W);
      const T bit = one << top;
      m0 = (m0 >> 1) | (b == 0 ? bit : T(0));
      m1 = (m1 >> 1) | (b == 1 ? bit : T(0));
      m2 = (m2 >> 1) | (b == 2 ? bit : T(0));
      m3 = (m3 >> 1) | (b == 3 ? bit : T(0));
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
        if (t) v += int(uint32_t(P >> t) & 1u) - int(uint32_t(M >> t) & 1u);
        if (t >= tlo && v <= best) {
          best = v;
          te = t;
        }
      }
    }
    // ---- traceback from (n, te); ops are emitted from the end
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
    auto dval = [&](const T& p, const T& m, uint32_t s, unsigned t) -> int {
      const T low = ((one << t) - one) << 1;  // bits 1..t
      return int(s) + int(BandBits<T>::popc(p & low)) - int(BandBits<T>::popc(m & low));
    };
    int64_t i = n;
    unsigned t = te;
    int cur = best;
    // a path has at most n + j_end steps; more means inconsistent DP rows
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
        --cur;
        continue;
      }
      if (j == 0) {
        emit(1);
        --i;
        ++t;
        --cur;
        continue;
      }
      const uint64_t o = uint64_t(i - 1) * a.nslots + slot;
      const T pu = sP[o], mu = sM[o];
      const uint32_t su = sS[o];
      const int dd = dval(pu, mu, su, t);
      if (dd + (read_base(uint32_t(i - 1)) == ref_base(rs + j - 1) ? 0 : 1) == cur) {
        emit(0);
        cur = dd;
        --i;
        continue;
      }
      if (t < top) {
        const int vu = dval(pu, mu, su, t + 1);
        if (vu + 1 == cur) {
          emit(1);
          cur = vu;
          --i;
          ++t;
          continue;
        }
      }
      emit(2);
      --t;
      --cur;
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
  ops.alloc(c, std::max<uint64_t>(n * max_ops, 1));
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
  a.cb = ref.d_cb.p;
  a.n_chrom = ref.n_chrom;
  a.W = band - 1;
  a.max_ops = max_ops;
  a.rows = reads.stride + 1;
  const bool wide = band > 32;
  const size_t per_row = (wide ? 32 : 16) + 2;
  // slots: enough warps per SM to hide the row recurrence, scratch bounded
  // (kept near L2 size for 100 bp reads)
  const uint64_t budget = uint64_t(256) << 20;
  uint64_t blocks = std::min<uint64_t>(ceil_div(n, 128), uint64_t(kSMs) * 4);
  blocks = std::max<uint64_t>(1, std::min<uint64_t>(blocks, budget / (uint64_t(a.rows) * per_row * 128)));
  a.nslots = uint32_t(blocks * 128);
  DBuf<uint8_t> scratch(c, uint64_t(a.rows) * a.nslots * per_row + 64);
  DBuf<unsigned int> bad(c, 1);
  bad.zero();
  a.ops = ops.p;
  a.info = info.p;
  a.bad = bad.p;
  const uint64_t cells = uint64_t(a.rows) * a.nslots;
  KernelScope ks(c, "k_cigar");
  if (wide) {
    auto* P = reinterpret_cast<U128*>(scratch.p);
    QGM_KERNEL(c, k_cigar<U128>, unsigned(blocks), 128, 0, a, P, P + cells,
               reinterpret_cast<uint16_t*>(P + 2 * cells));
  } else {
    auto* P = reinterpret_cast<uint64_t*>(scratch.p);
    QGM_KERNEL(c, k_cigar<uint64_t>, unsigned(blocks), 128, 0, a, P, P + cells,
               reinterpret_cast<uint16_t*>(P + 2 * cells));
  }
  unsigned int h_bad = 0;
  QGM_CUDA(cudaMemcpyAsync(&h_bad, bad.p, 4, cudaMemcpyDeviceToHost, c.stream));
  QGM_CUDA(cudaStreamSynchronize(c.stream));
  if (h_bad & 1u) throw InputError("cigar: a hit's read or chromosome is not in the given reads / reference");
  if (h_bad & 2u) throw InputError("cigar: a read is longer than the reads' stride");
  if (h_bad & 4u) throw InternalError("cigar: traceback left the band");
}

}  // namespace qgm
