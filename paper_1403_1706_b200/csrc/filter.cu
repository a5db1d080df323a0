// filter.cu -- stage 2: filtration of the reference and its reverse complement
// against the read-side q-group index (Alg. 2; contract of
// oracle::filter_hits, oracles.hpp:37-51, and SURVEY Appendix B.1-B.3).
//
// One warp streams 32 consecutive reference positions per step (coalesced
// loads of the 2-bit reference; the reverse-complement code is derived in
// registers, no RC copy of the reference exists). Per position and strand:
// Indexpair(g) = one occupancy word, and for set bits the group base and the
// two S' entries. The warp then expands the union of its occurrence intervals
// cooperatively (one occurrence per lane per step, so long intervals from
// repeats do not serialise a single lane), applies the run-start rule
// (QGM_FILTER_RUN_START: emit only if the (q+1)-gram extending the match to
// the left does not also match -- the candidate set is unchanged), and appends
// keys to a per-warp shared-memory staging buffer that is flushed to HBM with
// one atomic per 480+ keys.
//
// Candidate key (u64): read << (diag_bits+1) | strand << diag_bits | G',
// G' = cbp[chrom] + diagonal (padded coordinates, see internal.hpp).
#include "internal.hpp"

namespace qgm {
namespace {

constexpr int kFilterThreads = 256;
constexpr int kFilterWarps = kFilterThreads / 32;
constexpr int kStage = 512;

struct FilterArgs {
  const uint64_t* ref;
  const uint64_t* mask;
  const uint64_t* cb;
  const uint64_t* cbp;
  uint32_t n_chrom;
  uint64_t total;
  const void* I;
  const uint32_t* S;
  const uint32_t* S1;
  const uint32_t* O;
  unsigned q;
  const uint64_t* rwords;
  const uint32_t* rlen;
  uint32_t W, m;
  int strands;
  unsigned diag_bits;
  uint64_t* out;
  uint64_t cap;
  unsigned long long* counter;
  unsigned long long* stats;  // {lookups with bit set, occurrences visited}
};

__device__ __forceinline__ bool is_masked(const uint64_t* mask, uint64_t x) {
  return mask && ((__ldg(mask + (x >> 6)) >> (x & 63)) & 1ull);
}

__device__ __forceinline__ uint32_t chrom_of(const uint64_t* cb, uint32_t n_chrom, uint64_t x) {
  uint32_t lo = 0, hi = n_chrom;  // largest c with cb[c] <= x
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(cb + mid) <= x) lo = mid; else hi = mid;
  }
  return lo;
}

template <class W, bool kSampled>
__device__ __forceinline__ bool index_pair(const FilterArgs& a, uint32_t g, uint32_t& k0, uint32_t& k1) {
  constexpr unsigned w = GroupTraits<W>::width;
  const W* I = static_cast<const W*>(a.I);
  const uint64_t i = g / w;
  const unsigned j = g % w;
  const W word = __ldg(I + i);
  if (!((word >> j) & W(1))) return false;
  uint32_t base;
  if (kSampled) {
    base = __ldg(a.S + (i >> 1));
    if (i & 1) base += GroupTraits<W>::popc(__ldg(I + i - 1));
  } else {
    base = __ldg(a.S + i);
  }
  base += rank_below<W>(word, j);
  k0 = __ldg(a.S1 + base);
  k1 = __ldg(a.S1 + base + 1);
  return k1 > k0;
}

template <class W, bool kSampled, bool kRunStart>
__global__ void __launch_bounds__(kFilterThreads) k_filter(FilterArgs a) {
  QGM_GRID_DEP();
  __shared__ uint32_t s_k0[kFilterWarps][64];
  __shared__ uint32_t s_pre[kFilterWarps][65];
  __shared__ uint64_t s_x[kFilterWarps][64];
  __shared__ uint32_t s_p[kFilterWarps][64];
  __shared__ uint32_t s_meta[kFilterWarps][64];  // chrom | strand << 31
  __shared__ uint64_t s_out[kFilterWarps][kStage];

  const unsigned lane = lane_id(), wid = threadIdx.x >> 5;
  const uint64_t gwarp = (uint64_t(blockIdx.x) * kFilterThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * kFilterThreads) >> 5;
  const unsigned q = a.q;
  uint32_t staged = 0;
  unsigned long long n_hit = 0, n_occ = 0;

  auto flush = [&]() {
    unsigned long long base = 0;
    if (lane == 0 && staged) base = atomicAdd(a.counter, (unsigned long long)staged);
    base = __shfl_sync(kFull, base, 0);
    for (uint32_t i = lane; i < staged; i += 32)
      if (base + i < a.cap) a.out[base + i] = s_out[wid][i];
    staged = 0;
    __syncwarp();
  };

  for (uint64_t x0 = gwarp * 32; x0 < a.total; x0 += nwarps * 32) {
    const uint64_t x = x0 + lane;
    uint32_t nr = 0, cnt = 0;
    uint32_t rk0[2], rn[2], rmeta[2];
    uint32_t c = 0, p = 0;
    if (x < a.total && !is_masked(a.mask, x)) {
      c = chrom_of(a.cb, a.n_chrom, x);
      const uint64_t cbeg = __ldg(a.cb + c);
      const uint64_t Lc = __ldg(a.cb + c + 1) - cbeg;
      p = uint32_t(x - cbeg);
      if (uint64_t(p) + q <= Lc) {
        const uint32_t g = qgram_at(a.ref, x, q);
        uint32_t k0, k1;
        if ((a.strands & 1) && index_pair<W, kSampled>(a, g, k0, k1)) {
          rk0[nr] = k0; rn[nr] = k1 - k0; rmeta[nr] = c; cnt += k1 - k0; ++nr;
        }
        if ((a.strands & 2) && index_pair<W, kSampled>(a, rc_code(g, q), k0, k1)) {
          rk0[nr] = k0; rn[nr] = k1 - k0; rmeta[nr] = c | 0x80000000u; cnt += k1 - k0; ++nr;
        }
      }
    }
    n_hit += nr;
    n_occ += cnt;
    // lay out this warp's occurrence intervals in shared memory
    const uint32_t r_off = warp_inclusive_scan(nr) - nr;
    const uint32_t o_inc = warp_inclusive_scan(cnt);
    const uint32_t o_off = o_inc - cnt;
    const uint32_t R = __shfl_sync(kFull, r_off + nr, 31);
    const uint32_t T = __shfl_sync(kFull, o_inc, 31);
    if (T == 0) continue;
    uint32_t run = o_off;
    for (uint32_t i = 0; i < nr; ++i) {
      s_k0[wid][r_off + i] = rk0[i];
      s_pre[wid][r_off + i] = run;
      s_x[wid][r_off + i] = x;
      s_p[wid][r_off + i] = p;
      s_meta[wid][r_off + i] = rmeta[i];
      run += rn[i];
    }
    if (lane == 0) s_pre[wid][R] = T;
    __syncwarp();
    for (uint32_t j0 = 0; j0 < T; j0 += 32) {
      const uint32_t j = j0 + lane;
      bool emit = false;
      uint64_t key = 0;
      if (j < T) {
        uint32_t lo = 0, hi = R;  // largest e with s_pre[e] <= j
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (s_pre[wid][mid] <= j) lo = mid; else hi = mid;
        }
        const uint32_t pp = __ldg(a.O + s_k0[wid][lo] + (j - s_pre[wid][lo]));
        const uint32_t r = pp / a.m, o = pp - r * a.m;
        const uint32_t meta = s_meta[wid][lo];
        const uint32_t cc = meta & 0x7FFFFFFFu;
        const bool rev = meta >> 31;
        const uint32_t pr = s_p[wid][lo];
        const uint64_t xr = s_x[wid][lo];
        const uint64_t* rw = a.rwords + uint64_t(r) * a.W;
        int64_t d;
        emit = true;
        if (!rev) {
          d = int64_t(pr) - int64_t(o);
          if (kRunStart && pr >= 1 && o >= 1 && !is_masked(a.mask, xr - 1) &&
              base_at(a.ref, xr - 1) == base_at(rw, o - 1))
            emit = false;
        } else {
          const uint32_t n = __ldg(a.rlen + r);
          d = int64_t(pr) + int64_t(o) + int64_t(q) - int64_t(n);
          if (kRunStart && pr >= 1 && o + q + 1 <= n && !is_masked(a.mask, xr - 1) &&
              (3u - base_at(a.ref, xr - 1)) == base_at(rw, o + q))
            emit = false;
        }
        const uint64_t gp = uint64_t(int64_t(__ldg(a.cbp + cc)) + d);
        key = (uint64_t(r) << (a.diag_bits + 1)) | (uint64_t(rev) << a.diag_bits) | gp;
      }
      const unsigned m = __ballot_sync(kFull, emit);
      if (emit) s_out[wid][staged + __popc(m & lanemask_lt())] = key;
      staged += __popc(m);
      __syncwarp();
      if (staged > kStage - 32) flush();
    }
  }
  flush();
  n_hit = warp_reduce_sum(n_hit);
  n_occ = warp_reduce_sum(n_occ);
  if (lane == 0 && a.stats && n_hit) {
    atomicAdd(a.stats, n_hit);
    atomicAdd(a.stats + 1, n_occ);
  }
}

template <class W, bool kSampled>
void launch_filter(Ctx& c, const FilterArgs& a, int mode, unsigned grid) {
  if (mode == 1) QGM_KERNEL(c, (k_filter<W, kSampled, true>), grid, kFilterThreads, 0, a);
  else QGM_KERNEL(c, (k_filter<W, kSampled, false>), grid, kFilterThreads, 0, a);
}

}  // namespace

uint64_t filter_reference(Ctx& c, const Index& idx, const Reads& reads, const Ref& ref, int strands, int mode,
                          unsigned read_bits, DBuf<uint64_t>& keys, uint64_t* fstats) {
  if (idx.stride != reads.stride || idx.n_reads != reads.n)
    throw InputError("index was built over a different read buffer");
  if (read_bits + 1 + ref.diag_bits > 64) throw InputError("read batch too large for the 64-bit candidate key");
  if (uint64_t(reads.stride) + 64 > ref.gap) throw InputError("reads longer than the reference padding supports");
  FilterArgs a;
  a.ref = ref.words.p;
  a.mask = ref.mask.p;
  a.cb = ref.d_cb.p;
  a.cbp = ref.d_cbp.p;
  a.n_chrom = ref.n_chrom;
  a.total = ref.total;
  a.I = idx.I.p;
  a.S = idx.S.p;
  a.S1 = idx.S1.p;
  a.O = idx.O.p;
  a.q = idx.q;
  a.rwords = reads.words.p;
  a.rlen = reads.lengths.p;
  a.W = reads.W;
  a.m = reads.stride;
  a.strands = strands;
  a.diag_bits = ref.diag_bits;
  DBuf<unsigned long long> counter(c, 3);  // {emitted, lookups hit, occurrences}
  a.counter = counter.p;
  a.stats = counter.p + 1;
  // sized for the larger of 16 per read and the last batch's count on this
  // context (+1/8), so a steady stream of similar batches never re-runs
  if (keys.n == 0)
    keys.alloc(c, std::max<uint64_t>(std::max<uint64_t>(1 << 20, uint64_t(reads.n) * 16),
                                     c.last_raw_candidates + c.last_raw_candidates / 8));
  const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(ref.total, kFilterThreads * 4),
                                                                          uint64_t(kSMs) * 8)));
  for (int attempt = 0; attempt < 2; ++attempt) {
    counter.zero();
    a.out = keys.p;
    a.cap = keys.n;
    if (ref.total > 0) {
      KernelScope ks(c, "k_filter");
      if (idx.w == 32) {
        if (idx.sampled) launch_filter<uint32_t, true>(c, a, mode, grid);
        else launch_filter<uint32_t, false>(c, a, mode, grid);
      } else {
        if (idx.sampled) launch_filter<uint64_t, true>(c, a, mode, grid);
        else launch_filter<uint64_t, false>(c, a, mode, grid);
      }
    }
    unsigned long long h[3] = {0, 0, 0};
    read_back(c, {{counter.p, h, sizeof(h)}});
    if (fstats) {
      fstats[0] = h[1];
      fstats[1] = h[2];
    }
    c.last_raw_candidates = h[0];
    if (h[0] <= keys.n) return h[0];
    keys.alloc(c, h[0] + h[0] / 8);  // exact size known now: one re-run
  }
  throw InternalError("filtration: candidate buffer overflow after resize");
}

}  // namespace qgm
