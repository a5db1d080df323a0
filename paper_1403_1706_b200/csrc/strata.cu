// strata.cu -- stage 5: best-stratum / all-hits reduction (
// SURVEY Appendix B.6) over hits radix-sorted by (read, chrom, ref_start,
// strand). Identity (n-k)/n is monotone in k for a fixed read, so strata are
// compared on integer k.
//   K1: first hit of every (read, chrom, ref_start, strand) group keeps the
//       group's minimum k (hit-level dedup) and folds it into the read's
//       minimum with atomicMin;
//   K2: keep flag (all mode, or k == the read's minimum);
//   scan + K3: order-preserving compaction into 16-byte qgm_hit records.
#include "internal.hpp"

namespace qgm {
namespace {

__global__ void k_group_min(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t n,
                            unsigned diag_bits, uint32_t* __restrict__ readmin, uint32_t* __restrict__ first,
                            uint32_t* __restrict__ gmin) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = keys[i];
    const bool f = i == 0 || keys[i - 1] != k;
    first[i] = f;
    if (!f) continue;
    uint32_t m = vals[i];
    for (uint64_t j = i + 1; j < n && keys[j] == k; ++j) m = min(m, vals[j]);
    gmin[i] = m;
    atomicMin(readmin + (k >> (diag_bits + 1)), m);
  }
}

__global__ void k_keep(const uint64_t* __restrict__ keys, uint64_t n, unsigned diag_bits, int mode,
                       const uint32_t* __restrict__ readmin, const uint32_t* __restrict__ first,
                       const uint32_t* __restrict__ gmin, uint32_t* __restrict__ keep) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    keep[i] = first[i] && (mode == 1 || gmin[i] == readmin[keys[i] >> (diag_bits + 1)]);
}

__global__ void k_emit(const uint64_t* __restrict__ keys, uint64_t n, unsigned diag_bits,
                       const uint32_t* __restrict__ keep, const uint32_t* __restrict__ pos,
                       const uint32_t* __restrict__ gmin, const uint64_t* __restrict__ cbp, uint32_t n_chrom,
                       uint4* __restrict__ out) {
  const uint64_t dmask = (uint64_t(1) << diag_bits) - 1;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    if (!keep[i]) continue;
    const uint64_t k = keys[i];
    const uint32_t r = uint32_t(k >> (diag_bits + 1));
    const uint64_t gs = (k >> 1) & dmask;
    uint32_t lo = 0, hi = n_chrom;  // largest c with cbp[c] <= gs
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(cbp + mid) <= gs) lo = mid; else hi = mid;
    }
    const uint32_t start = uint32_t(gs - __ldg(cbp + lo));
    out[pos[i]] = make_uint4(r, lo, start, (gmin[i] & 0xFFFFu) | (uint32_t(k & 1) << 16));
  }
}

}  // namespace

uint64_t stratify_hits(Ctx& c, const Ref& ref, const uint64_t* hit_keys, const uint32_t* hit_vals, uint64_t n,
                       uint32_t n_reads, unsigned read_bits, int mode, DBuf<uint8_t>& out) {
  (void)read_bits;
  if (n == 0) {
    out.alloc(c, 16);
    return 0;
  }
  DBuf<uint32_t> readmin(c, std::max<uint32_t>(n_reads, 1));
  QGM_CUDA(cudaMemsetAsync(readmin.p, 0xFF, readmin.bytes(), c.stream));
  DBuf<uint32_t> first(c, n), gmin(c, n), keep(c, n), total(c, 1);
  const unsigned grid = unsigned(std::min<uint64_t>(ceil_div(n, 256), uint64_t(kSMs) * 16));
  QGM_KERNEL(c, k_group_min, grid, 256, 0, hit_keys, hit_vals, n, ref.diag_bits, readmin.p, first.p, gmin.p);
  QGM_KERNEL(c, k_keep, grid, 256, 0, hit_keys, n, ref.diag_bits, mode, readmin.p, first.p, gmin.p, keep.p);
  exclusive_scan_u32(c, keep.p, first.p, n, total.p, nullptr);  // first <- output slots
  uint32_t kept = 0;
  QGM_CUDA(cudaMemcpyAsync(&kept, total.p, 4, cudaMemcpyDeviceToHost, c.stream));
  QGM_CUDA(cudaStreamSynchronize(c.stream));
  out.alloc(c, std::max<uint64_t>(uint64_t(kept) * 16, 16));
  QGM_KERNEL(c, k_emit, grid, 256, 0, hit_keys, n, ref.diag_bits, keep.p, first.p, gmin.p, ref.d_cbp.p, ref.n_chrom,
             reinterpret_cast<uint4*>(out.p));
  return kept;
}

}  // namespace qgm
