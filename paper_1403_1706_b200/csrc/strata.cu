// strata.cu -- stage 5: best-stratum / all-hits reduction (
// SURVEY Appendix B.6). Identity (n-k)/n is monotone in k for a fixed read, so
// strata are compared on integer k. Output: 16-byte qgm_hit records sorted by
// (read, chrom, ref_start, strand), one per (read, chrom, ref_start, strand)
// group with the group's minimum k; best-stratum keeps the groups whose k is
// the read's minimum.
//
// Map path (stratify_unsorted): hits arrive in validation order. A counting
// sort by read (count, scan, scatter) gives every read its segment (~1.3 hits
// at C2); one thread per read sorts its segment in registers/local memory,
// dedups, finds the read's minimum and counts the kept groups; a scan of the
// kept counts places the records. Reads with more than kSmallSeg hits
// (repeats) are sorted by the LSD radix sort on the subset of their hits,
// written back into their (contiguous, read-ordered) segments.
//
// Sorted-input path (stratify_hits, hits radix-sorted by the caller):
//   K1: first hit of every group keeps the group's minimum k and folds it
//       into the read's minimum with atomicMin;
//   K2: keep flag (all mode, or k == the read's minimum);
//   scan + K3: order-preserving compaction.
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

// ------------------------------------------------------------ segmented path
constexpr uint32_t kSmallSeg = 32;

__global__ void k_count_reads(const uint64_t* __restrict__ keys, uint64_t n, unsigned rshift,
                              uint32_t* __restrict__ cnt) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    atomicAdd(cnt + (keys[i] >> rshift), 1u);
}

// cnt[r] counts down while hits are placed (segment filled from its end)
__global__ void k_scatter_reads(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t n,
                                unsigned rshift, const uint32_t* __restrict__ off, uint32_t* __restrict__ cnt,
                                uint64_t* __restrict__ skeys, uint32_t* __restrict__ svals) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = keys[i];
    const uint32_t r = uint32_t(k >> rshift);
    const uint32_t pos = off[r] + atomicSub(cnt + r, 1u) - 1u;
    skeys[pos] = k;
    svals[pos] = vals[i];
  }
}

// per read: sort the segment (small ones here, big ones by the caller),
// group minima, the read's minimum, keep marks (value ~0u = dropped), kept count
__global__ void k_seg_reduce(uint64_t* __restrict__ skeys, uint32_t* __restrict__ svals,
                             const uint32_t* __restrict__ off, uint32_t n_reads, int mode, int sorted_big,
                             uint32_t* __restrict__ kept, uint32_t* __restrict__ big) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_reads; r += gridDim.x * blockDim.x) {
    const uint32_t b = off[r], m = off[r + 1] - b;
    uint32_t nk = 0;
    if (sorted_big) {  // second launch: only the big segments, now sorted
      if (!big[r]) continue;
    } else if (m > kSmallSeg) {
      big[r] = m;  // sorted by the caller, then reduced in a second launch
      kept[r] = 0;
      continue;
    } else {
      big[r] = 0;
    }
    uint64_t* K = skeys + b;
    uint32_t* V = svals + b;
    if (m <= kSmallSeg) {  // insertion sort by key
      for (uint32_t i = 1; i < m; ++i) {
        const uint64_t x = K[i];
        const uint32_t v = V[i];
        uint32_t j = i;
        while (j > 0 && K[j - 1] > x) {
          K[j] = K[j - 1];
          V[j] = V[j - 1];
          --j;
        }
        K[j] = x;
        V[j] = v;
      }
    }
    // group minima in place (first of a group holds it; later members get
    // value ~0u), then the read minimum
    uint32_t rmin = 0xFFFFFFFFu;
    for (uint32_t i = 0; i < m;) {
      uint32_t j = i + 1, g = V[i];
      while (j < m && K[j] == K[i]) {
        g = min(g, V[j]);
        V[j] = 0xFFFFFFFFu;
        ++j;
      }
      V[i] = g;
      rmin = min(rmin, g);
      i = j;
    }
    for (uint32_t i = 0; i < m; ++i) {
      const uint32_t v = V[i];
      const bool first = i == 0 || K[i] != K[i - 1];
      const bool keep = first && (mode == 1 || v == rmin);
      if (!keep) V[i] = 0xFFFFFFFFu;
      nk += keep;
    }
    kept[r] = nk;
  }
}

__global__ void k_seg_emit(const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ svals,
                           const uint32_t* __restrict__ off, const uint32_t* __restrict__ kept_off, uint32_t n_reads,
                           unsigned diag_bits, const uint64_t* __restrict__ cbp, uint32_t n_chrom,
                           uint4* __restrict__ out) {
  const uint64_t dmask = (uint64_t(1) << diag_bits) - 1;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_reads; r += gridDim.x * blockDim.x) {
    uint32_t o = kept_off[r];
    if (kept_off[r + 1] == o) continue;
    for (uint32_t i = off[r]; i < off[r + 1]; ++i) {
      const uint32_t v = svals[i];
      if (v == 0xFFFFFFFFu) continue;
      const uint64_t k = skeys[i];
      const uint64_t gs = (k >> 1) & dmask;
      uint32_t lo = 0, hi = n_chrom;  // largest c with cbp[c] <= gs
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(cbp + mid) <= gs) lo = mid; else hi = mid;
      }
      out[o++] = make_uint4(r, lo, uint32_t(gs - __ldg(cbp + lo)), (v & 0xFFFFu) | (uint32_t(k & 1) << 16));
    }
  }
}

// big segments: flag[i] = 1 for hits of reads with big[r] != 0
__global__ void k_big_flags(const uint64_t* __restrict__ skeys, uint64_t n, unsigned rshift,
                            const uint32_t* __restrict__ big, uint32_t* __restrict__ flags,
                            uint32_t* __restrict__ n_big) {
  uint32_t mine = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t f = big[skeys[i] >> rshift] != 0;
    flags[i] = f;
    mine += f;
  }
  mine = warp_reduce_sum(mine);
  if (lane_id() == 0 && mine) atomicAdd(n_big, mine);
}

__global__ void k_big_writeback(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t nb,
                                const uint32_t* __restrict__ flags_pos, const uint32_t* __restrict__ flags,
                                uint64_t n, uint64_t* __restrict__ skeys, uint32_t* __restrict__ svals) {
  // the i-th flagged slot of the segment arrays receives the i-th sorted key
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    if (flags[i]) {
      const uint32_t j = flags_pos[i];
      skeys[i] = keys[j];
      svals[i] = vals[j];
    }
}

}  // namespace

uint64_t stratify_unsorted(Ctx& c, const Ref& ref, DBuf<uint64_t>& hit_keys, DBuf<uint32_t>& hit_vals, uint64_t n,
                           uint32_t n_reads, int mode, DBuf<uint8_t>& out) {
  if (n == 0 || n_reads == 0) {
    out.alloc(c, 16);
    return 0;
  }
  if (n > 0xFFFFFFFFull) throw InputError("strata: more than 2^32-1 hits");
  const unsigned rshift = ref.diag_bits + 1;
  const unsigned grid = unsigned(std::min<uint64_t>(ceil_div(n, 256), uint64_t(kSMs) * 16));
  const unsigned rgrid = unsigned(std::min<uint64_t>(ceil_div(n_reads, 128), uint64_t(kSMs) * 16));
  DBuf<uint32_t> cnt(c, uint64_t(n_reads) + 1), off(c, uint64_t(n_reads) + 1), kept(c, uint64_t(n_reads) + 1),
      big(c, n_reads), total(c, 2);
  cnt.zero();
  kept.zero();
  {
    KernelScope ks(c, "k_strata_seg");
    QGM_KERNEL(c, k_count_reads, grid, 256, 0, hit_keys.p, n, rshift, cnt.p);
    exclusive_scan_u32(c, cnt.p, off.p, uint64_t(n_reads) + 1, nullptr, nullptr);
    DBuf<uint64_t> skeys(c, n);
    DBuf<uint32_t> svals(c, n);
    QGM_KERNEL(c, k_scatter_reads, grid, 256, 0, hit_keys.p, hit_vals.p, n, rshift, off.p, cnt.p, skeys.p, svals.p);
    QGM_KERNEL(c, k_seg_reduce, rgrid, 128, 0, skeys.p, svals.p, off.p, n_reads, mode, 0, kept.p, big.p);
    // reads with more than kSmallSeg hits: radix-sort their hits, write them
    // back into their segments, reduce them (one host round trip when there
    // are none: their hit count is read back together with the kept total)
    DBuf<uint32_t> flags(c, n), fpos(c, n), kept_off(c, uint64_t(n_reads) + 1);
    total.zero();
    QGM_KERNEL(c, k_big_flags, grid, 256, 0, skeys.p, n, rshift, big.p, flags.p, total.p);
    exclusive_scan_u32(c, kept.p, kept_off.p, uint64_t(n_reads) + 1, total.p + 1, nullptr);
    uint32_t h[2] = {0, 0};
    QGM_CUDA(cudaMemcpyAsync(h, total.p, 8, cudaMemcpyDeviceToHost, c.stream));
    QGM_CUDA(cudaStreamSynchronize(c.stream));
    const uint32_t nb = h[0];
    if (nb) {
      exclusive_scan_u32(c, flags.p, fpos.p, n, nullptr, nullptr);
      DBuf<uint64_t> bk(c, nb), bk_alt;
      DBuf<uint32_t> bv(c, nb), bv_alt;
      select_u64(c, skeys.p, svals.p, flags.p, n, bk.p, bv.p);
      radix_sort(c, bk, bk_alt, &bv, &bv_alt, nb, 0, int(rshift + bit_width_u64(n_reads)));
      QGM_KERNEL(c, k_big_writeback, grid, 256, 0, bk.p, bv.p, nb, fpos.p, flags.p, n, skeys.p, svals.p);
      QGM_KERNEL(c, k_seg_reduce, rgrid, 128, 0, skeys.p, svals.p, off.p, n_reads, mode, 1, kept.p, big.p);
      exclusive_scan_u32(c, kept.p, kept_off.p, uint64_t(n_reads) + 1, total.p + 1, nullptr);
      QGM_CUDA(cudaMemcpyAsync(h + 1, total.p + 1, 4, cudaMemcpyDeviceToHost, c.stream));
      QGM_CUDA(cudaStreamSynchronize(c.stream));
    }
    const uint32_t nk = h[1];
    out.alloc(c, std::max<uint64_t>(uint64_t(nk) * 16, 16));
    QGM_KERNEL(c, k_seg_emit, rgrid, 128, 0, skeys.p, svals.p, off.p, kept_off.p, n_reads, ref.diag_bits, ref.d_cbp.p,
               ref.n_chrom, reinterpret_cast<uint4*>(out.p));
    return nk;
  }
}

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
