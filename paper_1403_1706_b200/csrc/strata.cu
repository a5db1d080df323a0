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
// kept counts places the records. A batch with a read of more than kSmallSeg
// hits (repeats; a thread would walk its segment serially) is instead radix-
// sorted as a whole and reduced by the sorted-input kernels below.
//
// Sorted-input path (stratify_hits, hits radix-sorted by the caller):
//   K1: first hit of every group keeps the group's minimum k and folds it
//       into the read's minimum with atomicMin;
//   K2: keep flag (all mode, or k == the read's minimum);
//   scan + K3: order-preserving compaction.
#include "internal.hpp"

namespace qgm {
uint64_t stratify_hits(Ctx& c, const Ref& ref, const uint64_t* hit_keys, const uint32_t* hit_vals, uint64_t n,
                       uint32_t n_reads, unsigned read_bits, int mode, DBuf<uint8_t>& out);
namespace {

__global__ void k_group_min(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t n,
                            unsigned diag_bits, uint32_t* __restrict__ readmin, uint32_t* __restrict__ first,
                            uint32_t* __restrict__ gmin) {
  QGM_GRID_DEP();
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
  QGM_GRID_DEP();
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    keep[i] = first[i] && (mode == 1 || gmin[i] == readmin[keys[i] >> (diag_bits + 1)]);
}

__global__ void k_emit(const uint64_t* __restrict__ keys, uint64_t n, unsigned diag_bits,
                       const uint32_t* __restrict__ keep, const uint32_t* __restrict__ pos,
                       const uint32_t* __restrict__ gmin, const uint64_t* __restrict__ cbp, uint32_t n_chrom,
                       uint4* __restrict__ out) {
  QGM_GRID_DEP();
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

// cnt[r] counts down while hits are placed (segment filled from its end).
// n_dev / big (nullable): device hit count, and the flag that hands the batch
// to the radix path (then nothing is placed)
__global__ void k_scatter_reads(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t n,
                                unsigned rshift, const uint32_t* __restrict__ off, uint32_t* __restrict__ cnt,
                                uint64_t* __restrict__ skeys, uint32_t* __restrict__ svals,
                                const unsigned long long* __restrict__ n_dev,
                                const unsigned long long* __restrict__ big) {
  QGM_GRID_DEP();
  if (big && *big) return;
  if (n_dev) n = *n_dev;
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
// per read (every segment <= kSmallSeg hits): sort the segment, group
// minima, the read's minimum, keep marks (value ~0u = dropped), kept count
__global__ void k_seg_reduce(uint64_t* __restrict__ skeys, uint32_t* __restrict__ svals,
                             const uint32_t* __restrict__ off, uint32_t n_reads, int mode,
                             uint32_t* __restrict__ kept, const unsigned long long* __restrict__ big) {
  QGM_GRID_DEP();
  // kept[0, n_reads] is written here in full (the scan after it reads n_reads
  // + 1 entries), also when the batch goes to the radix path (zeros then)
  if (blockIdx.x == 0 && threadIdx.x == 0) kept[n_reads] = 0;
  if (big && *big) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_reads; r += gridDim.x * blockDim.x) kept[r] = 0;
    return;
  }
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_reads; r += gridDim.x * blockDim.x) {
    const uint32_t b = off[r], m = off[r + 1] - b;
    uint32_t nk = 0;
    uint64_t* K = skeys + b;
    uint32_t* V = svals + b;
    for (uint32_t i = 1; i < m; ++i) {  // insertion sort by key
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
                           uint4* __restrict__ out, const unsigned long long* __restrict__ big) {
  QGM_GRID_DEP();
  if (big && *big) return;
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

// hit-rank: keys = read << 16 | edits of the output records,
// sorted; the rank of a record = #records of its read with edits <= its
// edits (identity is monotone in edits for a fixed read) = upper_bound(key) -
// lower_bound(read << 16) in the sorted keys.
__global__ void k_rank_keys(const uint4* __restrict__ hits, uint64_t n, uint64_t* __restrict__ keys,
                            uint32_t* __restrict__ idx) {
  QGM_GRID_DEP();
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint4 h = hits[i];
    keys[i] = (uint64_t(h.x) << 16) | (h.w & 0xFFFFu);
    idx[i] = uint32_t(i);
  }
}

__device__ __forceinline__ uint64_t lower_bound_u64(const uint64_t* a, uint64_t n, uint64_t v) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_ranks(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx, uint64_t n,
                        uint32_t* __restrict__ rank) {
  QGM_GRID_DEP();
  for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < n; j += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = keys[j];
    const uint64_t hi = lower_bound_u64(keys, n, k + 1), lo = lower_bound_u64(keys, n, (k >> 16) << 16);
    rank[idx[j]] = uint32_t(hi - lo);
  }
}

// hit-rank straight from the output order: the records of a read are
// contiguous (strata emits them read by read), so a record's rank is a count
// over its own run. Runs longer than kRankRun set *long_run and are left to
// the sorted path.
constexpr uint32_t kRankRun = 64;
__global__ void k_rank_runs(const uint4* __restrict__ hits, uint64_t n, uint32_t* __restrict__ rank,
                            unsigned int* __restrict__ long_run) {
  QGM_GRID_DEP();
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint4 h = __ldg(hits + i);
    const uint32_t e = h.w & 0xFFFFu;
    uint64_t lo = i, hi = i + 1;
    while (lo > 0 && i - lo < kRankRun && __ldg(&hits[lo - 1].x) == h.x) --lo;
    while (hi < n && hi - i < kRankRun && __ldg(&hits[hi].x) == h.x) ++hi;
    if (i - lo == kRankRun || hi - i == kRankRun) {
      atomicOr(long_run, 1u);
      continue;
    }
    uint32_t c = 0;
    for (uint64_t j = lo; j < hi; ++j) c += (__ldg(&hits[j].w) & 0xFFFFu) <= e;
    rank[i] = c;
  }
}

}  // namespace

void hit_ranks(Ctx& c, const DBuf<uint8_t>& hits, uint64_t n, uint32_t n_reads, DBuf<uint32_t>& rank) {
  rank.alloc(c, std::max<uint64_t>(n, 1));
  if (n == 0) return;
  KernelScope ks(c, "hit_rank");
  {
    DBuf<unsigned int> long_run(c, 1);
    long_run.zero();
    const unsigned g = unsigned(std::min<uint64_t>(ceil_div(n, 256), uint64_t(kSMs) * 16));
    QGM_KERNEL(c, k_rank_runs, g, 256, 0, reinterpret_cast<const uint4*>(hits.p), n, rank.p, long_run.p);
    unsigned int h_long = 0;
    read_back(c, {{long_run.p, &h_long, 4}});
    if (!h_long) return;
  }
  // a read with more than kRankRun records: sort (read, edits) keys
  DBuf<uint64_t> keys(c, n), keys_alt;
  DBuf<uint32_t> idx(c, n), idx_alt;
  const unsigned grid = unsigned(std::min<uint64_t>(ceil_div(n, 256), uint64_t(kSMs) * 16));
  QGM_KERNEL(c, k_rank_keys, grid, 256, 0, reinterpret_cast<const uint4*>(hits.p), n, keys.p, idx.p);
  radix_sort(c, keys, keys_alt, &idx, &idx_alt, n, 0, int(16 + bit_width_u64(n_reads)));
  QGM_KERNEL(c, k_ranks, grid, 256, 0, keys.p, idx.p, n, rank.p);
}

uint64_t stratify_unsorted(Ctx& c, const Ref& ref, DBuf<uint64_t>& hit_keys, DBuf<uint32_t>& hit_vals, uint64_t n,
                           uint32_t n_reads, int mode, DBuf<uint32_t>& cnt, bool big, DBuf<uint8_t>& out) {
  if (n == 0 || n_reads == 0) {
    out.alloc(c, 16);
    return 0;
  }
  if (n > 0xFFFFFFFFull) throw InputError("strata: more than 2^32-1 hits");
  const unsigned rshift = ref.diag_bits + 1;
  KernelScope ks(c, "k_strata_seg");
  if (big) {
    // a read with more than kSmallSeg hits (repeats): a thread would walk its
    // segment serially -- sort every hit and use the sorted-input kernels
    DBuf<uint64_t> k_alt;
    DBuf<uint32_t> v_alt;
    radix_sort(c, hit_keys, k_alt, &hit_vals, &v_alt, n, 0, int(rshift + bit_width_u64(n_reads)));
    return stratify_hits(c, ref, hit_keys.p, hit_vals.p, n, n_reads, 0, mode, out);
  }
  const unsigned grid = unsigned(std::min<uint64_t>(ceil_div(n, 256), uint64_t(kSMs) * 16));
  const unsigned rgrid = unsigned(std::min<uint64_t>(ceil_div(n_reads, 128), uint64_t(kSMs) * 16));
  DBuf<uint32_t> off(c, uint64_t(n_reads) + 1), kept(c, uint64_t(n_reads) + 1), total(c, 1);  // kept: k_seg_reduce
  exclusive_scan_u32(c, cnt.p, off.p, uint64_t(n_reads) + 1, nullptr, nullptr);
  DBuf<uint64_t> skeys(c, n);
  DBuf<uint32_t> svals(c, n);
  QGM_KERNEL(c, k_scatter_reads, grid, 256, 0, hit_keys.p, hit_vals.p, n, rshift, off.p, cnt.p, skeys.p, svals.p,
             nullptr, nullptr);
  QGM_KERNEL(c, k_seg_reduce, rgrid, 128, 0, skeys.p, svals.p, off.p, n_reads, mode, kept.p, nullptr);
  DBuf<uint32_t> kept_off(c, uint64_t(n_reads) + 1);
  exclusive_scan_u32(c, kept.p, kept_off.p, uint64_t(n_reads) + 1, total.p, nullptr);
  uint32_t nk = 0;
  read_back(c, {{total.p, &nk, 4}});
  out.alloc(c, std::max<uint64_t>(uint64_t(nk) * 16, 16));
  QGM_KERNEL(c, k_seg_emit, rgrid, 128, 0, skeys.p, svals.p, off.p, kept_off.p, n_reads, ref.diag_bits, ref.d_cbp.p,
             ref.n_chrom, reinterpret_cast<uint4*>(out.p), nullptr);
  return nk;
}

void stratify_unsorted_dev(Ctx& c, const Ref& ref, const uint64_t* hit_keys, const uint32_t* hit_vals,
                           const unsigned long long* d_n, uint64_t n_max, uint32_t n_reads, int mode,
                           DBuf<uint32_t>& cnt, const unsigned long long* d_big, DBuf<uint8_t>& out,
                           uint32_t* d_kept) {
  out.alloc(c, std::max<uint64_t>(n_max * 16, 16));
  if (n_max == 0 || n_reads == 0) {
    fill_bytes(c, d_kept, 0, 4);
    return;
  }
  if (n_max > 0xFFFFFFFFull) throw InputError("strata: more than 2^32-1 hits");
  const unsigned rshift = ref.diag_bits + 1;
  KernelScope ks(c, "k_strata_seg");
  const unsigned grid = unsigned(std::min<uint64_t>(ceil_div(n_max, 256), uint64_t(kSMs) * 16));
  const unsigned rgrid = unsigned(std::min<uint64_t>(ceil_div(n_reads, 128), uint64_t(kSMs) * 16));
  DBuf<uint32_t> off(c, uint64_t(n_reads) + 1), kept(c, uint64_t(n_reads) + 1);  // kept: written by k_seg_reduce
  exclusive_scan_u32(c, cnt.p, off.p, uint64_t(n_reads) + 1, nullptr, nullptr);
  DBuf<uint64_t> skeys(c, n_max);
  DBuf<uint32_t> svals(c, n_max);
  QGM_KERNEL(c, k_scatter_reads, grid, 256, 0, hit_keys, hit_vals, n_max, rshift, off.p, cnt.p, skeys.p, svals.p, d_n,
             d_big);
  QGM_KERNEL(c, k_seg_reduce, rgrid, 128, 0, skeys.p, svals.p, off.p, n_reads, mode, kept.p, d_big);
  DBuf<uint32_t> kept_off(c, uint64_t(n_reads) + 1);
  exclusive_scan_u32(c, kept.p, kept_off.p, uint64_t(n_reads) + 1, d_kept, nullptr);
  QGM_KERNEL(c, k_seg_emit, rgrid, 128, 0, skeys.p, svals.p, off.p, kept_off.p, n_reads, ref.diag_bits, ref.d_cbp.p,
             ref.n_chrom, reinterpret_cast<uint4*>(out.p), d_big);
}

uint64_t stratify_hits(Ctx& c, const Ref& ref, const uint64_t* hit_keys, const uint32_t* hit_vals, uint64_t n,
                       uint32_t n_reads, unsigned read_bits, int mode, DBuf<uint8_t>& out) {
  (void)read_bits;
  if (n == 0) {
    out.alloc(c, 16);
    return 0;
  }
  DBuf<uint32_t> readmin(c, std::max<uint32_t>(n_reads, 1));
  fill_bytes(c, readmin.p, 0xFF, readmin.bytes());
  DBuf<uint32_t> first(c, n), gmin(c, n), keep(c, n), total(c, 1);
  const unsigned grid = unsigned(std::min<uint64_t>(ceil_div(n, 256), uint64_t(kSMs) * 16));
  QGM_KERNEL(c, k_group_min, grid, 256, 0, hit_keys, hit_vals, n, ref.diag_bits, readmin.p, first.p, gmin.p);
  QGM_KERNEL(c, k_keep, grid, 256, 0, hit_keys, n, ref.diag_bits, mode, readmin.p, first.p, gmin.p, keep.p);
  exclusive_scan_u32(c, keep.p, first.p, n, total.p, nullptr);  // first <- output slots
  uint32_t kept = 0;
  read_back(c, {{total.p, &kept, 4}});
  out.alloc(c, std::max<uint64_t>(uint64_t(kept) * 16, 16));
  QGM_KERNEL(c, k_emit, grid, 256, 0, hit_keys, n, ref.diag_bits, keep.p, first.p, gmin.p, ref.d_cbp.p, ref.n_chrom,
             reinterpret_cast<uint4*>(out.p));
  return kept;
}

}  // namespace qgm
