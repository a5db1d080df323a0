// partition.cu -- per-batch read q-gram partition for the join (map path).
//
// The join (join.cu) only needs the batch's read q-grams grouped by the top
// bits of their code, so that consecutive items touch the same few KiB of the
// reference index; it never needs the full read-side index. Two passes over
// the (L2-resident) 2-bit reads, no per-item rank array:
//   P0 histogram : per-CTA shared-memory histogram over 2^cbits code bins
//                  (cbits = min(2q, 12)), one global atomic per non-empty bin;
//   scan         : bin offsets;
//   P1 scatter   : the CTA re-derives its items, reserves one contiguous run
//                  per bin with one global atomic, and writes its items into
//                  the run through shared-memory cursors, so each bin receives
//                  a contiguous block of ~35 items (coalesced) per CTA.
// Item = (full code << 32) | text position (r*stride + o), 8 bytes.
#include "internal.hpp"

namespace qgm {
namespace {

constexpr int kPartThreads = 512;
constexpr unsigned kMaxBinBits = 12;

struct ItemGen {
  const uint64_t* words;
  const uint32_t* lengths;
  uint32_t W, span, stride;
  FastDiv by_span;
  unsigned q;
  __device__ __forceinline__ bool item(uint64_t t, uint32_t& g, uint32_t& pos) const {
    const uint32_t r = by_span.div(uint32_t(t));  // slots < 2^32 (checked on the host)
    const uint32_t o = uint32_t(t) - r * span;
    if (o + q > __ldg(lengths + r)) return false;
    g = qgram_at(words + uint64_t(r) * W, o, q);
    pos = r * stride + o;
    return true;
  }
};

__global__ void __launch_bounds__(kPartThreads) k_part_hist(ItemGen gen, uint64_t n_items, uint64_t chunk,
                                                            unsigned shift, uint32_t bins, uint32_t* __restrict__ hist) {
  extern __shared__ uint32_t h[];
  for (uint32_t b = threadIdx.x; b < bins; b += kPartThreads) h[b] = 0;
  __syncthreads();
  const uint64_t c0 = blockIdx.x * chunk, c1 = min(n_items, c0 + chunk);
  for (uint64_t t = c0 + threadIdx.x; t < c1; t += kPartThreads) {
    uint32_t g, pos;
    if (gen.item(t, g, pos)) atomicAdd(h + (g >> shift), 1u);
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < bins; b += kPartThreads)
    if (h[b]) atomicAdd(hist + b, h[b]);
}

__global__ void __launch_bounds__(kPartThreads) k_part_scatter(ItemGen gen, uint64_t n_items, uint64_t chunk,
                                                               unsigned shift, uint32_t bins,
                                                               const uint32_t* __restrict__ boff,
                                                               uint32_t* __restrict__ cursor,
                                                               uint64_t* __restrict__ out) {
  extern __shared__ uint32_t h[];  // [bins] counts -> run bases, [bins] local cursors
  uint32_t* cur = h + bins;
  for (uint32_t b = threadIdx.x; b < bins; b += kPartThreads) { h[b] = 0; cur[b] = 0; }
  __syncthreads();
  const uint64_t c0 = blockIdx.x * chunk, c1 = min(n_items, c0 + chunk);
  for (uint64_t t = c0 + threadIdx.x; t < c1; t += kPartThreads) {
    uint32_t g, pos;
    if (gen.item(t, g, pos)) atomicAdd(h + (g >> shift), 1u);
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < bins; b += kPartThreads)
    if (h[b]) h[b] = boff[b] + atomicAdd(cursor + b, h[b]);
  __syncthreads();
  for (uint64_t t = c0 + threadIdx.x; t < c1; t += kPartThreads) {
    uint32_t g, pos;
    if (!gen.item(t, g, pos)) continue;
    const uint32_t b = g >> shift;
    out[h[b] + atomicAdd(cur + b, 1u)] = (uint64_t(g) << 32) | pos;
  }
}

}  // namespace

void partition_reads(Ctx& c, const Reads& reads, unsigned q, Partitioned& out) {
  if (q == 0 || q > 16) throw InputError("q must be in [1, 16]");
  ItemGen gen;
  gen.words = reads.words.p;
  gen.lengths = reads.lengths.p;
  gen.W = reads.W;
  gen.span = reads.stride >= q ? reads.stride - q + 1 : 0;
  gen.stride = reads.stride;
  gen.q = q;
  gen.by_span = FastDiv(std::max<uint32_t>(gen.span, 1));
  const uint64_t n_items = uint64_t(reads.n) * gen.span;
  if (n_items > 0xFFFFFFFFull) throw InputError("read batch has more than 2^32-1 q-gram slots");
  const unsigned bits = std::min(2 * q, kMaxBinBits);
  const uint32_t bins = 1u << bits;
  const unsigned shift = 2 * q - bits;
  out.q = q;
  out.bins = bins;
  out.boff.alloc(c, bins + 1);
  if (n_items == 0) {
    out.boff.zero();
    out.V = 0;
    out.pairs.alloc(c, 1);
    return;
  }
  // ~36 items per bin per CTA keeps the per-bin runs coalesced
  const uint64_t chunk = std::max<uint64_t>(uint64_t(bins) * 36, ceil_div(n_items, uint64_t(kSMs) * 16));
  const unsigned grid = unsigned(ceil_div(n_items, chunk));
  DBuf<uint32_t> hist(c, bins + 1);
  hist.zero();
  {
    KernelScope ks(c, "k_part_hist");
    QGM_KERNEL(c, k_part_hist, grid, kPartThreads, bins * 4, gen, n_items, chunk, shift, bins, hist.p);
  }
  DBuf<uint32_t> total(c, 1);
  exclusive_scan_u32(c, hist.p, out.boff.p, bins + 1, total.p, nullptr);
  uint32_t V = 0;
  QGM_CUDA(cudaMemcpyAsync(&V, total.p, 4, cudaMemcpyDeviceToHost, c.stream));
  QGM_CUDA(cudaStreamSynchronize(c.stream));
  out.V = V;
  out.pairs.alloc(c, std::max<uint64_t>(V, 1));
  hist.zero();  // reused as the per-bin global cursors
  {
    KernelScope ks(c, "k_part_scatter");
    QGM_KERNEL(c, k_part_scatter, grid, kPartThreads, bins * 8, gen, n_items, chunk, shift, bins, out.boff.p, hist.p,
               out.pairs.p);
  }
}

}  // namespace qgm
