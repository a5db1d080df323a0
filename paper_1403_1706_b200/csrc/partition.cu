// partition.cu -- per-batch read q-gram partition for the join (map path).
//
// The join (join.cu) only needs the batch's read q-grams grouped by the top
// bits of their code, so that the warps in flight touch a few MiB of the
// reference index (L2-resident) instead of all of it; it never needs the full
// read-side q-group index. Two passes over the (L2-resident) 2-bit reads, no
// per-item rank array:
//   P0 histogram : per-CTA shared-memory histogram over 2^bits code bins
//                  (bits = min(2q, 8)), one global atomic per non-empty bin;
//   scan         : bin offsets;
//   P1 scatter   : per chunk of 4096 q-gram slots, a local counting sort by
//                  bin in shared memory, one global atomic per bin to reserve
//                  the chunk's run, then runs copied out with consecutive
//                  threads writing consecutive 8-byte slots (full sectors;
//                  ~16 items = one 128 B line per bin per chunk at q=16).
// ncu on the previous single-pass scatter (12-bit bins, items written
// straight from registers) showed 1.6 GB of read-for-ownership and 2.1 GB of
// writes for 0.68 GB of output: partial sectors of 2.4M concurrently open runs.
// q-grams are keyed by their canonical code min(g, rc(g)) (RefQIndex).
// First-pass item = (canonical code << 32) | text position (r*stride + o);
// the refinement pass writes the final join items (internal.hpp: position,
// tail, the two run-start compare bases, the code bits below the sub-bin), so
// the join never touches the read text.
#include "internal.hpp"

namespace qgm {
namespace {

constexpr int kPartThreads = 512;
constexpr unsigned kBinBits = 8;
constexpr uint32_t kBins = 1u << kBinBits;
constexpr uint32_t kChunk = 4096;  // q-gram slots per chunk; staging = 32 KiB
constexpr uint32_t kPer = kChunk / kPartThreads;

struct ItemGen {
  const uint64_t* words;
  const uint32_t* lengths;
  uint32_t W, span, stride;
  FastDiv by_span;
  unsigned q;
  __device__ __forceinline__ bool item(uint32_t t, uint32_t& g, uint32_t& pos) const {
    const uint32_t r = by_span.div(t);
    const uint32_t o = t - r * span;
    if (o + q > __ldg(lengths + r)) return false;
    const uint32_t f = qgram_at(words + uint64_t(r) * W, o, q);
    g = min(f, rc_code(f, q));  // canonical code (RefQIndex)
    pos = r * stride + o;
    return true;
  }
};

__global__ void __launch_bounds__(kPartThreads) k_part_hist(ItemGen gen, uint32_t n_items, uint32_t chunk,
                                                            unsigned shift, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[kBins];
  for (uint32_t b = threadIdx.x; b < kBins; b += kPartThreads) h[b] = 0;
  __syncthreads();
  const uint32_t c0 = blockIdx.x * chunk, c1 = min(n_items, c0 + chunk);
  for (uint32_t t = c0 + threadIdx.x; t < c1; t += kPartThreads) {
    uint32_t g, pos;
    if (gen.item(t, g, pos)) atomicAdd(h + (g >> shift), 1u);
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < kBins; b += kPartThreads)
    if (h[b]) atomicAdd(hist + b, h[b]);
}

__global__ void __launch_bounds__(kPartThreads, 4) k_part_scatter(ItemGen gen, uint32_t n_items, unsigned shift,
                                                                  const uint32_t* __restrict__ boff,
                                                                  uint32_t* __restrict__ cursor,
                                                                  uint64_t* __restrict__ out) {
  extern __shared__ uint64_t stage[];  // kChunk items, bin-sorted
  __shared__ uint32_t cnt[kBins], lofs[kBins], gdst[kBins];
  __shared__ uint32_t ws[33];
  const uint32_t n_chunks = (n_items + kChunk - 1) / kChunk;
  for (uint32_t ch = blockIdx.x; ch < n_chunks; ch += gridDim.x) {
    const uint32_t c0 = ch * kChunk;
    for (uint32_t b = threadIdx.x; b < kBins; b += kPartThreads) cnt[b] = 0;
    __syncthreads();
    uint32_t g[kPer], pos[kPer];
    bool ok[kPer];
#pragma unroll
    for (uint32_t k = 0; k < kPer; ++k) {
      const uint32_t t = c0 + k * kPartThreads + threadIdx.x;
      ok[k] = t < n_items && gen.item(t, g[k], pos[k]);
      if (ok[k]) atomicAdd(cnt + (g[k] >> shift), 1u);
    }
    __syncthreads();
    {  // local exclusive offsets; reserve the chunk's run in every bin
      const uint32_t b = threadIdx.x;
      const uint32_t v = b < kBins ? cnt[b] : 0u;
      uint32_t tot;
      const uint32_t ex = block_exclusive_scan<uint32_t>(v, ws, &tot);
      if (b < kBins) {
        lofs[b] = ex;
        gdst[b] = v ? boff[b] + atomicAdd(cursor + b, v) : 0u;
        cnt[b] = ex;  // becomes the local placement cursor
      }
    }
    __syncthreads();
#pragma unroll
    for (uint32_t k = 0; k < kPer; ++k)
      if (ok[k]) stage[atomicAdd(cnt + (g[k] >> shift), 1u)] = (uint64_t(g[k]) << 32) | pos[k];
    __syncthreads();
    const uint32_t total = cnt[kBins - 1];  // == number of valid items in the chunk
    for (uint32_t i = threadIdx.x; i < total; i += kPartThreads) {
      const uint64_t it = stage[i];
      const uint32_t b = uint32_t(it >> 32) >> shift;
      out[gdst[b] + (i - lofs[b])] = it;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- refinement
// Second MSD pass: items already grouped by their top 8 code bits are
// regrouped by their top `key_bits` (<= 16) bits. A chunk of 4096 consecutive
// items spans few top-8 bins, so its keys fall in a small window
// [first_bin << sub, (last_bin + 1) << sub); the window is counted and
// staged in shared memory exactly like P1 (kLocal keys max), with a
// per-item global fallback for chunks whose window is wider (tiny bins).
constexpr uint32_t kLocal = 2048;

__device__ __forceinline__ uint32_t key_of(uint64_t it, unsigned kshift) { return uint32_t(it >> 32) >> kshift; }

// first-pass item -> join item (layout in internal.hpp). The read words and
// lengths are L2-resident; consecutive items of a chunk come from ascending
// reads.
struct ItemConv {
  const uint64_t* words;
  const uint32_t* lengths;
  uint32_t W, stride;
  FastDiv by_stride;
  unsigned q;
  uint32_t lmask;  // code bits below the sub-bin prefix
  __device__ __forceinline__ uint64_t operator()(uint64_t it) const {
    const uint32_t pp = uint32_t(it), c = uint32_t(it >> 32);
    const uint32_t r = by_stride.div(pp), o = pp - r * stride;
    // all loads depend only on (r, o): issue them together
    const uint32_t n = __ldg(lengths + r);
    const uint64_t* w = words + uint64_t(r) * W;
    const uint32_t f = qgram_at(w, o, q);
    const uint32_t bf = base_at(w, o ? o - 1 : 0);
    const uint32_t br = base_at(w, min(o + q, stride - 1));
    const uint32_t fb = o ? bf : 4u;
    const uint32_t rb = o + q < n ? 3u - br : 4u;
    const uint32_t tail = min(n - q - o, kItemTailMax);
    return (uint64_t(c & lmask) << kItemCodeShift) | (uint64_t(f != c) << kItemFrShift) |
           (uint64_t(rb) << kItemRbShift) | (uint64_t(fb) << kItemFbShift) | (uint64_t(tail) << kItemTailShift) | pp;
  }
};

__global__ void __launch_bounds__(kPartThreads) k_refine_hist(const uint64_t* __restrict__ in, uint32_t n,
                                                              unsigned kshift, unsigned sub,
                                                              uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[kLocal];
  const uint32_t n_chunks = (n + kChunk - 1) / kChunk;
  for (uint32_t ch = blockIdx.x; ch < n_chunks; ch += gridDim.x) {
    const uint32_t c0 = ch * kChunk, c1 = min(n, c0 + kChunk);
    const uint32_t base = (key_of(in[c0], kshift) >> sub) << sub;
    const uint32_t width = (((key_of(in[c1 - 1], kshift) >> sub) + 1) << sub) - base;
    if (width > kLocal) {  // rare: many tiny bins in one chunk
      for (uint32_t i = c0 + threadIdx.x; i < c1; i += kPartThreads) atomicAdd(hist + key_of(in[i], kshift), 1u);
      continue;
    }
    for (uint32_t b = threadIdx.x; b < width; b += kPartThreads) h[b] = 0;
    __syncthreads();
    for (uint32_t i = c0 + threadIdx.x; i < c1; i += kPartThreads) atomicAdd(h + key_of(in[i], kshift) - base, 1u);
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < width; b += kPartThreads)
      if (h[b]) atomicAdd(hist + base + b, h[b]);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kPartThreads, 2) k_refine_scatter(const uint64_t* __restrict__ in, uint32_t n,
                                                                    unsigned kshift, unsigned sub,
                                                                    const uint32_t* __restrict__ off,
                                                                    uint32_t* __restrict__ cursor,
                                                                    ItemConv conv, uint64_t* __restrict__ out) {
  extern __shared__ uint64_t stage[];  // kChunk converted items, then kChunk u16 window keys
  uint16_t* skey = reinterpret_cast<uint16_t*>(stage + kChunk);
  __shared__ uint32_t cnt[kLocal], lofs[kLocal], gdst[kLocal];
  __shared__ uint32_t ws[33];
  const uint32_t n_chunks = (n + kChunk - 1) / kChunk;
  for (uint32_t ch = blockIdx.x; ch < n_chunks; ch += gridDim.x) {
    const uint32_t c0 = ch * kChunk, c1 = min(n, c0 + kChunk);
    const uint32_t base = (key_of(in[c0], kshift) >> sub) << sub;
    const uint32_t width = (((key_of(in[c1 - 1], kshift) >> sub) + 1) << sub) - base;
    if (width > kLocal) {
      for (uint32_t i = c0 + threadIdx.x; i < c1; i += kPartThreads) {
        const uint64_t it = in[i];
        const uint32_t k = key_of(it, kshift);
        out[off[k] + atomicAdd(cursor + k, 1u)] = conv(it);
      }
      continue;
    }
    for (uint32_t b = threadIdx.x; b < width; b += kPartThreads) cnt[b] = 0;
    __syncthreads();
    // convert on load: consecutive first-pass items come from the same few
    // reads, so the read-word / length loads of a warp hit the same lines
    uint64_t v[kPer];
    uint32_t kk[kPer];
#pragma unroll
    for (uint32_t k = 0; k < kPer; ++k) {
      const uint32_t i = c0 + k * kPartThreads + threadIdx.x;
      const uint64_t it = i < c1 ? in[i] : 0ull;
      kk[k] = i < c1 ? key_of(it, kshift) - base : ~0u;
      v[k] = i < c1 ? conv(it) : 0ull;
      if (i < c1) atomicAdd(cnt + kk[k], 1u);
    }
    __syncthreads();
    // exclusive scan of cnt[0, width): each thread owns a contiguous run
    const uint32_t per = (width + kPartThreads - 1) / kPartThreads;
    const uint32_t b0 = threadIdx.x * per, b1 = min(width, b0 + per);
    uint32_t s = 0;
    for (uint32_t b = b0; b < b1; ++b) s += cnt[b];
    uint32_t tot;
    uint32_t run = block_exclusive_scan<uint32_t>(s, ws, &tot);
    for (uint32_t b = b0; b < b1; ++b) {
      const uint32_t cv = cnt[b];
      lofs[b] = run;
      gdst[b] = cv ? off[base + b] + atomicAdd(cursor + base + b, cv) : 0u;
      cnt[b] = run;
      run += cv;
    }
    __syncthreads();
#pragma unroll
    for (uint32_t k = 0; k < kPer; ++k)
      if (kk[k] != ~0u) {
        const uint32_t slot = atomicAdd(cnt + kk[k], 1u);
        stage[slot] = v[k];
        skey[slot] = uint16_t(kk[k]);
      }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < c1 - c0; i += kPartThreads) {
      const uint32_t b = skey[i];
      out[gdst[b] + (i - lofs[b])] = stage[i];
    }
    __syncthreads();
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
  gen.by_span = FastDiv(std::max<uint32_t>(gen.span, 1));
  gen.q = q;
  const uint64_t n_items64 = uint64_t(reads.n) * gen.span;
  if (n_items64 > 0xFFFFFFFFull - kChunk) throw InputError("read batch has more than 2^32-1 q-gram slots");
  const uint32_t n_items = uint32_t(n_items64);
  const unsigned bits = std::min(2 * q, kBinBits);
  const unsigned shift = 2 * q - bits;
  out.q = q;
  out.bins = 1u << bits;
  out.boff.alloc(c, kBins + 1);
  if (n_items == 0) {
    out.boff.zero();
    out.V = 0;
    out.pairs.alloc(c, 1);
    return;
  }
  const uint32_t chunk = uint32_t(std::max<uint64_t>(kChunk, ceil_div(n_items, uint64_t(kSMs) * 8)));
  DBuf<uint32_t> hist(c, kBins + 1);
  hist.zero();
  {
    KernelScope ks(c, "k_part_hist");
    QGM_KERNEL(c, k_part_hist, unsigned(ceil_div(n_items, chunk)), kPartThreads, 0, gen, n_items, chunk, shift,
               hist.p);
  }
  DBuf<uint32_t> total(c, 1);
  exclusive_scan_u32(c, hist.p, out.boff.p, kBins + 1, total.p, nullptr);
  uint32_t V = 0;
  QGM_CUDA(cudaMemcpyAsync(&V, total.p, 4, cudaMemcpyDeviceToHost, c.stream));
  QGM_CUDA(cudaStreamSynchronize(c.stream));
  out.V = V;
  out.pairs.alloc(c, std::max<uint64_t>(V, 1));
  hist.zero();  // reused as the per-bin global cursors
  const size_t smem = kChunk * sizeof(uint64_t);
  QGM_CUDA(cudaFuncSetAttribute(k_part_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const unsigned grid = unsigned(std::min<uint64_t>(ceil_div(n_items, kChunk), uint64_t(kSMs) * 4));
  {
    KernelScope ks(c, "k_part_scatter");
    QGM_KERNEL(c, k_part_scatter, grid, kPartThreads, smem, gen, n_items, shift, out.boff.p, hist.p, out.pairs.p);
  }
  // P2: refine to the top min(2q, 16) code bits (short reuse distance of the
  // reference-index sectors in the join) and convert to join items. Runs even
  // when the first pass already grouped by every key bit (2q <= 8): then it
  // only converts.
  const unsigned key_bits = std::min(2 * q, 16u);
  out.sub_bits = key_bits;
  if (V == 0) {  // every read shorter than q
    out.soff.alloc(c, (1u << key_bits) + 1);
    out.soff.zero();
    return;
  }
  const unsigned kshift = 2 * q - key_bits, sub = key_bits - bits;
  const uint32_t keys = 1u << key_bits;
  DBuf<uint32_t> h2(c, keys + 1);
  out.soff.alloc(c, keys + 1);
  DBuf<uint32_t>& off = out.soff;
  h2.zero();
  const unsigned grid2 = unsigned(std::min<uint64_t>(ceil_div(V, kChunk), uint64_t(kSMs) * 4));
  {
    KernelScope ks(c, "k_refine_hist");
    QGM_KERNEL(c, k_refine_hist, grid2, kPartThreads, 0, out.pairs.p, V, kshift, sub, h2.p);
  }
  exclusive_scan_u32(c, h2.p, off.p, keys + 1, nullptr, nullptr);
  h2.zero();  // per-key cursors
  DBuf<uint64_t> refined(c, std::max<uint64_t>(V, 1));
  const size_t smem2 = kChunk * (sizeof(uint64_t) + sizeof(uint16_t));
  QGM_CUDA(cudaFuncSetAttribute(k_refine_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2)));
  ItemConv conv;
  conv.words = reads.words.p;
  conv.lengths = reads.lengths.p;
  conv.W = reads.W;
  conv.stride = reads.stride;
  conv.by_stride = FastDiv(std::max<uint32_t>(reads.stride, 1));
  conv.q = q;
  conv.lmask = kshift ? (1u << kshift) - 1u : 0u;
  {
    KernelScope ks(c, "k_refine_scatter");
    QGM_KERNEL(c, k_refine_scatter, grid2, kPartThreads, smem2, out.pairs.p, V, kshift, sub, off.p, h2.p, conv,
               refined.p);
  }
  out.pairs.swap(refined);
}

}  // namespace qgm
