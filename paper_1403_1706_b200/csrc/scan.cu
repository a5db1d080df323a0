// scan.cu -- device exclusive scan and order-preserving selection: the B200
// equivalents of par::exclusive_scan_in_place (parallel.hpp:64-108, with the
// u32 overflow check of :53-58) and par::compact (parallel.hpp:124-141).
//
// Reduce-then-scan over 4096-element tiles: (1) per-tile u64 sums, (2) one
// CTA scans the tile sums, (3) every tile re-reads its elements, scans them in
// shared memory and writes out. HBM traffic: 2 reads + 1 write per element.
// Up to 2^14 elements one CTA scans them in registers (k_scan_single).
#include "internal.hpp"

#include <cstdlib>
#include <cstring>
#include <stdexcept>

namespace qgm {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanPer = 16;
constexpr int kScanTile = kScanThreads * kScanPer;

__device__ __forceinline__ uint32_t pad_idx(uint32_t i) { return i + (i >> 5); }

__global__ void __launch_bounds__(kScanThreads) k_tile_sums(const uint32_t* __restrict__ in, uint64_t n,
                                                            uint64_t* __restrict__ sums) {
  QGM_GRID_DEP();
  __shared__ uint64_t ws[33];
  const uint64_t base = uint64_t(blockIdx.x) * kScanTile;
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    const uint64_t i = base + uint64_t(j) * kScanThreads + threadIdx.x;
    if (i < n) s += in[i];
  }
  uint64_t tot;
  block_exclusive_scan<uint64_t>(s, ws, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_sums(uint64_t* __restrict__ sums, uint64_t n_tiles,
                                                    uint32_t* __restrict__ d_total, int* __restrict__ d_overflow) {
  QGM_GRID_DEP();
  __shared__ uint64_t ws[33];
  uint64_t carry = 0;
  for (uint64_t b = 0; b < n_tiles; b += blockDim.x) {
    const uint64_t i = b + threadIdx.x;
    const uint64_t v = i < n_tiles ? sums[i] : 0;
    uint64_t tot;
    const uint64_t ex = block_exclusive_scan<uint64_t>(v, ws, &tot);
    if (i < n_tiles) sums[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    if (d_total) *d_total = uint32_t(carry);
    if (d_overflow) *d_overflow = carry > 0xFFFFFFFFull ? 1 : 0;
  }
}

__global__ void __launch_bounds__(kScanThreads) k_tile_scan(const uint32_t* in, uint32_t* out, uint64_t n,
                                                            const uint64_t* __restrict__ sums) {
  QGM_GRID_DEP();
  __shared__ uint32_t tile[kScanTile + kScanTile / 32];
  __shared__ uint64_t ws[33];
  const uint64_t base = uint64_t(blockIdx.x) * kScanTile;
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    const uint32_t li = j * kScanThreads + threadIdx.x;
    const uint64_t i = base + li;
    tile[pad_idx(li)] = i < n ? in[i] : 0u;
  }
  __syncthreads();
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) s += tile[pad_idx(threadIdx.x * kScanPer + j)];
  uint64_t run = block_exclusive_scan<uint64_t>(s, ws, nullptr) + sums[blockIdx.x];
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    const uint32_t li = pad_idx(threadIdx.x * kScanPer + j);
    const uint32_t v = tile[li];
    tile[li] = uint32_t(run);
    run += v;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    const uint32_t li = j * kScanThreads + threadIdx.x;
    const uint64_t i = base + li;
    if (i < n) out[i] = tile[pad_idx(li)];
  }
}

// Small inputs (the partition's key offsets, per-read counts of small
// batches): one CTA, one tile; every thread scans 16 consecutive elements in
// registers (16-byte vector loads and stores when aligned). One launch instead
// of three, one read and one write per element.
constexpr int kSingleThreads = 1024;
constexpr uint64_t kSingleMax = uint64_t(kSingleThreads) * kScanPer;

__global__ void __launch_bounds__(kSingleThreads) k_scan_single(const uint32_t* in, uint32_t* out, uint64_t n,
                                                                uint32_t* __restrict__ d_total,
                                                                int* __restrict__ d_overflow) {
  QGM_GRID_DEP();
  __shared__ uint64_t ws[33];
  static_assert(kScanPer % 4 == 0, "");
  const uint64_t b = uint64_t(threadIdx.x) * kScanPer;
  const bool vec = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0 &&
                   b + kScanPer <= n;
  uint32_t v[kScanPer];
  if (vec) {
#pragma unroll
    for (int j = 0; j < kScanPer / 4; ++j) {
      const uint4 x = reinterpret_cast<const uint4*>(in + b)[j];
      v[4 * j] = x.x;
      v[4 * j + 1] = x.y;
      v[4 * j + 2] = x.z;
      v[4 * j + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) v[j] = b + j < n ? in[b + j] : 0u;
  }
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) s += v[j];
  uint64_t tot;
  // in == out is allowed: the scan's barriers order every read before any write
  uint64_t run = block_exclusive_scan<uint64_t>(s, ws, &tot);
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    const uint32_t x = v[j];
    v[j] = uint32_t(run);
    run += x;
  }
  if (vec) {
#pragma unroll
    for (int j = 0; j < kScanPer / 4; ++j)
      reinterpret_cast<uint4*>(out + b)[j] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  } else {
#pragma unroll
    for (int j = 0; j < kScanPer; ++j)
      if (b + j < n) out[b + j] = v[j];
  }
  if (threadIdx.x == 0) {
    if (d_total) *d_total = uint32_t(tot);
    if (d_overflow) *d_overflow = tot > 0xFFFFFFFFull ? 1 : 0;
  }
}

__global__ void k_select_flags(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ flags, uint64_t n,
                               uint32_t* __restrict__ f) {
  QGM_GRID_DEP();
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    f[i] = flags ? (flags[i] != 0) : (i == 0 || keys[i] != keys[i - 1]);
}

__global__ void k_select_scatter(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                                 const uint32_t* __restrict__ flags, const uint32_t* __restrict__ pos, uint64_t n,
                                 uint64_t* __restrict__ out_keys, uint32_t* __restrict__ out_vals) {
  QGM_GRID_DEP();
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const bool sel = flags ? (flags[i] != 0) : (i == 0 || keys[i] != keys[i - 1]);
    if (sel) {
      out_keys[pos[i]] = keys[i];
      if (vals) out_vals[pos[i]] = vals[i];
    }
  }
}

}  // namespace

void exclusive_scan_u32(Ctx& c, const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* d_total,
                        int* d_overflow) {
  if (n == 0) {
    if (d_total) fill_bytes(c, d_total, 0, sizeof(uint32_t));
    if (d_overflow) fill_bytes(c, d_overflow, 0, sizeof(int));
    return;
  }
  if (n <= kSingleMax) {
    QGM_KERNEL(c, k_scan_single, 1, kSingleThreads, 0, in, out, n, d_total, d_overflow);
    return;
  }
  const uint64_t tiles = ceil_div(n, kScanTile);
  DBuf<uint64_t> sums(c, tiles);
  QGM_KERNEL(c, k_tile_sums, unsigned(tiles), kScanThreads, 0, in, n, sums.p);
  QGM_KERNEL(c, k_scan_sums, 1, 1024, 0, sums.p, tiles, d_total, d_overflow);
  QGM_KERNEL(c, k_tile_scan, unsigned(tiles), kScanThreads, 0, in, out, n, sums.p);
}

uint64_t select_u64(Ctx& c, const uint64_t* keys, const uint32_t* vals, const uint32_t* flags, uint64_t n,
                    uint64_t* out_keys, uint32_t* out_vals) {
  if (n == 0) return 0;
  DBuf<uint32_t> f(c, n);
  DBuf<uint32_t> total(c, 1);
  const unsigned grid = unsigned(std::min<uint64_t>(ceil_div(n, 256), uint64_t(kSMs) * 16));
  QGM_KERNEL(c, k_select_flags, grid, 256, 0, keys, flags, n, f.p);
  exclusive_scan_u32(c, f.p, f.p, n, total.p, nullptr);
  QGM_KERNEL(c, k_select_scatter, grid, 256, 0, keys, vals, flags, f.p, n, out_keys, out_vals);
  uint32_t h = 0;
  read_back(c, {{total.p, &h, sizeof(h)}});
  return h;
}

namespace {
__global__ void __launch_bounds__(256) k_fill_bytes(uint8_t* __restrict__ p, uint32_t pattern, size_t bytes) {
  QGM_GRID_DEP();
  const size_t head = std::min<size_t>(bytes, (16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15);
  const size_t body = (bytes - head) / 16, tail = head + body * 16;
  const size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x, stride = size_t(gridDim.x) * blockDim.x;
  if (t < head) p[t] = uint8_t(pattern);
  if (t < bytes - tail) p[tail + t] = uint8_t(pattern);
  uint4* q = reinterpret_cast<uint4*>(p + head);
  const uint4 v = make_uint4(pattern, pattern, pattern, pattern);
  for (size_t i = t; i < body; i += stride) q[i] = v;
}
}  // namespace

namespace {
struct ReadSegs {
  const uint32_t* src[kMaxReadSegs];
  uint32_t words[kMaxReadSegs];
  int n;
};
// gathers small device counters into the context's mapped pinned page
__global__ void k_read_back(ReadSegs s, uint32_t* __restrict__ out) {
  QGM_GRID_DEP();
  uint32_t o = 0;
  for (int k = 0; k < s.n; ++k) {
    for (uint32_t i = threadIdx.x; i < s.words[k]; i += blockDim.x) out[o + i] = s.src[k][i];
    o += s.words[k];
  }
}
}  // namespace

void read_back(Ctx& c, std::initializer_list<ReadSeg> segs) {
  if (!c.tail_h) {
    QGM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c.tail_h), kReadBackBytes, cudaHostAllocMapped));
    QGM_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c.tail_d), c.tail_h, 0));
  }
  ReadSegs s{};
  size_t total = 0;
  for (const ReadSeg& g : segs) {
    if (s.n == kMaxReadSegs || g.bytes % 4 || total + g.bytes > kReadBackBytes)
      throw std::logic_error("read_back: too many or unaligned segments");
    s.src[s.n] = static_cast<const uint32_t*>(g.src);
    s.words[s.n++] = uint32_t(g.bytes / 4);
    total += g.bytes;
  }
  QGM_KERNEL(c, k_read_back, 1, 256, 0, s, c.tail_d);
  QGM_CUDA(cudaStreamSynchronize(c.stream));
  const uint8_t* h = reinterpret_cast<const uint8_t*>(c.tail_h);
  for (const ReadSeg& g : segs) {
    std::memcpy(g.dst, h, g.bytes);
    h += g.bytes;
  }
}

void fill_bytes(Ctx& c, void* p, int value, size_t bytes) {
  if (bytes == 0) return;
  const unsigned grid = unsigned(std::min<size_t>(std::max<size_t>(ceil_div(bytes, size_t(16) * 256), 1), kSMs * 8));
  QGM_KERNEL(c, k_fill_bytes, grid, 256, 0, static_cast<uint8_t*>(p), uint32_t(uint8_t(value)) * 0x01010101u, bytes);
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("QGM_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace qgm
