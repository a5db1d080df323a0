// radix_sort.cu -- stable LSD radix sort of u64 keys (+ optional u32 values),
// 8-bit digits over an arbitrary bit range. Used for the candidate sort/dedup
// (stage 3) and the hit sort of the strata reduction (stage 5).
//
// Per digit pass (reduce-then-scan):
//   upsweep   : per 2048-key tile, a shared-memory digit histogram, written
//               digit-major so one exclusive scan yields every (digit, tile)
//               output offset;
//   scan      : exclusive_scan_u32 over 256 x tiles counts;
//   downsweep : stable tile-local ranks (warp match_any + per-warp shared
//               counters), keys reordered by digit in shared memory, then
//               written out so consecutive threads write consecutive slots.
// HBM traffic per pass: 8 B read (upsweep) + 8 B read + 8 B write (downsweep)
// per key, +4/+4 B per value.
#include "internal.hpp"

namespace qgm {
namespace {

constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixPer = 8;
constexpr int kRadixTile = kRadixThreads * kRadixPer;  // 2048
constexpr int kBins = 256;

__device__ __forceinline__ uint32_t digit_of(uint64_t k, int shift) { return uint32_t(k >> shift) & 0xFFu; }

__global__ void __launch_bounds__(kRadixThreads) k_upsweep(const uint64_t* __restrict__ keys, uint64_t n, int shift,
                                                           uint32_t* __restrict__ hist, uint32_t n_tiles) {
  QGM_GRID_DEP();
  __shared__ uint32_t h[kBins];
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = uint64_t(blockIdx.x) * kRadixTile;
#pragma unroll
  for (int j = 0; j < kRadixPer; ++j) {
    const uint64_t i = base + uint64_t(j) * kRadixThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[digit_of(keys[i], shift)], 1u);
  }
  __syncthreads();
  hist[uint64_t(threadIdx.x) * n_tiles + blockIdx.x] = h[threadIdx.x];
}

template <bool kVals>
__global__ void __launch_bounds__(kRadixThreads) k_downsweep(const uint64_t* __restrict__ keys,
                                                             const uint32_t* __restrict__ vals, uint64_t n, int shift,
                                                             const uint32_t* __restrict__ offs, uint32_t n_tiles,
                                                             uint64_t* __restrict__ out_keys,
                                                             uint32_t* __restrict__ out_vals) {
  QGM_GRID_DEP();
  __shared__ uint32_t wcnt[kRadixWarps][kBins];
  __shared__ uint32_t tile_off[kBins];
  __shared__ uint32_t glob_off[kBins];
  __shared__ uint64_t skeys[kRadixTile];
  __shared__ uint32_t svals[kVals ? kRadixTile : 1];
  __shared__ uint32_t ws[33];

  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < kRadixWarps * kBins; d += kRadixThreads) (&wcnt[0][0])[d] = 0;
  glob_off[threadIdx.x] = offs[uint64_t(threadIdx.x) * n_tiles + blockIdx.x];
  __syncthreads();

  const uint64_t base = uint64_t(blockIdx.x) * kRadixTile;
  const uint32_t valid_in_tile = n - base < uint64_t(kRadixTile) ? uint32_t(n - base) : uint32_t(kRadixTile);
  uint64_t k[kRadixPer];
  uint32_t v[kRadixPer];
  uint32_t local[kRadixPer];
  // warp-striped: item (warp, round j, lane) -> tile index warp*256 + j*32 + lane
#pragma unroll
  for (int j = 0; j < kRadixPer; ++j) {
    const uint32_t ti = warp * (kRadixPer * 32) + j * 32 + lane;
    const bool ok = ti < valid_in_tile;
    k[j] = ok ? keys[base + ti] : 0;
    if (kVals) v[j] = ok ? vals[base + ti] : 0;
    const uint32_t d = ok ? digit_of(k[j], shift) : 0x100u;  // invalid lanes form their own group
    const unsigned peers = __match_any_sync(kFull, d);
    const int leader = __ffs(peers) - 1;
    uint32_t b = 0;
    if (ok) b = wcnt[warp][d];
    __syncwarp();
    if (ok && int(lane) == leader) wcnt[warp][d] = b + __popc(peers);
    __syncwarp();
    local[j] = b + __popc(peers & lanemask_lt());
  }
  __syncthreads();
  {  // per digit: exclusive prefix over warps, tile total, then scan over digits
    const uint32_t d = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) {
      const uint32_t t = wcnt[w][d];
      wcnt[w][d] = run;
      run += t;
    }
    uint32_t tot;
    tile_off[d] = block_exclusive_scan<uint32_t>(run, ws, &tot);
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kRadixPer; ++j) {
    const uint32_t ti = warp * (kRadixPer * 32) + j * 32 + lane;
    if (ti < valid_in_tile) {
      const uint32_t d = digit_of(k[j], shift);
      const uint32_t pos = tile_off[d] + wcnt[warp][d] + local[j];
      skeys[pos] = k[j];
      if (kVals) svals[pos] = v[j];
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kRadixPer; ++j) {
    const uint32_t idx = j * kRadixThreads + threadIdx.x;
    if (idx < valid_in_tile) {
      const uint64_t key = skeys[idx];
      const uint32_t d = digit_of(key, shift);
      const uint64_t dst = uint64_t(glob_off[d]) + (idx - tile_off[d]);
      out_keys[dst] = key;
      if (kVals) out_vals[dst] = svals[idx];
    }
  }
}

__global__ void k_digit_starts(const uint32_t* __restrict__ hist, uint32_t n_tiles, uint64_t n,
                               uint32_t* __restrict__ starts) {
  QGM_GRID_DEP();
  const uint32_t d = threadIdx.x;
  if (d < kBins) starts[d] = hist[uint64_t(d) * n_tiles];
  if (d == 0) starts[kBins] = uint32_t(n);
}

}  // namespace

void radix_digit_pass(Ctx& c, const uint64_t* in, uint64_t* out, uint64_t n, int shift, uint32_t* starts) {
  if (n > 0xFFFFFFFFull) throw InputError("radix pass: more than 2^32-1 keys");
  const uint32_t tiles = uint32_t(std::max<uint64_t>(ceil_div(n, kRadixTile), 1));
  DBuf<uint32_t> hist(c, uint64_t(kBins) * tiles);
  QGM_KERNEL(c, k_upsweep, tiles, kRadixThreads, 0, in, n, shift, hist.p, tiles);
  exclusive_scan_u32(c, hist.p, hist.p, uint64_t(kBins) * tiles, nullptr, nullptr);
  QGM_KERNEL(c, k_downsweep<false>, tiles, kRadixThreads, 0, in, nullptr, n, shift, hist.p, tiles, out, nullptr);
  QGM_KERNEL(c, k_digit_starts, 1, kRadixThreads, 0, hist.p, tiles, n, starts);
}

void radix_sort(Ctx& c, DBuf<uint64_t>& keys, DBuf<uint64_t>& keys_alt, DBuf<uint32_t>* vals,
                DBuf<uint32_t>* vals_alt, uint64_t n, int begin_bit, int end_bit) {
  if (n <= 1 || end_bit <= begin_bit) return;
  if (n > 0xFFFFFFFFull) throw InputError("radix_sort: more than 2^32-1 keys");
  if (keys_alt.n < n) keys_alt.alloc(c, n);
  if (vals && vals_alt->n < n) vals_alt->alloc(c, n);
  const uint32_t tiles = uint32_t(ceil_div(n, kRadixTile));
  DBuf<uint32_t> hist(c, uint64_t(kBins) * tiles);
  KernelScope ks(c, vals ? "radix_sort_kv" : "radix_sort_keys");
  for (int shift = begin_bit; shift < end_bit; shift += 8) {
    QGM_KERNEL(c, k_upsweep, tiles, kRadixThreads, 0, keys.p, n, shift, hist.p, tiles);
    exclusive_scan_u32(c, hist.p, hist.p, uint64_t(kBins) * tiles, nullptr, nullptr);
    if (vals) {
      QGM_KERNEL(c, k_downsweep<true>, tiles, kRadixThreads, 0, keys.p, vals->p, n, shift, hist.p, tiles,
                 keys_alt.p, vals_alt->p);
      vals->swap(*vals_alt);
    } else {
      QGM_KERNEL(c, k_downsweep<false>, tiles, kRadixThreads, 0, keys.p, nullptr, n, shift, hist.p, tiles,
                 keys_alt.p, nullptr);
    }
    keys.swap(keys_alt);
  }
}

}  // namespace qgm
