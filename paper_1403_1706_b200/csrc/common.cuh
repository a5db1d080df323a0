// common.cuh -- shared device helpers for the sm_100a read-mapping kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace qgm {

// ------------------------------------------------------------------ errors
struct InputError : std::runtime_error {  // -> QGM_ERR_INPUT (qgmap::input_error)
  explicit InputError(const std::string& w) : std::runtime_error(w) {}
};
struct InternalError : std::runtime_error {  // -> QGM_ERR_INTERNAL (std::logic_error)
  explicit InternalError(const std::string& w) : std::runtime_error(w) {}
};
struct CudaError : std::runtime_error {  // -> QGM_ERR_CUDA
  explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};

#define QGM_CUDA(expr)                                                                      \
  do {                                                                                      \
    cudaError_t qgm_e_ = (expr);                                                            \
    if (qgm_e_ != cudaSuccess)                                                              \
      throw ::qgm::CudaError(std::string(#expr) + ": " + cudaGetErrorString(qgm_e_) + " (" + \
                             __FILE__ + ":" + std::to_string(__LINE__) + ")");              \
  } while (0)

#define QGM_LAUNCH_CHECK() QGM_CUDA(cudaGetLastError())

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs

__host__ __device__ inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// ------------------------------------------------------------------ 2-bit codec
// Base j of a 2-bit MSB-first stream: bits [62-2(j%32), 63-2(j%32)] of word j/32.
__device__ __forceinline__ uint32_t base_at(const uint64_t* __restrict__ w, uint64_t j) {
  return uint32_t(__ldg(w + (j >> 5)) >> (62 - 2 * (j & 31))) & 3u;
}

// q-gram code at base offset j (encode_qgram, seq.hpp:80-84: first base in the
// most significant digit). Requires one readable word past the last base.
__device__ __forceinline__ uint32_t qgram_at(const uint64_t* __restrict__ w, uint64_t j, unsigned q) {
  const uint64_t k = j >> 5;
  const unsigned s = unsigned(j & 31) * 2;
  uint64_t hi = __ldg(w + k) << s;
  if (s) hi |= __ldg(w + k + 1) >> (64 - s);
  return uint32_t(hi >> (64 - 2 * q));
}

// Code of the reverse complement of the q-gram with code g: complement every
// 2-bit digit (c -> 3-c == c^3) and reverse the digit order.
__device__ __forceinline__ uint32_t rc_code(uint32_t g, unsigned q) {
  uint32_t x = ~g;
  x = __brev(x);
  x = ((x >> 1) & 0x55555555u) | ((x & 0x55555555u) << 1);
  return x >> (32 - 2 * q);
}

// Canonical code of the pair {g, rc(g)} used to key both strands with one
// lookup (RefQIndex): the member with the smaller g * 0x9E3779B1 mod 2^32 (an
// odd multiplier is a bijection, so the two members tie only for a
// palindrome, g == rc(g)). Choosing by this hash rather than min(g, rc(g))
// keeps canonical codes uniformly spread over the code space (min() would put
// 7/16 of them below 4^(q-1)), so partition bins and join sub-bins stay
// balanced.
__device__ __forceinline__ uint32_t canon_code(uint32_t g, unsigned q) {
  const uint32_t r = rc_code(g, q);
  return g * 0x9E3779B1u <= r * 0x9E3779B1u ? g : r;
}

// Exact division of a 32-bit numerator by a runtime divisor d >= 1 with one
// 64-bit multiply-high: M = floor((2^64-1)/d) + 1 (d == 1 is the identity).
// Error of t*M/2^64 vs t/d is < t/2^64 < 1/d for t < 2^32, so the floor is exact.
struct FastDiv {
  uint64_t M = 0;
  uint32_t d = 1;
  FastDiv() = default;
  explicit FastDiv(uint32_t div) : M(div > 1 ? ~uint64_t(0) / div + 1 : 0), d(div) {}
  __device__ __forceinline__ uint32_t div(uint32_t t) const { return d == 1 ? t : uint32_t(__umul64hi(t, M)); }
};

// ------------------------------------------------------------------ group words
template <class W> struct GroupTraits;
template <> struct GroupTraits<uint32_t> {
  static constexpr unsigned width = 32;
  __device__ static __forceinline__ unsigned popc(uint32_t x) { return __popc(x); }
};
template <> struct GroupTraits<uint64_t> {
  static constexpr unsigned width = 64;
  __device__ static __forceinline__ unsigned popc(uint64_t x) { return __popcll(x); }
};

// Grouprank (qgroup_index.hpp:80-83): set bits of `word` strictly below bit j.
template <class W>
__device__ __forceinline__ uint32_t rank_below(W word, unsigned j) {
  const W m = (W(1) << j) - W(1);  // j < width; j==0 -> 0
  return GroupTraits<W>::popc(word & m);
}

// ------------------------------------------------------------------ warp utils
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <class T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(kFull, v, o);
    if (lane_id() >= unsigned(o)) v += n;
  }
  return v;
}

template <class T>
__device__ __forceinline__ T warp_reduce_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Exclusive scan of one value per thread across the block (blockDim.x <= 1024,
// multiple of 32). `ws` must hold 33 entries. Returns the exclusive prefix;
// *total receives the block sum. Contains __syncthreads.
template <class T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* ws, T* total) {
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T inc = warp_inclusive_scan(v);
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T s = lane < nw ? ws[lane] : T(0);
    T si = warp_inclusive_scan(s);
    if (lane < nw) ws[lane] = si - s;
    if (lane == 31) ws[32] = si;  // nw <= 32: lane 31 holds the full sum
  }
  __syncthreads();
  T res = ws[warp] + inc - v;
  if (total) *total = ws[32];
  __syncthreads();
  return res;
}

// In-place exclusive scan of n (<= blockDim.x * per) u32 values in shared
// memory; each thread scans a contiguous run. Returns the total. All threads
// of the block must call it.
__device__ __forceinline__ uint32_t block_scan_smem(uint32_t* a, uint32_t n, uint32_t* ws) {
  const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
  const uint32_t b = threadIdx.x * per, e = min(n, b + per);
  uint32_t s = 0;
  for (uint32_t i = b; i < e; ++i) s += a[i];
  uint32_t tot;
  uint32_t run = block_exclusive_scan<uint32_t>(s, ws, &tot);
  for (uint32_t i = b; i < e; ++i) {
    uint32_t v = a[i];
    a[i] = run;
    run += v;
  }
  __syncthreads();
  return tot;
}

// ------------------------------------------------------------------ bulk copies
// 1-D TMA bulk copy global -> shared completing on an mbarrier (sm_90+; no
// tensor map). Addresses 16-byte aligned, sizes multiples of 16 bytes.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps until the phase
// completes (or the hint expires) instead of re-issuing the probe, so waiting
// warps leave the issue slots to the working ones
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(0x989680u)
        : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// generic-proxy shared-memory accesses before a later async-proxy write
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Warp-aggregated append: every lane of the (converged) warp calls it; lanes
// with pred get consecutive slots from *counter. Returns the slot (valid only
// where pred).
__device__ __forceinline__ unsigned long long warp_append(bool pred, unsigned long long* counter) {
  const unsigned m = __ballot_sync(kFull, pred);
  unsigned long long base = 0;
  if (m) {
    const int leader = __ffs(m) - 1;
    if (int(lane_id()) == leader) base = atomicAdd(counter, (unsigned long long)__popc(m));
    base = __shfl_sync(kFull, base, leader);
  }
  return base + __popc(m & lanemask_lt());
}

}  // namespace qgm
