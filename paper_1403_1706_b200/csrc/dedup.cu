// dedup.cu -- stage 3 on the map path: the unique (read, strand, diagonal)
// candidate keys, by hashing instead of sorting.
//
// Validation is a pure function of the key and the strata stage sorts its
// hits itself, so the unique candidates need no order: every raw key is
// inserted into an open-addressing table (64-bit atomicCAS, linear probing,
// load factor <= 2/3) and the table is compacted in slot order. Replaces the
// 6-pass LSD radix sort + adjacent-unique of the standalone qgm_cands_unique
// (radix_sort.cu), which cost ~0.5 ms on C2's 5.2M keys; here: one memset,
// one insert pass (8 B read + one CAS per key) and two streaming passes over
// the table.
#include <cstdlib>

#include "internal.hpp"

namespace qgm {
namespace {

constexpr uint64_t kEmpty = ~0ull;  // never a key (the padded diagonal field is < 2^diag_bits - 1)
constexpr int kTile = 4096;         // table slots per compaction tile
constexpr int kDedupThreads = 256;
constexpr uint64_t kPartKeys = uint64_t(2) << 20;  // keys per partition of dedup_keys_partitioned (at most)

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

__global__ void k_hash_insert(const uint64_t* __restrict__ keys, uint64_t n, uint64_t* __restrict__ table,
                              uint64_t tmask) {
  QGM_GRID_DEP();
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t key = keys[i];
    uint64_t slot = mix64(key) & tmask;
    while (true) {
      const uint64_t prev = atomicCAS(reinterpret_cast<unsigned long long*>(table + slot), kEmpty, key);
      if (prev == kEmpty || prev == key) break;
      slot = (slot + 1) & tmask;
    }
  }
}

__global__ void __launch_bounds__(kDedupThreads) k_tile_count(const uint64_t* __restrict__ table, uint64_t T,
                                                              uint32_t* __restrict__ counts) {
  QGM_GRID_DEP();
  __shared__ uint32_t ws[33];
  const uint64_t base = uint64_t(blockIdx.x) * kTile;
  uint32_t c = 0;
  for (uint32_t j = threadIdx.x; j < kTile; j += kDedupThreads) c += table[base + j] != kEmpty;
  uint32_t tot;
  block_exclusive_scan<uint32_t>(c, ws, &tot);
  if (threadIdx.x == 0) counts[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kDedupThreads) k_tile_emit(const uint64_t* __restrict__ table,
                                                             const uint32_t* __restrict__ offs,
                                                             uint64_t* __restrict__ out) {
  QGM_GRID_DEP();
  __shared__ uint32_t ws[33];
  const uint64_t base = uint64_t(blockIdx.x) * kTile;
  uint32_t run = offs[blockIdx.x];
  for (uint32_t j0 = 0; j0 < kTile; j0 += kDedupThreads) {
    const uint64_t v = table[base + j0 + threadIdx.x];
    const uint32_t f = v != kEmpty;
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan<uint32_t>(f, ws, &tot);
    if (f) out[run + ex] = v;
    run += tot;
  }
}

// One pass over the table: each CTA reserves its tile's run of the output
// with one atomic (tile order is irrelevant: validation is per key) and
// writes the tile's keys there. The counter ends as the unique count.
template <bool kReset>  // kReset: leave the tile empty again (the next partition reuses the table)
__global__ void __launch_bounds__(kDedupThreads) k_tile_compact(uint64_t* __restrict__ table,
                                                                uint64_t* __restrict__ out,
                                                                unsigned long long* __restrict__ counter) {
  QGM_GRID_DEP();
  __shared__ uint32_t ws[33];
  __shared__ unsigned long long s_base;
  constexpr int kPerThread = kTile / kDedupThreads;
  const uint64_t base = uint64_t(blockIdx.x) * kTile;
  uint64_t v[kPerThread];
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < kPerThread; ++j) {  // coalesced; a thread's keys go to consecutive outputs
    v[j] = table[base + uint64_t(j) * kDedupThreads + threadIdx.x];
    c += v[j] != kEmpty;
    if (kReset && v[j] != kEmpty) table[base + uint64_t(j) * kDedupThreads + threadIdx.x] = kEmpty;
  }
  uint32_t tot;
  const uint32_t ex = block_exclusive_scan<uint32_t>(c, ws, &tot);
  if (threadIdx.x == 0) s_base = tot ? atomicAdd(counter, (unsigned long long)tot) : 0ull;
  __syncthreads();
  uint64_t o = s_base + ex;
#pragma unroll
  for (int j = 0; j < kPerThread; ++j)
    if (v[j] != kEmpty) out[o++] = v[j];
}

// ---- device-sized variant (the host knows only a bound of the key count)
// table slots for n keys: a power of two >= kTile with load <= 2/3 (the host
// rule of dedup_keys / dedup_keys_async)
__host__ __device__ __forceinline__ uint64_t table_slots(uint64_t n) {
  uint64_t T = kTile;
  while (T < n + n / 2) T <<= 1;
  return T;
}

__device__ __forceinline__ uint64_t dev_count(const unsigned long long* d_n, uint64_t n_max) {
  return min(uint64_t(*d_n), n_max);
}

__global__ void k_table_clear(uint64_t* __restrict__ table, const unsigned long long* __restrict__ d_n,
                              uint64_t n_max) {
  QGM_GRID_DEP();
  const uint64_t T = table_slots(dev_count(d_n, n_max));
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < T; i += uint64_t(gridDim.x) * blockDim.x)
    table[i] = kEmpty;
}

__global__ void k_hash_insert_dev(const uint64_t* __restrict__ keys, const unsigned long long* __restrict__ d_n,
                                  uint64_t n_max, uint64_t* __restrict__ table) {
  QGM_GRID_DEP();
  const uint64_t n = dev_count(d_n, n_max), tmask = table_slots(n) - 1;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t key = keys[i];
    uint64_t slot = mix64(key) & tmask;
    while (true) {
      const uint64_t prev = atomicCAS(reinterpret_cast<unsigned long long*>(table + slot), kEmpty, key);
      if (prev == kEmpty || prev == key) break;
      slot = (slot + 1) & tmask;
    }
  }
}

// k_tile_compact over the table of the device count (blocks past it return)
__global__ void __launch_bounds__(kDedupThreads) k_tile_compact_dev(const uint64_t* __restrict__ table,
                                                                    const unsigned long long* __restrict__ d_n,
                                                                    uint64_t n_max, uint64_t* __restrict__ out,
                                                                    unsigned long long* __restrict__ counter) {
  QGM_GRID_DEP();
  __shared__ uint32_t ws[33];
  __shared__ unsigned long long s_base;
  constexpr int kPerThread = kTile / kDedupThreads;
  const uint64_t base = uint64_t(blockIdx.x) * kTile;
  if (base >= table_slots(dev_count(d_n, n_max))) return;  // CTA-uniform
  uint64_t v[kPerThread];
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < kPerThread; ++j) {
    v[j] = table[base + uint64_t(j) * kDedupThreads + threadIdx.x];
    c += v[j] != kEmpty;
  }
  uint32_t tot;
  const uint32_t ex = block_exclusive_scan<uint32_t>(c, ws, &tot);
  if (threadIdx.x == 0) s_base = tot ? atomicAdd(counter, (unsigned long long)tot) : 0ull;
  __syncthreads();
  uint64_t o = s_base + ex;
#pragma unroll
  for (int j = 0; j < kPerThread; ++j)
    if (v[j] != kEmpty) out[o++] = v[j];
}

// keys of every (mask+1)-th read (read id = key >> rshift) appended to out
// (at most cap are stored; n_out keeps counting past cap so the caller sees
// the overflow). Each CTA takes a tile of 16 keys per thread and reserves its
// run of the output with one atomic (one per warp contended on the counter
// like the join's did: C3, 118M keys).
constexpr int kSamplePer = 16;
__global__ void __launch_bounds__(256) k_sample_reads(const uint64_t* __restrict__ keys, uint64_t n, unsigned rshift,
                                                     uint64_t mask, uint64_t* __restrict__ out, uint64_t cap,
                                                     unsigned long long* __restrict__ n_out) {
  QGM_GRID_DEP();
  __shared__ uint32_t ws[33];
  __shared__ unsigned long long s_base;
  const uint64_t tile = uint64_t(blockDim.x) * kSamplePer;
  for (uint64_t t0 = blockIdx.x * tile; t0 < n; t0 += uint64_t(gridDim.x) * tile) {  // CTA-uniform trip count
    uint64_t k[kSamplePer];
    uint32_t take = 0;
#pragma unroll
    for (int j = 0; j < kSamplePer; ++j) {
      const uint64_t i = t0 + uint64_t(j) * blockDim.x + threadIdx.x;
      k[j] = i < n ? keys[i] : 0ull;
      take |= uint32_t(i < n && ((k[j] >> rshift) & mask) == 0) << j;
    }
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan<uint32_t>(__popc(take), ws, &tot);
    if (threadIdx.x == 0) s_base = tot ? atomicAdd(n_out, (unsigned long long)tot) : 0ull;
    __syncthreads();
    uint64_t at = s_base + ex;
#pragma unroll
    for (int j = 0; j < kSamplePer; ++j)
      if ((take >> j) & 1u) {
        if (at < cap) out[at] = k[j];
        ++at;
      }
    __syncthreads();  // s_base is rewritten by the next tile
  }
}

}  // namespace

void dedup_keys_async(Ctx& c, const uint64_t* keys, uint64_t n, DBuf<uint64_t>& out, unsigned long long* d_count) {
  if (n == 0) {
    fill_bytes(c, d_count, 0, sizeof(unsigned long long));
    if (out.n == 0) out.alloc(c, 1);
    return;
  }
  uint64_t T = kTile;
  while (T < n + n / 2) T <<= 1;  // load factor <= 2/3
  DBuf<uint64_t> table(c, T);
  fill_bytes(c, table.p, 0xFF, T * sizeof(uint64_t));
  {
    KernelScope ks(c, "k_hash_insert");
    const unsigned grid = unsigned(std::min<uint64_t>(ceil_div(n, 256), uint64_t(kSMs) * 16));
    QGM_KERNEL(c, k_hash_insert, grid, 256, 0, keys, n, table.p, T - 1);
  }
  const uint32_t tiles = uint32_t(T / kTile);
  if (out.n < n) out.alloc(c, n);
  fill_bytes(c, d_count, 0, sizeof(unsigned long long));
  QGM_KERNEL(c, k_tile_compact<false>, tiles, kDedupThreads, 0, table.p, out.p, d_count);
}

void dedup_keys_dev(Ctx& c, const uint64_t* keys, uint64_t n_max, const unsigned long long* d_n,
                    DBuf<uint64_t>& out, unsigned long long* d_count) {
  fill_bytes(c, d_count, 0, sizeof(unsigned long long));
  if (out.n < std::max<uint64_t>(n_max, 1)) out.alloc(c, std::max<uint64_t>(n_max, 1));
  if (n_max == 0) return;
  const uint64_t T = table_slots(n_max);
  DBuf<uint64_t> table(c, T);
  const unsigned grid = unsigned(std::min<uint64_t>(ceil_div(n_max, 256), uint64_t(kSMs) * 16));
  QGM_KERNEL(c, k_table_clear, unsigned(std::min<uint64_t>(ceil_div(T, 256), uint64_t(kSMs) * 16)), 256, 0, table.p,
             d_n, n_max);
  {
    KernelScope ks(c, "k_hash_insert");
    QGM_KERNEL(c, k_hash_insert_dev, grid, 256, 0, keys, d_n, n_max, table.p);
  }
  QGM_KERNEL(c, k_tile_compact_dev, unsigned(T / kTile), kDedupThreads, 0, table.p, d_n, n_max, out.p, d_count);
}

void dedup_keys_partitioned(Ctx& c, const uint64_t* keys, uint64_t n, DBuf<uint64_t>& out,
                            unsigned long long* d_count) {
  fill_bytes(c, d_count, 0, sizeof(unsigned long long));
  if (out.n < std::max<uint64_t>(n, 1)) out.alloc(c, std::max<uint64_t>(n, 1));
  if (n == 0) return;
  KernelScope ks(c, "k_hash_insert");
  DBuf<uint64_t> part(c, n);
  DBuf<uint32_t> starts(c, 257);
  radix_digit_pass(c, keys, part.p, n, 0, starts.p);
  std::vector<uint32_t> h(257);
  read_back(c, {{starts.p, h.data(), 257 * 4}});
  // 256 / span partitions of consecutive digits, ~kPartKeys keys each (a
  // table of <= 2^23 slots, 64 MB, stays in the 126 MB L2); fewer, larger
  // partitions when the set is smaller (each costs two launches)
  uint64_t part_keys = kPartKeys;
  const char* e = std::getenv("QGM_DEDUP_PART_KEYS");  // test knob: smaller partitions
  if (e && e[0]) part_keys = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10));
  int span = 256;
  while (span > 1 && n / (256 / span) > part_keys) span >>= 1;
  uint64_t most = 0;
  for (int d = 0; d < 256; d += span) most = std::max<uint64_t>(most, h[d + span] - h[d]);
  uint64_t T = kTile;
  while (T < most + most / 2) T <<= 1;
  DBuf<uint64_t> table(c, T);
  fill_bytes(c, table.p, 0xFF, T * sizeof(uint64_t));  // once: each compaction resets its tiles
  for (int d = 0; d < 256; d += span) {
    const uint64_t np = h[d + span] - h[d];
    if (np == 0) continue;
    uint64_t Tp = kTile;
    while (Tp < np + np / 2) Tp <<= 1;
    const unsigned grid = unsigned(std::min<uint64_t>(ceil_div(np, 256), uint64_t(kSMs) * 16));
    QGM_KERNEL(c, k_hash_insert, grid, 256, 0, part.p + h[d], np, table.p, Tp - 1);
    QGM_KERNEL(c, k_tile_compact<true>, unsigned(Tp / kTile), kDedupThreads, 0, table.p, out.p, d_count);
  }
}

uint64_t dedup_keys(Ctx& c, const uint64_t* keys, uint64_t n, DBuf<uint64_t>& out) {
  if (n == 0) return 0;
  uint64_t T = kTile;
  while (T < n + n / 2) T <<= 1;  // load factor <= 2/3: at C2 the table (64 MiB) stays L2-resident
  DBuf<uint64_t> table(c, T);
  fill_bytes(c, table.p, 0xFF, T * sizeof(uint64_t));
  {
    KernelScope ks(c, "k_hash_insert_sample");  // the dedup-skip estimate: not the batch's dedup
    const unsigned grid = unsigned(std::min<uint64_t>(ceil_div(n, 256), uint64_t(kSMs) * 16));
    QGM_KERNEL(c, k_hash_insert, grid, 256, 0, keys, n, table.p, T - 1);
  }
  const uint32_t tiles = uint32_t(T / kTile);
  DBuf<uint32_t> counts(c, tiles + 1), total(c, 1);
  QGM_KERNEL(c, k_tile_count, tiles, kDedupThreads, 0, table.p, T, counts.p);
  exclusive_scan_u32(c, counts.p, counts.p, tiles, total.p, nullptr);
  uint32_t h = 0;
  read_back(c, {{total.p, &h, sizeof(h)}});
  if (out.n < h) out.alloc(c, std::max<uint64_t>(h, 1));
  QGM_KERNEL(c, k_tile_emit, tiles, kDedupThreads, 0, table.p, counts.p, out.p);
  return h;
}

// Duplicate fraction 1 - unique/raw of a candidate set, estimated from the
// keys of every 64th read: duplicates are (read, strand, diagonal) repeats of
// one read, so a read sample keeps their rate. One pass over the keys, a small
// (L2-resident) hash of the sample, one host round trip.
double estimate_dup_fraction(Ctx& c, const uint64_t* keys, uint64_t n, unsigned rshift) {
  if (n == 0) return 0.0;
  const uint64_t cap = n / 16 + 4096;  // expected n / 64
  DBuf<uint64_t> sample(c, cap);
  DBuf<unsigned long long> ns(c, 1);
  ns.zero();
  QGM_KERNEL(c, k_sample_reads, unsigned(std::min<uint64_t>(ceil_div(n, 256 * kSamplePer), uint64_t(kSMs) * 8)), 256,
             0, keys, n, rshift, 63ull, sample.p, cap, ns.p);
  unsigned long long m = 0;
  read_back(c, {{ns.p, &m, sizeof(m)}});
  if (m == 0 || m > cap) return 1.0;  // no usable sample: assume duplicates (keep the dedup)
  DBuf<uint64_t> uniq;
  const uint64_t u = dedup_keys(c, sample.p, m, uniq);
  return 1.0 - double(u) / double(m);
}

}  // namespace qgm
