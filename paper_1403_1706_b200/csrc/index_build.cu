// index_build.cu -- stage 1: the q-group index, built on the device.
//
// Same arrays and semantics as build_qgroup_index<W> (qgroup_index.hpp:124-180,
// Alg. 1 of PAPER.md:153-193): occupancy I, group starts S (+ sentinel,
// optionally sampled), per-q-gram occurrence starts S' (+ sentinel), positions
// O bucketed by numeric q-gram order. Position order inside one interval is
// unspecified, exactly as in the reference (qgroup_index.hpp:120-123);
// qgm_index_normalize sorts it.
//
// B200 design: a two-level counting sort on the q-gram code instead of the
// reference's six passes of random atomics into 4^q/w-sized arrays.
//   K1 rank    : one thread per item (a read q-gram, or a reference position
//                of one strand); code g, bucket = g >> lb (the top 2q-lb
//                bits); warp-aggregated atomicAdd on the bucket's count (L2
//                resident) returns the item's rank inside the bucket.
//   scan       : bucket offsets.
//   K2 scatter : (extra, g & lowmask, position) packed in one u64 per item.
//   -- the bucketed items are all the per-batch join of join.cu needs --
//   K3 occupy  : one CTA per bucket (2^lb codes = 2^lb/w group words) builds
//                the bucket's occupancy words in shared memory, writes I and
//                the bucket's distinct count.
//   scan       : distinct offsets (the global base of S for every bucket).
//   K4 emit    : one CTA per bucket rebuilds the local ranks from I, writes S
//                (popcount prefix), S' (occurrence prefix) and scatters the
//                positions (and the per-item extra byte) into O through
//                shared-memory cursors.
// Every HBM write of I/S/S'/O is coalesced; the only random traffic is the
// bucket scatter of K2.
#include <cstdlib>

#include "internal.hpp"

namespace qgm {
namespace {

constexpr unsigned kLowBits = 13;  // codes per bucket = 8192
constexpr int kBuildThreads = 256;
constexpr size_t kMaxBuildSmem = 200 * 1024;  // dynamic shared memory of one emit CTA
struct BuildRetry {};                         // a bucket geometry the emit cannot stage

// Read q-grams: one slot per (read, offset) with offset <= stride-q; slots
// past a read's length are idle (seq.hpp:135-137).
struct ReadSource {
  const uint64_t* words;
  const uint32_t* lengths;
  uint32_t W, span, stride;
  FastDiv by_span;
  unsigned q;
  __device__ __forceinline__ bool item(uint64_t t, uint32_t& g, uint32_t& pos, uint32_t& extra) const {
    const uint32_t r = by_span.div(uint32_t(t));  // slots < 2^32 (checked on the host)
    const uint32_t o = uint32_t(t) - r * span;
    if (o + q > __ldg(lengths + r)) return false;
    g = qgram_at(words + uint64_t(r) * W, o, q);
    pos = r * stride + o;
    extra = 0;
    return true;
  }
};

// Reference positions under canonical codes (RefQIndex): source index t < L
// is position t; t >= L is the palindromic position pal[t - L], listed a
// second time with flag 1. A position is indexed iff its window lies inside
// its chromosome and it is not masked.
// pos = the padded coordinate cbp[c] + p; extra = b | flag << 3, b = ref[x-1]
// or 4 when x-1 is outside the chromosome or masked; with `packed`, extra
// goes into pos's top 4 bits.
struct RefSource {
  const uint64_t* ref;
  const uint64_t* mask;
  const uint64_t* cb;
  const uint64_t* pal;
  uint64_t L;
  uint32_t n_chrom;
  unsigned q;
  bool packed;
  uint64_t gap;
  __device__ __forceinline__ bool masked(uint64_t x) const {
    return mask && ((__ldg(mask + (x >> 6)) >> (x & 63)) & 1ull);
  }
  // window of x inside its chromosome and unmasked; returns the chromosome
  __device__ __forceinline__ bool indexed(uint64_t x, uint32_t& chrom, uint64_t& p) const {
    if (masked(x)) return false;
    uint32_t lo = 0, hi = n_chrom;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(cb + mid) <= x) lo = mid; else hi = mid;
    }
    const uint64_t cbeg = __ldg(cb + lo);
    p = x - cbeg;
    chrom = lo;
    return p + q <= __ldg(cb + lo + 1) - cbeg;
  }
  __device__ __forceinline__ bool item(uint64_t t, uint32_t& g, uint32_t& pos, uint32_t& extra) const {
    const bool dup = t >= L;
    const uint64_t x = dup ? __ldg(pal + (t - L)) : t;
    uint32_t c;
    uint64_t p;
    if (!indexed(x, c, p)) return false;
    const uint32_t f = qgram_at(ref, x, q);
    g = canon_code(f, q);
    pos = uint32_t(x + uint64_t(c + 1) * gap);
    const uint32_t b = (p >= 1 && !masked(x - 1)) ? base_at(ref, x - 1) : 4u;
    extra = b | (uint32_t(dup || f != g) << 3);
    if (packed) {
      pos |= extra << kPackedPosBits;
      extra = 0;
    }
    return true;
  }
};

// Forward q-grams of one chromosome [c0, c1) for the repeat mask: every
// window inside the chromosome (the existing mask is ignored: frequencies are
// over all windows); pos = the chromosome-relative position.
struct FwdChromSource {
  const uint64_t* ref;
  uint64_t c0, c1;
  unsigned q;
  __device__ __forceinline__ bool item(uint64_t t, uint32_t& g, uint32_t& pos, uint32_t& extra) const {
    const uint64_t x = c0 + t;
    if (x + q > c1) return false;
    g = qgram_at(ref, x, q);
    pos = uint32_t(t);
    extra = 0;
    return true;
  }
};

// One CTA per bucket of 2^lb codes: count the bucket's codes in shared memory,
// then set the mask bit of every position whose code occurs more than
// `threshold` times (positions of too-frequent q-grams leave P).
__global__ void __launch_bounds__(kBuildThreads) k_bucket_mask(const uint64_t* __restrict__ pairs,
                                                               const uint32_t* __restrict__ boff, uint64_t buckets,
                                                               uint32_t lmask, uint64_t threshold, uint64_t c0,
                                                               unsigned long long* __restrict__ mask) {
  QGM_GRID_DEP();
  extern __shared__ uint32_t cnt[];  // 2^lb counters
  for (uint64_t bk = blockIdx.x; bk < buckets; bk += gridDim.x) {
    for (uint32_t i = threadIdx.x; i <= lmask; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    const uint32_t b0 = boff[bk], b1 = boff[bk + 1];
    for (uint32_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) atomicAdd(cnt + (uint32_t(pairs[i] >> 32) & lmask), 1u);
    __syncthreads();
    for (uint32_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
      const uint64_t pr = pairs[i];
      if (cnt[uint32_t(pr >> 32) & lmask] > threshold) {
        const uint64_t x = c0 + uint32_t(pr);
        atomicOr(mask + (x >> 6), 1ull << (x & 63));
      }
    }
    __syncthreads();
  }
}

// Palindromic indexed positions (f == rc(f); even q only): count, then list.
__global__ void k_pal_scan(RefSource src, uint64_t* __restrict__ out, unsigned long long* __restrict__ count) {
  QGM_GRID_DEP();
  for (uint64_t base = blockIdx.x * uint64_t(blockDim.x); base < src.L; base += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t x = base + threadIdx.x;
    uint32_t c;
    uint64_t p;
    bool pal = false;
    if (x < src.L && src.indexed(x, c, p)) {
      const uint32_t f = qgram_at(src.ref, x, src.q);
      pal = f == rc_code(f, src.q);
    }
    const unsigned long long slot = warp_append(pal, count);
    if (pal && out) out[slot] = x;
  }
}

// bucketed item: extra (4 bits) << 48 | low code bits (lb <= 16) << 32 | pos
__device__ __forceinline__ uint64_t pack_item(uint32_t extra, uint32_t glow, uint32_t pos) {
  return (uint64_t(extra) << 48) | (uint64_t(glow) << 32) | pos;
}
// kG = 32 for these items, 40 for join items (partition.cu) of a raw-code
// partition, whose low 16 code bits sit at bit 40 and position in bits 0..31
template <int kG = 32>
__device__ __forceinline__ uint32_t item_glow(uint64_t pr) { return uint32_t(pr >> kG) & 0xFFFFu; }

template <class Src>
__global__ void k_bucket_rank(Src src, uint64_t n_items, unsigned lb, uint32_t* __restrict__ bucket_cnt,
                              uint32_t* __restrict__ rank) {
  QGM_GRID_DEP();
  for (uint64_t base = blockIdx.x * uint64_t(blockDim.x); base < n_items; base += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t t = base + threadIdx.x;
    uint32_t g = 0, pos, extra, b = 0xFFFFFFFFu;
    const bool ok = t < n_items && src.item(t, g, pos, extra);
    if (ok) b = g >> lb;
    const unsigned peers = __match_any_sync(kFull, b);
    const int leader = __ffs(peers) - 1;
    uint32_t base_rank = 0;
    if (ok && int(lane_id()) == leader) base_rank = atomicAdd(bucket_cnt + b, __popc(peers));
    base_rank = __shfl_sync(kFull, base_rank, leader);
    if (ok) rank[t] = base_rank + __popc(peers & lanemask_lt());
  }
}

template <class Src>
__global__ void k_bucket_scatter(Src src, uint64_t n_items, unsigned lb, const uint32_t* __restrict__ boff,
                                 const uint32_t* __restrict__ rank, uint64_t* __restrict__ pairs) {
  QGM_GRID_DEP();
  const uint32_t lmask = (1u << lb) - 1u;
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < n_items;
       t += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t g, pos, extra;
    if (!src.item(t, g, pos, extra)) continue;
    pairs[boff[g >> lb] + rank[t]] = pack_item(extra, g & lmask, pos);
  }
}

// Items of one bucket held in registers: the first kItemRegs * kBuildThreads
// are loaded together (all in flight at once -- the bucket kernels are bound
// by the latency of these loads, not by bandwidth), the rest, if any, by a
// plain loop.
#ifndef QGM_IB_ITEMS
#define QGM_IB_ITEMS 6
#endif
#ifndef QGM_IB_MINB
#define QGM_IB_MINB 6
#endif
constexpr int kItemRegs = QGM_IB_ITEMS;

// kPer > 0: gpb == kPer * kBuildThreads, thread t owns the contiguous group
// words [t * kPer, (t + 1) * kPer) (16-byte vector accesses, popcounts
// prefix-summed in registers); kPer == 0: any gpb, strided loops.
template <class W, int kPer>
struct GroupRun {
  W x[kPer > 0 ? kPer : 1];
  __device__ __forceinline__ void load(const W* __restrict__ src) {
    static_assert(kPer == 0 || (kPer * sizeof(W)) % 16 == 0, "whole 16-byte vectors per thread");
#pragma unroll
    for (int v = 0; v < int(kPer * sizeof(W) / 16); ++v) {
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(src) + v);
      reinterpret_cast<uint4*>(x)[v] = q;
    }
  }
  __device__ __forceinline__ void store(W* dst) const {
#pragma unroll
    for (int v = 0; v < int(kPer * sizeof(W) / 16); ++v) reinterpret_cast<uint4*>(dst)[v] = reinterpret_cast<const uint4*>(x)[v];
  }
};

template <class W, int kG, int kPer>
__global__ void __launch_bounds__(kBuildThreads) k_bucket_occupy(const uint64_t* __restrict__ pairs,
                                                                 const uint32_t* __restrict__ boff,
                                                                 uint64_t buckets, uint32_t gpb,
                                                                 W* __restrict__ I, uint32_t* __restrict__ dcnt) {
  QGM_GRID_DEP();
  using AW = typename std::conditional<sizeof(W) == 8, unsigned long long, unsigned>::type;
  constexpr unsigned w = GroupTraits<W>::width;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  W* occ = reinterpret_cast<W*>(smem_raw);
  __shared__ uint32_t ws[33];
  for (uint64_t bk = blockIdx.x; bk < buckets; bk += gridDim.x) {
    const uint32_t b0 = boff[bk], b1 = boff[bk + 1];
    uint64_t pr[kItemRegs];
#pragma unroll
    for (int u = 0; u < kItemRegs; ++u) {
      const uint32_t i = b0 + threadIdx.x + u * kBuildThreads;
      pr[u] = i < b1 ? pairs[i] : 0;
    }
    for (uint32_t i = threadIdx.x; i < gpb; i += blockDim.x) occ[i] = W(0);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kItemRegs; ++u) {
      const uint32_t i = b0 + threadIdx.x + u * kBuildThreads;
      if (i < b1) {
        const uint32_t gl = item_glow<kG>(pr[u]);
        atomicOr(reinterpret_cast<AW*>(occ + gl / w), AW(W(1) << (gl % w)));
      }
    }
    for (uint32_t i = b0 + threadIdx.x + kItemRegs * kBuildThreads; i < b1; i += blockDim.x) {
      const uint32_t gl = item_glow<kG>(pairs[i]);
      atomicOr(reinterpret_cast<AW*>(occ + gl / w), AW(W(1) << (gl % w)));
    }
    __syncthreads();
    uint32_t pc = 0;
    if constexpr (kPer > 0) {
      GroupRun<W, kPer> g;
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        g.x[u] = occ[threadIdx.x * kPer + u];
        pc += GroupTraits<W>::popc(g.x[u]);
      }
      g.store(I + bk * gpb + uint64_t(threadIdx.x) * kPer);
    } else {
      for (uint32_t i = threadIdx.x; i < gpb; i += blockDim.x) {
        const W x = occ[i];
        I[bk * gpb + i] = x;
        pc += GroupTraits<W>::popc(x);
      }
    }
    uint32_t tot;
    block_exclusive_scan<uint32_t>(pc, ws, &tot);
    if (threadIdx.x == 0) dcnt[bk] = tot;
    __syncthreads();
  }
}

template <class W, bool kSampled, bool kExtra, int kG, int kPer>
__global__ void __launch_bounds__(kBuildThreads, QGM_IB_MINB) k_bucket_emit(const uint64_t* __restrict__ pairs,
                                                               const uint32_t* __restrict__ boff,
                                                               const uint32_t* __restrict__ dbase,
                                                               uint64_t buckets, uint32_t gpb,
                                                               const W* __restrict__ I, uint32_t* __restrict__ S,
                                                               uint32_t* __restrict__ S1, uint32_t* __restrict__ O,
                                                               uint8_t* __restrict__ X) {
  QGM_GRID_DEP();
  constexpr unsigned w = GroupTraits<W>::width;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  W* occ = reinterpret_cast<W*>(smem_raw);
  uint32_t* sloc = reinterpret_cast<uint32_t*>(occ + gpb);
  uint32_t* cnt = sloc + gpb;  // up to gpb*w counters
  __shared__ uint32_t ws[33];
  for (uint64_t bk = blockIdx.x; bk < buckets; bk += gridDim.x) {
    const uint32_t b0 = boff[bk], b1 = boff[bk + 1];
    const uint32_t db = dbase[bk];
    // the bucket's items, kept in registers for both passes below
    uint64_t pr[kItemRegs];
#pragma unroll
    for (int u = 0; u < kItemRegs; ++u) {
      const uint32_t i = b0 + threadIdx.x + u * kBuildThreads;
      pr[u] = i < b1 ? pairs[i] : 0;
    }
    uint32_t D;
    if constexpr (kPer > 0) {
      const uint32_t g0 = threadIdx.x * kPer;
      GroupRun<W, kPer> g;
      g.load(I + bk * gpb + g0);
      uint32_t ex[kPer], sum = 0;
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        ex[u] = sum;
        sum += GroupTraits<W>::popc(g.x[u]);
      }
      const uint32_t run = block_exclusive_scan<uint32_t>(sum, ws, &D);
      g.store(occ + g0);
      if constexpr (kPer % 4 == 0) {  // the thread's group starts as whole 16-byte vectors
#pragma unroll
        for (int v = 0; v < kPer / 4; ++v) {
          const uint4 loc = make_uint4(run + ex[4 * v], run + ex[4 * v + 1], run + ex[4 * v + 2], run + ex[4 * v + 3]);
          reinterpret_cast<uint4*>(sloc + g0)[v] = loc;
          if (!kSampled)
            reinterpret_cast<uint4*>(S + bk * gpb + g0)[v] = make_uint4(db + loc.x, db + loc.y, db + loc.z, db + loc.w);
        }
      } else {
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          sloc[g0 + u] = run + ex[u];
          if (!kSampled) S[bk * gpb + g0 + u] = db + run + ex[u];
        }
      }
      if (kSampled) {
#pragma unroll
        for (int u = 0; u < kPer; u += 2) S[(bk * gpb + g0 + u) >> 1] = db + run + ex[u];  // g0 + u even
      }
    } else {
      for (uint32_t i = threadIdx.x; i < gpb; i += blockDim.x) {
        const W x = I[bk * gpb + i];
        occ[i] = x;
        sloc[i] = GroupTraits<W>::popc(x);
      }
      __syncthreads();
      D = block_scan_smem(sloc, gpb, ws);
      for (uint32_t i = threadIdx.x; i < gpb; i += blockDim.x) {
        const uint64_t gi = bk * gpb + i;
        if (!kSampled) S[gi] = db + sloc[i];
        else if ((gi & 1) == 0) S[gi >> 1] = db + sloc[i];
      }
    }
    for (uint32_t i = threadIdx.x; i < D; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    auto counter = [&](uint64_t p) {
      const uint32_t gl = item_glow<kG>(p);
      const uint32_t wi = gl / w;
      return cnt + sloc[wi] + rank_below<W>(occ[wi], gl % w);
    };
#pragma unroll
    for (int u = 0; u < kItemRegs; ++u)
      if (b0 + threadIdx.x + u * kBuildThreads < b1) atomicAdd(counter(pr[u]), 1u);
    for (uint32_t i = b0 + threadIdx.x + kItemRegs * kBuildThreads; i < b1; i += blockDim.x)
      atomicAdd(counter(pairs[i]), 1u);
    __syncthreads();
    block_scan_smem(cnt, D, ws);
    for (uint32_t i = threadIdx.x; i < D; i += blockDim.x) S1[db + i] = b0 + cnt[i];
    __syncthreads();
    auto place = [&](uint64_t p) {
      const uint32_t slot = atomicAdd(counter(p), 1u);
      O[b0 + slot] = uint32_t(p);
      if (kExtra) X[b0 + slot] = uint8_t(p >> 48);
    };
#pragma unroll
    for (int u = 0; u < kItemRegs; ++u)
      if (b0 + threadIdx.x + u * kBuildThreads < b1) place(pr[u]);
    for (uint32_t i = b0 + threadIdx.x + kItemRegs * kBuildThreads; i < b1; i += blockDim.x) place(pairs[i]);
    __syncthreads();
  }
}

__global__ void k_set_u32(uint32_t* p, uint32_t v) {
  QGM_GRID_DEP(); *p = v; }

__global__ void k_max_u32(const uint32_t* __restrict__ a, uint64_t n, uint32_t* __restrict__ out) {
  QGM_GRID_DEP();
  uint32_t m = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    m = max(m, a[i]);
  m = __reduce_max_sync(kFull, m);
  if (lane_id() == 0 && m) atomicMax(out, m);
}

// group start of word w relative to its sub-bin (< 2^16: a sub-bin holds at
// most 2^16 codes and this is an exclusive prefix)
__global__ void k_rank16(const uint32_t* __restrict__ S, uint64_t groups, unsigned wshift,
                         const uint32_t* __restrict__ sb_d, uint16_t* __restrict__ r16) {
  QGM_GRID_DEP();
  for (uint64_t w = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < groups; w += uint64_t(gridDim.x) * blockDim.x)
    r16[w] = uint16_t(S[w] - sb_d[w >> wshift]);
}

// sub-bin s covers group words [(s << cs) / 32, ((s+1) << cs) / 32): its S'
// range starts at S of its first word, its O range at S' of that
__global__ void k_subbin_bounds(const uint32_t* __restrict__ S, const uint32_t* __restrict__ S1, uint32_t n_sub,
                                unsigned cs, uint32_t* __restrict__ sb_d, uint32_t* __restrict__ sb_o) {
  QGM_GRID_DEP();
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s <= n_sub; s += gridDim.x * blockDim.x) {
    const uint32_t d = S[uint32_t((uint64_t(s) << cs) >> 5)];
    sb_d[s] = d;
    sb_o[s] = S1[d];
  }
}

__global__ void k_sample_S(const uint32_t* __restrict__ S, uint64_t len_in, uint32_t* __restrict__ out,
                           uint64_t len_out) {
  QGM_GRID_DEP();
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < len_out; i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = S[2 * i];
}

// Thread per interval: insertion sort for short intervals, heap sort otherwise.
__global__ void k_sort_intervals(const uint32_t* __restrict__ S1, uint64_t distinct, uint32_t* __restrict__ O) {
  QGM_GRID_DEP();
  for (uint64_t b = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; b < distinct; b += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t* a = O + S1[b];
    const uint32_t n = S1[b + 1] - S1[b];
    if (n <= 32) {
      for (uint32_t i = 1; i < n; ++i) {
        const uint32_t x = a[i];
        uint32_t j = i;
        while (j > 0 && a[j - 1] > x) { a[j] = a[j - 1]; --j; }
        a[j] = x;
      }
    } else {
      auto sift = [&](uint32_t root, uint32_t end) {
        while (2 * root + 1 < end) {
          uint32_t ch = 2 * root + 1;
          if (ch + 1 < end && a[ch] < a[ch + 1]) ++ch;
          if (a[root] >= a[ch]) return;
          const uint32_t t = a[root]; a[root] = a[ch]; a[ch] = t;
          root = ch;
        }
      };
      for (uint32_t s = n / 2; s-- > 0;) sift(s, n);
      for (uint32_t e = n; e-- > 1;) {
        const uint32_t t = a[0]; a[0] = a[e]; a[e] = t;
        sift(0, e);
      }
    }
  }
}

template <class W>
__global__ void k_lookup(const W* __restrict__ I, const uint32_t* __restrict__ S, const uint32_t* __restrict__ S1,
                         bool sampled, const uint32_t* __restrict__ codes, uint64_t n, uint32_t* __restrict__ begin,
                         uint32_t* __restrict__ end) {
  QGM_GRID_DEP();
  constexpr unsigned w = GroupTraits<W>::width;
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < n; t += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t g = codes[t];
    const uint64_t i = g / w;
    const unsigned j = g % w;
    const W word = I[i];
    uint32_t b0 = 0xFFFFFFFFu, b1 = 0xFFFFFFFFu;
    if ((word >> j) & W(1)) {
      uint32_t base = sampled ? S[i >> 1] + ((i & 1) ? GroupTraits<W>::popc(I[i - 1]) : 0u) : S[i];
      base += rank_below<W>(word, j);
      b0 = S1[base];
      b1 = S1[base + 1];
    }
    begin[t] = b0;
    end[t] = b1;
  }
}

template <class Src>
void bucket_impl(Ctx& c, const Src& src, uint64_t n_items, Buckets& B) {
  DBuf<uint32_t> bucket_cnt(c, B.buckets + 1);
  bucket_cnt.zero();
  DBuf<uint32_t> rank(c, std::max<uint64_t>(n_items, 1));
  const unsigned grid = unsigned(std::min<uint64_t>(std::max<uint64_t>(ceil_div(n_items, 256), 1), kSMs * 32));
  if (n_items) {
    KernelScope ks(c, "k_bucket_rank");
    QGM_KERNEL(c, k_bucket_rank<Src>, grid, 256, 0, src, n_items, B.lb, bucket_cnt.p, rank.p);
  }
  B.boff.alloc(c, B.buckets + 1);
  DBuf<uint32_t> vtotal(c, 1);
  exclusive_scan_u32(c, bucket_cnt.p, B.boff.p, B.buckets + 1, vtotal.p, nullptr);
  uint32_t V = 0;
  read_back(c, {{vtotal.p, &V, 4}});
  B.V = V;
  B.pairs.alloc(c, std::max<uint64_t>(V, 1));
  if (n_items) {
    KernelScope ks(c, "k_bucket_scatter");
    QGM_KERNEL(c, k_bucket_scatter<Src>, grid, 256, 0, src, n_items, B.lb, B.boff.p, rank.p, B.pairs.p);
  }
}

template <class W, int kG>
void finish_impl(Ctx& c, const Buckets& B, bool sampled, Index& out, DBuf<uint8_t>* extra) {
  out.q = B.q;
  out.w = B.w;
  out.sampled = sampled;
  out.groups = B.groups;
  out.gs_len = sampled ? (B.groups + 1 + 1) / 2 : B.groups + 1;
  out.occ = B.V;
  out.I.alloc(c, B.groups * sizeof(W));
  out.S.alloc(c, out.gs_len);
  out.O.alloc(c, std::max<uint64_t>(B.V, 1));
  if (extra) extra->alloc(c, std::max<uint64_t>(B.V, 1));

  const unsigned grid_b = unsigned(std::min<uint64_t>(B.buckets, uint64_t(kSMs) * 8));
  DBuf<uint32_t> dcnt(c, B.buckets + 1);
  fill_bytes(c, dcnt.p + B.buckets, 0, 4);
  // group words per thread of the vectorised bucket kernels (0: strided)
  const int per = B.gpb * sizeof(W) == size_t(kBuildThreads) * 32 ? int(32 / sizeof(W))
                  : B.gpb * sizeof(W) == size_t(kBuildThreads) * 16 ? int(16 / sizeof(W)) : 0;
  {
    KernelScope ks(c, "k_bucket_occupy");
    auto occupy = [&](auto kernel) {
      QGM_KERNEL(c, kernel, grid_b, kBuildThreads, B.gpb * sizeof(W), B.pairs.p, B.boff.p, B.buckets,
                 uint32_t(B.gpb), reinterpret_cast<W*>(out.I.p), dcnt.p);
    };
    if (per == int(32 / sizeof(W))) occupy(k_bucket_occupy<W, kG, int(32 / sizeof(W))>);
    else if (per == int(16 / sizeof(W))) occupy(k_bucket_occupy<W, kG, int(16 / sizeof(W))>);
    else occupy(k_bucket_occupy<W, kG, 0>);
  }
  DBuf<uint32_t> dbase(c, B.buckets + 1);
  DBuf<uint32_t> dtotal(c, 2);  // total distinct codes, largest bucket's distinct count
  dtotal.zero();
  exclusive_scan_u32(c, dcnt.p, dbase.p, B.buckets + 1, dtotal.p, nullptr);
  QGM_KERNEL(c, k_max_u32, unsigned(std::min<uint64_t>(ceil_div(B.buckets, 256), uint64_t(kSMs) * 4)), 256, 0,
             dcnt.p, B.buckets, dtotal.p + 1);
  uint32_t Dm[2] = {0, 0};
  read_back(c, {{dtotal.p, Dm, 8}});
  const uint32_t D = Dm[0];
  out.distinct = D;
  out.S1.alloc(c, uint64_t(D) + 1);

  // the emit's per-code counters: one per distinct code of the bucket (the
  // largest bucket's count), not one per code of the bucket's range
  const size_t smem = B.gpb * sizeof(W) + B.gpb * 4 + size_t(std::max<uint32_t>(Dm[1], 1)) * 4;
  if (smem > kMaxBuildSmem) throw BuildRetry{};
  auto launch = [&](auto kernel) {
    ensure_dynamic_smem(reinterpret_cast<const void*>(kernel), size_t(smem));
    KernelScope ks(c, "k_bucket_emit");
    QGM_KERNEL(c, kernel, grid_b, kBuildThreads, smem, B.pairs.p, B.boff.p, dbase.p, B.buckets, uint32_t(B.gpb),
               reinterpret_cast<const W*>(out.I.p), out.S.p, out.S1.p, out.O.p, extra ? extra->p : nullptr);
  };
  auto by_per = [&](auto kSampled, auto kExtra) {
    constexpr bool S_ = decltype(kSampled)::value, E_ = decltype(kExtra)::value;
    if (per == int(32 / sizeof(W))) launch(k_bucket_emit<W, S_, E_, kG, int(32 / sizeof(W))>);
    else if (per == int(16 / sizeof(W))) launch(k_bucket_emit<W, S_, E_, kG, int(16 / sizeof(W))>);
    else launch(k_bucket_emit<W, S_, E_, kG, 0>);
  };
  if (sampled) {
    if (extra) by_per(std::true_type{}, std::true_type{});
    else by_per(std::true_type{}, std::false_type{});
  } else {
    if (extra) by_per(std::false_type{}, std::true_type{});
    else by_per(std::false_type{}, std::false_type{});
  }
  // sentinels: S[groups] = D (kept by sampling iff groups is even), S'[D] = V
  if (!sampled) QGM_KERNEL(c, k_set_u32, 1, 1, 0, out.S.p + B.groups, D);
  else if ((B.groups & 1) == 0) QGM_KERNEL(c, k_set_u32, 1, 1, 0, out.S.p + B.groups / 2, D);
  QGM_KERNEL(c, k_set_u32, 1, 1, 0, out.S1.p + D, B.V);
}

void init_geometry(Buckets& B, unsigned q, unsigned w, unsigned lb_max = kLowBits) {
  if (q == 0 || q > 16) throw InputError("q must be in [1, 16]");
  if (w != 32 && w != 64) throw InputError("group width must be 32 or 64");
  B.q = q;
  B.w = w;
  B.lb = std::min(2 * q, lb_max);
  B.hb = 2 * q - B.lb;
  const uint64_t space = uint64_t(1) << (2 * q);
  B.groups = ceil_div(space, w);
  B.buckets = uint64_t(1) << B.hb;
  B.gpb = std::max<uint64_t>(1, (uint64_t(1) << B.lb) / w);
  if (B.buckets * B.gpb != B.groups) throw InternalError("index geometry mismatch");
}

}  // namespace

void bucket_reads(Ctx& c, const Reads& reads, unsigned q, unsigned w, Buckets& out, unsigned lb_max) {
  init_geometry(out, q, w, lb_max);
  ReadSource src;
  src.words = reads.words.p;
  src.lengths = reads.lengths.p;
  src.W = reads.W;
  src.span = reads.stride >= q ? reads.stride - q + 1 : 0;
  src.stride = reads.stride;
  src.by_span = FastDiv(std::max<uint32_t>(src.span, 1));
  src.q = q;
  if (uint64_t(reads.n) * src.span > 0xFFFFFFFFull) throw InputError("read batch has more than 2^32-1 q-gram slots");
  bucket_impl(c, src, uint64_t(reads.n) * src.span, out);
}

void bucket_ref(Ctx& c, const Ref& ref, unsigned q, bool packed, Buckets& out, uint64_t* n_pal) {
  init_geometry(out, q, 32);
  if (ref.padded_total >= (uint64_t(1) << 32)) throw InputError("reference index: more than 2^32-1 padded bases");
  RefSource src;
  src.ref = ref.words.p;
  src.mask = ref.mask.p;
  src.cb = ref.d_cb.p;
  src.pal = nullptr;
  src.L = ref.total;
  src.n_chrom = ref.n_chrom;
  src.q = q;
  src.packed = packed;
  src.gap = ref.gap;
  DBuf<uint64_t> pal;
  unsigned long long np = 0;
  if (q % 2 == 0 && ref.total) {
    DBuf<unsigned long long> cnt(c, 1);
    cnt.zero();
    const unsigned grid = unsigned(std::min<uint64_t>(ceil_div(ref.total, 256), kSMs * 32));
    QGM_KERNEL(c, k_pal_scan, grid, 256, 0, src, nullptr, cnt.p);
    read_back(c, {{cnt.p, &np, sizeof(np)}});
    if (np) {
      pal.alloc(c, np);
      cnt.zero();
      QGM_KERNEL(c, k_pal_scan, grid, 256, 0, src, pal.p, cnt.p);
      src.pal = pal.p;
    }
  }
  *n_pal = np;
  bucket_impl(c, src, ref.total + np, out);
}

void mask_repeats(Ctx& c, Ref& ref, unsigned q, uint64_t threshold) {
  if (q == 0 || q > 16) throw InputError("q must be in [1, 16]");
  const uint64_t mw = ceil_div(ref.total, 64);
  if (!ref.mask.p) {
    ref.mask.alloc(c, std::max<uint64_t>(mw, 1));
    ref.mask.zero();
  }
  for (uint32_t k = 0; k < ref.n_chrom; ++k) {
    const uint64_t c0 = ref.cb[k], c1 = ref.cb[k + 1];
    if (c1 - c0 < q) continue;
    Buckets B;
    init_geometry(B, q, 32);
    FwdChromSource src{ref.words.p, c0, c1, q};
    bucket_impl(c, src, c1 - c0, B);
    if (B.V == 0) continue;
    const uint32_t lmask = uint32_t((uint64_t(1) << B.lb) - 1);
    const size_t smem = size_t(lmask + 1) * sizeof(uint32_t);
    ensure_dynamic_smem(reinterpret_cast<const void*>(k_bucket_mask), size_t(smem));
    QGM_KERNEL(c, k_bucket_mask, unsigned(std::min<uint64_t>(B.buckets, uint64_t(kSMs) * 8)), kBuildThreads, smem,
               B.pairs.p, B.boff.p, B.buckets, lmask, threshold, c0,
               reinterpret_cast<unsigned long long*>(ref.mask.p));
  }
  ref.qidx = RefQIndex();  // the reference index depends on the mask
}

void index_from_buckets(Ctx& c, const Buckets& B, bool sampled, Index& out, DBuf<uint8_t>* extra) {
  if (B.join_items) {  // a raw-code partition's items (no extra byte)
    if (B.w == 32) finish_impl<uint32_t, 40>(c, B, sampled, out, nullptr);
    else finish_impl<uint64_t, 40>(c, B, sampled, out, nullptr);
  } else if (B.w == 32) {
    finish_impl<uint32_t, 32>(c, B, sampled, out, extra);
  } else {
    finish_impl<uint64_t, 32>(c, B, sampled, out, extra);
  }
}

void build_index(Ctx& c, const Reads& reads, unsigned q, unsigned w, bool sampled, Index& out) {
  if (reads.lens.p) {  // the upload's length check (qgm_reads_upload does not synchronise)
    uint32_t lens[2] = {0, 0};
    read_back(c, {{reads.lens.p, lens, 8}});
    if (lens[0] > reads.stride) throw InputError("read longer than the stride");
  }
  // buckets of 2^16 codes when that leaves ~8k q-grams per bucket or fewer
  // (C2: 65536 buckets of ~1300): 8x fewer per-bucket passes of the occupy /
  // emit kernels and a scatter into 8x fewer frontiers than 2^13-code
  // buckets; a bucket with too many distinct codes for the emit's shared
  // counters falls back to 2^13
  const uint64_t n_items = uint64_t(reads.n) * (reads.stride >= q ? reads.stride - q + 1 : 0);
  const bool wide = 2 * q >= 24 && (n_items >> (2 * q - 16)) <= 8192;
  for (int attempt = wide ? 0 : 1; attempt < 2; ++attempt) {
    Buckets B;
    if (attempt == 0) {
      // 2^16-code buckets from the map path's two staged counting sorts over
      // raw codes (partition.cu): the buckets are its sub-bins
      init_geometry(B, q, w, 16);
      Partitioned rp;
      partition_reads(c, reads, q, rp, /*raw=*/true, /*force_key_bits=*/2 * q - B.lb);
      uint32_t fl[4] = {0, 0, 0, 0};
      read_back(c, {{rp.flags.p, fl, sizeof(fl)}});
      B.V = fl[0];
      B.boff.swap(rp.soff);
      B.pairs.swap(rp.pairs);
      B.join_items = true;
    } else {
      bucket_reads(c, reads, q, w, B, kLowBits);
    }
    try {
      index_from_buckets(c, B, sampled, out, nullptr);
    } catch (const BuildRetry&) {
      continue;
    }
    break;
  }
  out.stride = reads.stride;
  out.n_reads = reads.n;
}

void prepare_ref_index(Ctx& c, const Ref& ref, unsigned q) {
  if (ref.qidx.q == q) return;
  ref.qidx = RefQIndex();
  // QGM_REF_UNPACKED=1 forces the separate extra-byte array (test knob: the
  // packed layout covers every reference below 2^28 padded bases)
  const char* force = std::getenv("QGM_REF_UNPACKED");
  const bool packed = ref.padded_total < (uint64_t(1) << kPackedPosBits) && !(force && force[0] == '1');
  Buckets B;
  uint64_t n_pal = 0;
  bucket_ref(c, ref, q, packed, B, &n_pal);
  index_from_buckets(c, B, false, ref.qidx.can, packed ? nullptr : &ref.qidx.extra);
  if (packed && ref.qidx.can.distinct) {
    // sort every interval's packed words: (extra bits, position) order groups
    // the occurrences by (strand flag, compare base) for the join's
    // suppression skip (once per reference and q)
    QGM_KERNEL(c, k_sort_intervals, unsigned(std::min<uint64_t>(ceil_div(ref.qidx.can.distinct, 128), kSMs * 16)),
               128, 0, ref.qidx.can.S1.p, ref.qidx.can.distinct, ref.qidx.can.O.p);
    ref.qidx.ex_sorted = true;
  }
  ref.qidx.packed = packed;
  ref.qidx.palindromes = n_pal;
  ref.qidx.positions = B.V - n_pal;
  ref.qidx.q = q;
  subbin_tables(c, ref, std::min(2 * q, 16u));
}

void subbin_tables(Ctx& c, const Ref& ref, unsigned sub_bits) {
  RefQIndex& X = ref.qidx;
  if (X.sub_bits == sub_bits) return;
  const unsigned q = X.q, cs = 2 * q - sub_bits;
  X.sub_bits = sub_bits;
  X.sb_d.release();
  X.sb_o.release();
  X.r16.release();
  // >= 8 group words per sub-bin (whole 16-byte bulk copies of I and r16) and
  // <= 2^16 codes (group starts inside a sub-bin fit 16 bits)
  if (cs >= 8 && cs <= 16) {
    const uint32_t n_sub = 1u << sub_bits;
    X.sb_d.alloc(c, n_sub + 1);
    X.sb_o.alloc(c, n_sub + 1);
    QGM_KERNEL(c, k_subbin_bounds, unsigned(ceil_div(n_sub + 1, 256)), 256, 0, X.can.S.p, X.can.S1.p, n_sub, cs,
               X.sb_d.p, X.sb_o.p);
    const uint64_t groups = X.can.groups;
    X.r16.alloc(c, groups);
    QGM_KERNEL(c, k_rank16, unsigned(std::min<uint64_t>(ceil_div(groups, 256), kSMs * 16)), 256, 0, X.can.S.p,
               groups, cs - 5, X.sb_d.p, X.r16.p);
  }
}

void sample_index(Ctx& c, const Index& in, Index& out) {
  out.q = in.q; out.w = in.w; out.groups = in.groups; out.distinct = in.distinct; out.occ = in.occ;
  out.stride = in.stride; out.n_reads = in.n_reads;
  out.I.alloc(c, in.I.n);
  QGM_CUDA(cudaMemcpyAsync(out.I.p, in.I.p, in.I.n, cudaMemcpyDeviceToDevice, c.stream));
  out.S1.alloc(c, in.S1.n);
  QGM_CUDA(cudaMemcpyAsync(out.S1.p, in.S1.p, in.S1.n * 4, cudaMemcpyDeviceToDevice, c.stream));
  out.O.alloc(c, in.O.n);
  QGM_CUDA(cudaMemcpyAsync(out.O.p, in.O.p, in.O.n * 4, cudaMemcpyDeviceToDevice, c.stream));
  if (in.sampled) {
    out.sampled = true;
    out.gs_len = in.gs_len;
    out.S.alloc(c, in.S.n);
    QGM_CUDA(cudaMemcpyAsync(out.S.p, in.S.p, in.S.n * 4, cudaMemcpyDeviceToDevice, c.stream));
    return;
  }
  out.sampled = true;
  out.gs_len = (in.gs_len + 1) / 2;
  out.S.alloc(c, out.gs_len);
  QGM_KERNEL(c, k_sample_S, unsigned(std::min<uint64_t>(ceil_div(out.gs_len, 256), kSMs * 8)), 256, 0, in.S.p,
             in.gs_len, out.S.p, out.gs_len);
}

void normalize_index(Ctx& c, Index& idx) {
  if (idx.distinct == 0) return;
  QGM_KERNEL(c, k_sort_intervals, unsigned(std::min<uint64_t>(ceil_div(idx.distinct, 128), kSMs * 16)), 128, 0,
             idx.S1.p, idx.distinct, idx.O.p);
}

void lookup_index(Ctx& c, const Index& idx, const uint32_t* d_codes, uint64_t n, uint32_t* d_begin,
                  uint32_t* d_end) {
  if (n == 0) return;
  const unsigned grid = unsigned(std::min<uint64_t>(ceil_div(n, 256), kSMs * 16));
  if (idx.w == 32)
    QGM_KERNEL(c, k_lookup<uint32_t>, grid, 256, 0, reinterpret_cast<const uint32_t*>(idx.I.p), idx.S.p, idx.S1.p,
               idx.sampled, d_codes, n, d_begin, d_end);
  else
    QGM_KERNEL(c, k_lookup<uint64_t>, grid, 256, 0, reinterpret_cast<const uint64_t*>(idx.I.p), idx.S.p, idx.S1.p,
               idx.sampled, d_codes, n, d_begin, d_end);
}

}  // namespace qgm
