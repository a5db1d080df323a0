// partition.cu -- per-batch read q-gram partition for the join (map path).
//
// The join (join.cu) only needs the batch's read q-grams grouped by the top
// bits of their canonical code (canon_code, RefQIndex), so that the warps in
// flight touch a few MiB of the reference index (L2-resident) instead of all
// of it; it never needs the full read-side q-group index. Passes:
//   P0 histogram : one CTA per SM counts the refined keys (top min(2q, 16)
//                  code bits) in shared memory (packed u16 counters) and
//                  flushes them with global atomics;
//   scan         : sub-bin offsets; the P1 bin offsets are their prefixes;
//   P1 scatter   : per chunk of 4096 q-gram slots (runs of 8 consecutive
//                  slots per thread sharing one register window of read
//                  bases), a local counting sort by bin in shared memory
//                  (the count atomic's return value is the item's rank),
//                  one global atomic per bin to reserve the chunk's run,
//                  then runs copied out with consecutive threads writing
//                  consecutive 8-byte slots;
//   P2 refine    : the same staged counting sort on the next code bits (up
//                  to 16 in total), per chunk of 2048 bin-ordered items that
//                  a bulk copy (mbarrier) brings into shared memory while
//                  the previous chunk is written out, producing the final
//                  join items at the offsets P0 already counted.
// ncu on an earlier single-pass scatter (12-bit bins, items written straight
// from registers) showed 1.6 GB of read-for-ownership and 2.1 GB of writes for
// 0.68 GB of output: partial sectors of 2.4M concurrently open runs.
//
// Everything the join needs from the read text is gathered in P1, where the
// read words are at hand (the join and P2 never touch the reads' bases): P1
// writes the final join item (layout in internal.hpp), P2 only moves it.
#include "internal.hpp"

namespace qgm {
namespace {

// P1 geometry (measured, C2 P1 ms: 256 threads x 3 CTAs/SM 0.455, 384 x 2
// 0.469, 512 x 2 0.407, 768 x 1 0.521, 1024 x 1 0.456): chunks of 4096 slots
// give bin runs of ~16 items (128 B) per chunk, two CTAs per SM keep 64
// registers free of spills for the pipelined loop.
#ifndef QGM_PART_THREADS
#define QGM_PART_THREADS 512
#endif
constexpr int kPartThreads = QGM_PART_THREADS;
#ifndef QGM_PART_MINB
#define QGM_PART_MINB 2
#endif
constexpr int kPartMinBlocks = QGM_PART_MINB;
constexpr unsigned kBinBits = 8;
constexpr uint32_t kBins = 1u << kBinBits;
constexpr uint32_t kChunk = 8 * kPartThreads;  // q-gram slots per chunk; staging = 8 B each
static_assert(kPartThreads >= int(kBins), "the P1 chunk scan gives every bin its own thread");
constexpr uint32_t kPer = kChunk / kPartThreads;
static_assert(kBins <= 256 && kChunk <= (1u << 24), "P1 packs bin | rank << 8 in 32 bits");
constexpr int kRun = 8;  // consecutive q-gram slots per thread (P0, P1)
static_assert(kPer % kRun == 0, "");
constexpr unsigned kP1CodeShift = kItemCodeShift, kP1MetaShift = kItemFbShift;  // P1 writes final join items

// Runs: R consecutive q-gram slots of ONE read -- a read's slots [0, span)
// are rpr = ceil(span / R) runs, the last one partial -- all cut from one
// 32-base register window that starts at base o0 - 1 (q + R + 1 <= 32), so a
// slot's code, left base and right base are constant shifts of a register.
// Q = compile-time q (0: the runtime value), so every shift is an immediate.
struct Run {
  uint32_t r, o0, n;
  uint64_t A;  // 32 read bases from o0 - 1, MSB-first
};

// reverse complement of 32 MSB-first bases: complement, reverse the 2-bit groups
__device__ __forceinline__ uint64_t revcomp32(uint64_t a) {
  const uint64_t x = ~a;
  const uint64_t r = (uint64_t(__brev(uint32_t(x))) << 32) | __brev(uint32_t(x >> 32));
  return ((r >> 1) & 0x5555555555555555ull) | ((r & 0x5555555555555555ull) << 1);
}

// kRaw: the q-gram's own code instead of its canonical code (the read-side
// q-group index of qgm_index_build, keyed by raw codes)
template <int Q, bool kRaw = false>
struct ItemGen {
  const uint64_t* words;
  const uint32_t* lengths;
  uint32_t W, stride, rpr, n_runs;
  FastDiv by_rpr;
  unsigned q_rt;
  __device__ __forceinline__ unsigned q() const { return Q ? unsigned(Q) : q_rt; }
  __device__ __forceinline__ uint64_t window(uint32_t r, uint32_t o) const {
    const uint64_t* w = words + uint64_t(r) * W;
    const uint32_t b = o + 31;  // base o-1, one word up: word -1 (zero) for o == 0
    const int k = int(b >> 5) - 1;
    const unsigned sh = 2 * (b & 31);
    const uint64_t w0 = k >= 0 ? __ldg(w + k) : 0ull;
    const uint64_t w1 = __ldg(w + k + 1);  // the read's own word, the next read's or the guard word
    return (w0 << sh) | ((w1 >> 1) >> (63 - sh));
  }
  template <int R>
  __device__ __forceinline__ void fetch_run(uint32_t run, Run& u) const {
    run = min(run, n_runs - 1);  // runs past the end load something valid and are dropped
    u.r = by_rpr.div(run);
    u.o0 = (run - u.r * rpr) * R;
    // a read longer than the stride is an input error (reported from the
    // batch flags); clamped, every pass counts the same slots and no item
    // exceeds the slot bound the buffers are sized by
    u.n = min(__ldg(lengths + u.r), stride);
    u.A = window(u.r, u.o0);
  }
  // Staged read words: the 16-byte-aligned word range [a0, a0 + nw) under
  // runs [c0, c1), up to and including the word after the range's last read
  // (the next read's first word or a guard word).
  __device__ __forceinline__ void word_range(uint32_t c0, uint32_t c1, uint32_t& a0, uint32_t& nw) const {
    const uint32_t rlo = by_rpr.div(c0), rhi = by_rpr.div(c1 - 1);
    a0 = (rlo * W) & ~1u;
    nw = (((rhi + 1) * W + 2) & ~1u) - a0;
  }
  // fetch_run from words staged in shared memory (sw holds words from a0);
  // n_uni: every read has this length (0: load it)
  template <int R>
  __device__ __forceinline__ void fetch_run_staged(uint32_t run, Run& u, const uint64_t* sw, uint32_t a0,
                                                   uint32_t n_uni) const {
    run = min(run, n_runs - 1);
    u.r = by_rpr.div(run);
    u.o0 = (run - u.r * rpr) * R;
    u.n = n_uni ? n_uni : min(__ldg(lengths + u.r), stride);
    const uint64_t* w = sw + (u.r * W - a0);
    const uint32_t b = u.o0 + 31;
    const int k = int(b >> 5) - 1;
    const unsigned sh = 2 * (b & 31);
    const uint64_t w0 = k >= 0 ? w[k] : 0ull;
    const uint64_t w1 = w[k + 1];
    u.A = (w0 << sh) | ((w1 >> 1) >> (63 - sh));
  }
  // slot j of a fetched run: canonical code g, own code f, meta, position.
  // RC = revcomp32(u.A), computed once per run by the caller.
  template <int R>
  __device__ __forceinline__ bool run_slot(uint32_t run, const Run& u, uint64_t RC, uint32_t j, uint32_t& f,
                                           uint32_t& g, uint32_t& m, uint32_t& pos) const {
    const unsigned q = this->q();
    const uint32_t o = u.o0 + j;
    f = uint32_t((u.A << (2 * j + 2)) >> (64 - 2 * q));
    // rc(f): bases j+1 .. j+q of A sit at bits [2j+2, 2j+2+2q) of RC
    const uint32_t rc = uint32_t(RC >> (2 * j + 2)) & (q == 16 ? 0xFFFFFFFFu : (1u << (2 * q)) - 1u);
    g = kRaw || f * 0x9E3779B1u <= rc * 0x9E3779B1u ? f : rc;  // canon_code(f, q)
    const uint32_t bl = uint32_t(u.A >> (62 - 2 * j)) & 3u;
    const uint32_t br = uint32_t(u.A >> (62 - 2 * (j + q + 1))) & 3u;
    m = (o ? bl : 4u) | ((o + q < u.n ? 3u - br : 4u) << 3) | (uint32_t(f != g) << 6);
    pos = u.r * stride + o;
    return run < n_runs && o + q <= u.n;
  }
};

// P0 over the refined keys: one CTA per SM counts the top key_bits bits of
// its contiguous share of the slots in shared memory -- two u16 counters per
// u32 word (128 KiB for 16-bit keys) -- and flushes the non-zero counts with
// global atomics. The P1 bin offsets and the P2 sub-bin offsets both come
// from this one histogram, so the refinement needs no counting pass. A u16
// counter hands 0x8000 to the global count whenever it reaches 0x8000.
constexpr int kHistThreads = 1024;
template <int Q, int R, bool kRaw>
__global__ void __launch_bounds__(kHistThreads, 1) k_part_hist16(ItemGen<Q, kRaw> gen, uint32_t per_cta, unsigned kshift,
                                                                 uint32_t keys, uint32_t* __restrict__ hist) {
  QGM_GRID_DEP();
  extern __shared__ uint32_t h2[];  // keys / 2 words (keys >= 2)
  const uint32_t words = (keys + 1) / 2;
  for (uint32_t i = threadIdx.x; i < words; i += kHistThreads) h2[i] = 0;
  __syncthreads();
  const uint32_t c0 = blockIdx.x * per_cta, c1 = min(gen.n_runs, c0 + per_cta);  // runs
  // Hand-off at half range: the increment that takes a counter from 0x7FFF
  // to 0x8000 moves 0x8000 to the global count and subtracts it. Counters
  // rise by 1 per atomic, so exactly one increment sees 0x7FFF per 0x8000
  // counted. Until the subtraction lands the counter can only climb by the
  // increments issued in that window (same-address shared atomics retire at
  // most one per clock: a window of 0x8000 cycles would be needed), so it
  // never reaches 0xFFFF and never carries into its neighbour.
  // The hand-offs of a run are collected in a bit mask and applied after its
  // slots (no branch around every counting atomic).
  constexpr int kRuns = R == 1 ? 4 : 1;  // runs in flight per thread
  constexpr int kSlots = kRuns * R;
  for (uint32_t t0 = c0; t0 < c1; t0 += kRuns * kHistThreads) {
    Run u[kRuns];
#pragma unroll
    for (int h = 0; h < kRuns; ++h) gen.template fetch_run<R>(t0 + h * kHistThreads + threadIdx.x, u[h]);
    uint32_t key[kSlots];
    uint32_t pend = 0;
#pragma unroll
    for (int h = 0; h < kRuns; ++h) {
      const uint32_t tr = t0 + h * kHistThreads + threadIdx.x;
      const uint64_t RC = revcomp32(u[h].A);
#pragma unroll
      for (int j = 0; j < R; ++j) {
        uint32_t f, g, m, pos;
        const bool ok = gen.template run_slot<R>(tr, u[h], RC, j, f, g, m, pos) && tr < c1;
        const uint32_t k = g >> kshift, sh = (k & 1u) * 16u;
        key[h * R + j] = k;
        // unconditional (an invalid slot adds 0): no branch around the atomic
        const uint32_t old = atomicAdd(h2 + (k >> 1), uint32_t(ok) << sh);
        pend |= uint32_t(ok && ((old >> sh) & 0xFFFFu) == 0x7FFFu) << (h * R + j);
      }
    }
    if (pend) {
#pragma unroll
      for (int e = 0; e < kSlots; ++e)
        if ((pend >> e) & 1u) {
          const uint32_t sh = (key[e] & 1u) * 16u;
          atomicAdd(hist + key[e], 0x8000u);
          atomicSub(h2 + (key[e] >> 1), 0x8000u << sh);
        }
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < words; i += kHistThreads) {
    const uint32_t w = h2[i];
    if (w & 0xFFFFu) atomicAdd(hist + 2 * i, w & 0xFFFFu);
    if (w >> 16) atomicAdd(hist + 2 * i + 1, w >> 16);
  }
}

// P1 bin offsets from the refined-key offsets: boff[b] = soff[b << sub]; and
// the batch flags (Partitioned::flags) from the upload's length extremes
__global__ void k_bin_offsets(const uint32_t* __restrict__ soff, uint32_t nbins, unsigned sub,
                              uint32_t* __restrict__ boff, const uint32_t* __restrict__ lens, uint32_t stride,
                              uint32_t keys, uint32_t* __restrict__ flags, uint32_t* __restrict__ cursors) {
  QGM_GRID_DEP();
  for (uint32_t b = threadIdx.x; b <= nbins; b += blockDim.x) boff[b] = soff[b << sub];
  for (uint32_t b = threadIdx.x; b <= kBins; b += blockDim.x) cursors[b] = 0;  // P1's per-bin cursors
  if (threadIdx.x == 0) {
    flags[0] = soff[keys];
    flags[1] = ~lens[1] == stride;
    flags[2] = lens[0] > stride;
  }
}

// P1, software-pipelined over the CTA's chunks: while chunk i's bin runs are
// being reserved (one global cursor atomic per bin, the round trip that
// dominated the stalls of the unpipelined loop) and written out, the items of
// chunk i+1 are generated and counted, and the read words of chunk i+2 (a
// contiguous range of reads) are on their way into shared memory by one bulk
// copy (C2: 0.407 -> 0.403 ms; staging P0's words the same way cost more in
// per-step barriers than it saved, 0.126 -> 0.146 ms).
template <int Q, int R, bool kRaw>
__global__ void __launch_bounds__(kPartThreads, kPartMinBlocks) k_part_scatter(ItemGen<Q, kRaw> gen, unsigned shift,
                                                                  const uint32_t* __restrict__ boff,
                                                                  uint32_t* __restrict__ cursor,
                                                                  uint64_t* __restrict__ out, uint32_t sw_words,
                                                                  const uint32_t* __restrict__ lens,
                                                                  uint32_t* __restrict__ clear, uint32_t n_clear) {
  QGM_GRID_DEP();
  // P0's histogram, read by the scan before this grid, becomes P2's per-key cursors
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_clear; i += gridDim.x * blockDim.x) clear[i] = 0;
  // kChunk items, bin-sorted | kChunk u8 bins | 2 x sw_words staged read words
  extern __shared__ __align__(16) uint64_t stage[];
  uint8_t* sbin = reinterpret_cast<uint8_t*>(stage + kChunk);
  uint64_t* swb = reinterpret_cast<uint64_t*>(sbin + kChunk);
  __shared__ uint32_t cnt[2][kBins], lofs[kBins], delta[kBins];
  __shared__ uint32_t ws[33];
  __shared__ __align__(8) uint64_t wbar[2];
  const uint32_t lmask = shift ? (1u << shift) - 1u : 0u;
  constexpr uint32_t kRuns = kPer / R;  // runs per thread per chunk
  constexpr uint32_t kChunkRuns = kRuns * kPartThreads;
  const uint32_t n_chunks = (gen.n_runs + kChunkRuns - 1) / kChunkRuns;
  uint32_t ch = blockIdx.x;
  if (ch >= n_chunks) return;  // CTA-uniform
  const uint32_t b = threadIdx.x;  // the bin this thread scans / reserves (b < kBins)
  for (uint32_t i = b; i < 2 * kBins; i += kPartThreads) (&cnt[0][0])[i] = 0;
  // every read of the batch as long as the stride: no per-run length load
  const uint32_t n_uni = ~__ldg(lens + 1) == gen.stride ? gen.stride : 0u;
  // the read words of the CTA's i-th chunk arrive by one bulk copy into
  // buffer i & 1, issued two chunks ahead
  auto issue = [&](uint32_t i, uint32_t c) {  // thread 0
    const uint32_t c0 = c * kChunkRuns, c1 = min(gen.n_runs, c0 + kChunkRuns);
    uint32_t a0, nw;
    gen.word_range(c0, c1, a0, nw);
    fence_proxy_async();
    mbar_arrive_expect_tx(&wbar[i & 1], nw * 8u);
    bulk_g2s(swb + (i & 1) * sw_words, gen.words + a0, nw * 8u, &wbar[i & 1]);
  };
  if (b == 0) {
    mbar_init(&wbar[0], 1);
    mbar_init(&wbar[1], 1);
    issue(0, ch);
    if (ch + gridDim.x < n_chunks) issue(1, ch + gridDim.x);
  }
  Run u[kRuns];
  auto fetch = [&](uint32_t i, uint32_t c) {  // the runs of the CTA's i-th chunk (chunk c)
    mbar_wait(&wbar[i & 1], (i >> 1) & 1u);
    const uint32_t c0 = c * kChunkRuns;
    uint32_t a0, nw;
    gen.word_range(c0, min(gen.n_runs, c0 + kChunkRuns), a0, nw);
#pragma unroll
    for (uint32_t h = 0; h < kRuns; ++h)
      gen.template fetch_run_staged<R>(c0 + h * kPartThreads + b, u[h], swb + (i & 1) * sw_words, a0, n_uni);
  };
  uint64_t item[kPer];
  uint32_t bin[kPer];  // bin | rank among the chunk's items of that bin << 8; ~0u = no q-gram at this slot
  // items of chunk c from the fetched runs (counted into cnt[par]); then the
  // runs of the CTA's next chunk are fetched
  auto generate = [&](uint32_t i, uint32_t c, uint32_t par) {
    fetch(i, c);
#pragma unroll
    for (uint32_t h = 0; h < kRuns; ++h) {
      const uint32_t tr = c * kChunkRuns + h * kPartThreads + b;
      const uint64_t RC = revcomp32(u[h].A);
#pragma unroll
      for (uint32_t j = 0; j < R; ++j) {
        const uint32_t e = h * R + j;
        uint32_t f, g, m, pos;
        const bool ok = gen.template run_slot<R>(tr, u[h], RC, j, f, g, m, pos);
        item[e] = (uint64_t(g & lmask) << kP1CodeShift) | (uint64_t(m) << kP1MetaShift) | pos;
        // the count's atomic returns the rank: placement needs no second atomic
        bin[e] = ok ? (g >> shift) | (atomicAdd(&cnt[par][g >> shift], 1u) << 8) : ~0u;
      }
    }
  };
  // local exclusive offsets of cnt[par]; the chunk's run in every bin reserved
  // (the reservation's value is only needed at the write-out); cnt[par] reset
  auto scan = [&](uint32_t par, uint32_t& g, uint32_t& total) {
    const uint32_t v = b < kBins ? cnt[par][b] : 0u;
    const uint32_t ex = block_exclusive_scan<uint32_t>(v, ws, &total);
    if (b < kBins) {
      lofs[b] = ex;
      g = v ? boff[b] + atomicAdd(cursor + b, v) : 0u;
      cnt[par][b] = 0;
    }
  };
  auto place = [&] {
#pragma unroll
    for (uint32_t k = 0; k < kPer; ++k)
      if (bin[k] != ~0u) {
        const uint32_t bb = bin[k] & 0xFFu, slot = lofs[bb] + (bin[k] >> 8);
        stage[slot] = item[k];
        sbin[slot] = uint8_t(bb);
      }
  };
  __syncthreads();  // counters zeroed, barriers initialised
  uint32_t par = 0, g = 0, total = 0, i = 0;
  generate(0, ch, par);
  __syncthreads();
  scan(par, g, total);
  __syncthreads();
  place();
  for (;; ++i) {
    const uint32_t nxt = ch + gridDim.x;
    const bool more = nxt < n_chunks;  // CTA-uniform
    if (more) generate(i + 1, nxt, par ^ 1u);  // overlaps the reservation round trip
    if (b < kBins) delta[b] = g - lofs[b];
    __syncthreads();  // staged chunk and its destinations visible; chunk i's words no longer read
    if (b == 0 && nxt + gridDim.x < n_chunks) issue(i + 2, nxt + gridDim.x);
    for (uint32_t x = b; x < total; x += kPartThreads) out[delta[sbin[x]] + x] = stage[x];
    if (!more) break;
    par ^= 1u;
    scan(par, g, total);  // its first barrier also ends the write-out
    __syncthreads();
    place();
    ch = nxt;
  }
}

// ---------------------------------------------------------------- refinement
// Second MSD pass: items grouped by their P1 bin (top `bits` code bits) are
// regrouped by their top `key_bits` (<= 16) bits. A chunk of 4096 consecutive
// items spans few P1 bins, so its keys fall in a small window
// [first_bin << sub, (last_bin + 1) << sub); the window is counted and staged
// in shared memory exactly like P1 (kLocal keys max), with a per-item global
// fallback for chunks whose window is wider (tiny bins). The P1 bin of item i
// is found from the bin offsets (staged in shared memory) with a per-thread
// cursor that only moves forward.
constexpr uint32_t kLocal = 1024;
// P2 geometry: its own chunk (items bulk-copied into shared memory) and CTA size
#ifndef QGM_P2_THREADS
#define QGM_P2_THREADS 256
#endif
constexpr int kP2Threads = QGM_P2_THREADS;
#ifndef QGM_P2_PER
#define QGM_P2_PER 8
#endif
#ifndef QGM_P2_MINB
#define QGM_P2_MINB (1024 / QGM_P2_THREADS)
#endif
constexpr int kP2MinBlocks = QGM_P2_MINB;
constexpr uint32_t kP2Per = QGM_P2_PER;
constexpr uint32_t kP2Chunk = kP2Per * kP2Threads;

struct Refine {
  unsigned shift;    // code bits below the P1 bin (in the item)
  unsigned kshift;   // code bits below the refined key
  uint32_t nbins;    // P1 bins
  __device__ __forceinline__ uint32_t key(uint64_t it, uint32_t bin) const {
    return (bin << (shift - kshift)) | (uint32_t(it >> kP1CodeShift) >> kshift);
  }
};

// largest b with boff[b] <= i (i < total)
__device__ __forceinline__ uint32_t bin_search(const uint32_t* sboff, uint32_t nbins, uint32_t i) {
  uint32_t lo = 0, hi = nbins;  // invariant: boff[lo] <= i < boff[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (sboff[mid] <= i) lo = mid; else hi = mid;
  }
  return lo;
}

// per P2 chunk: {first P1 bin | last P1 bin << 16, first key of the
// chunk's key window, window width}, so a scatter CTA starts a chunk without
// a dependent load or a binary search
__global__ void k_chunk_info(const uint64_t* __restrict__ in, const uint32_t* __restrict__ n_dev,
                             const uint32_t* __restrict__ boff, Refine rf, unsigned sub, uint4* __restrict__ info) {
  QGM_GRID_DEP();
  const uint32_t n = *n_dev;
  const uint32_t n_chunks = (n + kP2Chunk - 1) / kP2Chunk;
  for (uint32_t ch = blockIdx.x * blockDim.x + threadIdx.x; ch < n_chunks; ch += gridDim.x * blockDim.x) {
    const uint32_t c0 = ch * kP2Chunk, c1 = min(n, c0 + kP2Chunk);
    const uint32_t bfirst = bin_search(boff, rf.nbins, c0), blast = bin_search(boff, rf.nbins, c1 - 1);
    const uint32_t base = (rf.key(in[c0], bfirst) >> sub) << sub;
    const uint32_t width = (((rf.key(in[c1 - 1], blast) >> sub) + 1) << sub) - base;
    info[ch] = make_uint4(bfirst | (blast << 16), base, width, 0u);
  }
}

__global__ void __launch_bounds__(kP2Threads, kP2MinBlocks) k_refine_scatter(const uint64_t* __restrict__ in,
                                                                    const uint32_t* __restrict__ n_dev,
                                                                    const uint32_t* __restrict__ boff, Refine rf,
                                                                    unsigned sub, const uint32_t* __restrict__ off,
                                                                    uint32_t* __restrict__ cursor,
                                                                    const uint4* __restrict__ chunk_info,
                                                                    uint64_t* __restrict__ out) {
  QGM_GRID_DEP();
  // dynamic: the chunk's items as loaded by TMA (kP2Chunk u64), the sorted
  // join items (kP2Chunk u64), their window keys (kP2Chunk u16)
  extern __shared__ __align__(16) uint64_t sdyn[];
  uint64_t* sin = sdyn;
  uint64_t* stage = sdyn + kP2Chunk;
  uint16_t* skey = reinterpret_cast<uint16_t*>(stage + kP2Chunk);
  __shared__ uint32_t cnt[kLocal], lofs[kLocal], gdst[kLocal];
  __shared__ uint32_t sboff[kBins + 1];
  __shared__ uint32_t ws[33];
  __shared__ __align__(8) uint64_t s_bar;
  const uint32_t n = *n_dev;  // V (the grid is sized by its host-side bound)
  for (uint32_t b = threadIdx.x; b <= rf.nbins; b += kP2Threads) sboff[b] = boff[b];
  const uint32_t n_chunks = (n + kP2Chunk - 1) / kP2Chunk;
  // one elected thread moves each chunk's items into shared memory with a
  // bulk copy issued while the previous chunk is sorted and written out
  auto fetch = [&](uint32_t ch) {
    const uint32_t a0 = ch * kP2Chunk, a1 = min(n, a0 + kP2Chunk);
    const uint32_t bytes = ((a1 - a0) * 8u + 15u) & ~15u;  // the buffer holds n + 2 items
    fence_proxy_async();
    mbar_arrive_expect_tx(&s_bar, bytes);
    bulk_g2s(sin, in + a0, bytes, &s_bar);
  };
  if (threadIdx.x == 0) {
    mbar_init(&s_bar, 1);
    if (blockIdx.x < n_chunks) fetch(blockIdx.x);
  }
  __syncthreads();
  uint32_t phase = 0;
  uint4 ci_next = blockIdx.x < n_chunks ? __ldg(chunk_info + blockIdx.x) : make_uint4(0, 0, 0, 0);
  for (uint32_t ch = blockIdx.x; ch < n_chunks; ch += gridDim.x) {
    const uint32_t c0 = ch * kP2Chunk, c1 = min(n, c0 + kP2Chunk);
    const uint4 ci = ci_next;
    const bool more = ch + gridDim.x < n_chunks;
    if (more) ci_next = __ldg(chunk_info + ch + gridDim.x);  // next chunk's info one iteration ahead
    mbar_wait(&s_bar, phase);
    phase ^= 1u;
    const uint32_t bfirst = ci.x & 0xFFFFu, blast = ci.x >> 16;
    const uint32_t base = ci.y, width = ci.z;
    uint32_t b = bfirst;
    if (width > kLocal) {
      for (uint32_t i = c0 + threadIdx.x; i < c1; i += kP2Threads) {
        while (sboff[b + 1] <= i) ++b;
        const uint64_t it = sin[i - c0];
        const uint32_t k = rf.key(it, b);
        out[off[k] + atomicAdd(cursor + k, 1u)] = it;
      }
      __syncthreads();  // every thread is done with sin
      if (threadIdx.x == 0 && more) fetch(ch + gridDim.x);
      continue;
    }
    for (uint32_t k = threadIdx.x; k < width; k += kP2Threads) cnt[k] = 0;
    __syncthreads();
    uint64_t v[kP2Per];
    uint32_t kk[kP2Per];
#pragma unroll
    for (uint32_t k = 0; k < kP2Per; ++k) {
      const uint32_t i = c0 + k * kP2Threads + threadIdx.x;
      v[k] = sin[min(i, c1 - 1) - c0];
    }
#pragma unroll
    for (uint32_t k = 0; k < kP2Per; ++k) {
      const uint32_t i = c0 + k * kP2Threads + threadIdx.x;
      if (i < c1 && bfirst != blast)
        while (sboff[b + 1] <= i) ++b;
      kk[k] = i < c1 ? rf.key(v[k], b) - base : ~0u;
      if (i < c1) atomicAdd(cnt + kk[k], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0 && more) fetch(ch + gridDim.x);  // every thread has its items in registers
    // exclusive scan of cnt[0, width): each thread owns a contiguous run
    const uint32_t per = (width + kP2Threads - 1) / kP2Threads;
    const uint32_t k0 = threadIdx.x * per, k1 = min(width, k0 + per);
    uint32_t s = 0;
    for (uint32_t k = k0; k < k1; ++k) s += cnt[k];
    // the first key's reservation is issued before the scan (its round trip
    // overlaps the barriers); usually per == 1
    const uint32_t c_first = k0 < k1 ? cnt[k0] : 0u;
    const uint32_t g_first = c_first ? off[base + k0] + atomicAdd(cursor + base + k0, c_first) : 0u;
    uint32_t tot;
    uint32_t run = block_exclusive_scan<uint32_t>(s, ws, &tot);
    for (uint32_t k = k0; k < k1; ++k) {
      const uint32_t cv = cnt[k];
      lofs[k] = run;
      gdst[k] = k == k0 ? g_first : cv ? off[base + k] + atomicAdd(cursor + base + k, cv) : 0u;
      cnt[k] = run;
      run += cv;
    }
    __syncthreads();
#pragma unroll
    for (uint32_t k = 0; k < kP2Per; ++k)
      if (kk[k] != ~0u) {
        const uint32_t slot = atomicAdd(cnt + kk[k], 1u);
        stage[slot] = v[k];
        skey[slot] = uint16_t(kk[k]);
      }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < c1 - c0; i += kP2Threads) {
      const uint32_t k = skey[i];
      out[gdst[k] + (i - lofs[k])] = stage[i];
    }
    __syncthreads();
  }
}

}  // namespace

// P0 + P1 for one (Q, R) instantiation (Q = compile-time q or 0, R = run length).
template <int Q, int R, bool kRaw>
static void p0_p1(Ctx& c, const ItemGen<Q, kRaw>& gen, const Reads& reads, unsigned q, unsigned key_bits, unsigned bits,
                  Partitioned& out, DBuf<uint32_t>& h2, DBuf<uint64_t>& p1, uint32_t& V) {
  const uint32_t keys = 1u << key_bits;
  const unsigned sub = key_bits - bits, shift = 2 * q - bits;
  {
    const uint32_t per_cta = uint32_t(ceil_div(ceil_div(gen.n_runs, uint64_t(kSMs)), kHistThreads) * kHistThreads);
    const size_t hsmem = size_t((keys + 1) / 2) * 4;
    auto kern = k_part_hist16<Q, R, kRaw>;
    ensure_dynamic_smem(reinterpret_cast<const void*>(kern), size_t(hsmem));
    KernelScope ks(c, "k_part_hist");
    QGM_KERNEL(c, kern, unsigned(ceil_div(gen.n_runs, per_cta)), kHistThreads, hsmem, gen, per_cta,
               2 * q - key_bits, keys, h2.p);
  }
  exclusive_scan_u32(c, h2.p, out.soff.p, keys + 1, nullptr, nullptr);
  // no host round trip: V stays on the device (flags[0]); buffers are sized by
  // the slot count, which equals V for a batch of full-length reads
  DBuf<uint32_t> hist(c, kBins + 1);  // per-bin cursors of P1 (zeroed by k_bin_offsets)
  QGM_KERNEL(c, k_bin_offsets, 1, 256, 0, out.soff.p, 1u << bits, sub, out.boff.p, reads.lens.p, reads.stride, keys,
             out.flags.p, hist.p);
  p1.alloc(c, uint64_t(V) + 2);  // +2: P2 bulk-copies whole 16-byte pairs
  const uint32_t chunk_runs = kChunk / R;
  // staged words per chunk: the reads under chunk_runs runs (+2 partial) and
  // the following word, rounded to 16-byte pairs
  const uint32_t sw_words = ((chunk_runs / gen.rpr + 2) * reads.W + 4 + 1) & ~1u;
  const size_t smem = kChunk * (sizeof(uint64_t) + sizeof(uint8_t)) + size_t(2) * sw_words * sizeof(uint64_t);
  auto p1kern = k_part_scatter<Q, R, kRaw>;
  ensure_dynamic_smem(reinterpret_cast<const void*>(p1kern), size_t(smem));
  const unsigned grid = unsigned(std::min<uint64_t>(ceil_div(gen.n_runs, chunk_runs), uint64_t(kSMs) * kPartMinBlocks));
  KernelScope ks(c, "k_part_scatter");
  QGM_KERNEL(c, p1kern, grid, kPartThreads, smem, gen, shift, out.boff.p, hist.p, p1.p, sw_words, reads.lens.p, h2.p,
             keys + 1);
}

template <int Q, bool kRaw>
static void p0_p1_runs(Ctx& c, const Reads& reads, unsigned q, uint32_t span, unsigned key_bits, unsigned bits,
                       Partitioned& out, DBuf<uint32_t>& h2, DBuf<uint64_t>& p1, uint32_t& V) {
  ItemGen<Q, kRaw> gen;
  gen.words = reads.words.p;
  gen.lengths = reads.lengths.p;
  gen.W = reads.W;
  gen.stride = reads.stride;
  gen.q_rt = q;
  // runs of kRun slots per thread; one slot per thread for reads with fewer
  // than kRun q-gram slots
  const int R = span >= uint32_t(kRun) ? kRun : 1;
  gen.rpr = uint32_t(ceil_div(span, R));
  gen.by_rpr = FastDiv(std::max<uint32_t>(gen.rpr, 1));
  const uint64_t n_runs = uint64_t(reads.n) * gen.rpr;
  if (n_runs * R > 0xFFFFFFFFull - kChunk) throw InputError("read batch has more than 2^32-1 q-gram slots");
  gen.n_runs = uint32_t(n_runs);
  if (R == kRun) p0_p1<Q, kRun, kRaw>(c, gen, reads, q, key_bits, bits, out, h2, p1, V);
  else p0_p1<Q, 1, kRaw>(c, gen, reads, q, key_bits, bits, out, h2, p1, V);
}

void partition_reads(Ctx& c, const Reads& reads, unsigned q, Partitioned& out, bool raw, unsigned force_key_bits) {
  if (q == 0 || q > 16) throw InputError("q must be in [1, 16]");
  const uint32_t span = reads.stride >= q ? reads.stride - q + 1 : 0;
  const uint64_t n_items64 = uint64_t(reads.n) * span;
  if (n_items64 > 0xFFFFFFFFull - kChunk) throw InputError("read batch has more than 2^32-1 q-gram slots");
  const uint32_t n_items = uint32_t(n_items64);
  const unsigned bits = std::min(2 * q, kBinBits);
  const unsigned shift = 2 * q - bits;
  // sub-bins of ~256+ read q-grams: small batches get fewer, wider sub-bins
  // (per-sub-bin staging and synchronisation are the join's fixed costs);
  // at most 16 bits, at least the first pass's bits, and a sub-bin never
  // spans more than 2^16 codes (u16 group starts) -- so q=16 always uses 16
  unsigned key_bits = std::min(2 * q, 16u);
  {
    unsigned want = 8;
    while (want < 16 && (uint64_t(n_items) >> (want + 1)) >= 256) ++want;
    want = std::max(want, 2 * q > 16 ? 2 * q - 16 : 0u);
    key_bits = std::min(key_bits, std::max(want, std::min(2 * q, kBinBits)));
  }
  if (force_key_bits) {
    if (force_key_bits < std::min(2 * q, kBinBits) || force_key_bits > std::min(2 * q, 16u))
      throw InternalError("partition: key width outside [first-pass bits, 16]");
    key_bits = force_key_bits;
  }
  out.q = q;
  out.bins = 1u << bits;
  out.sub_bits = key_bits;
  out.boff.alloc(c, kBins + 1);
  out.flags.alloc(c, 4);
  out.V = 0;
  if (n_items == 0) {  // no read has a q-gram
    out.flags.zero();
    out.boff.zero();
    out.pairs.alloc(c, 1);
    out.soff.alloc(c, (1u << key_bits) + 1);
    out.soff.zero();
    return;
  }
  // P0: histogram of the refined keys (the P1 bins are its prefixes); P1
  const uint32_t keys = 1u << key_bits;
  const unsigned sub = key_bits - bits;
  out.soff.alloc(c, keys + 1);
  DBuf<uint32_t> h2(c, keys + 1);
  h2.zero();
  DBuf<uint64_t> p1;
  uint32_t V = n_items;  // bound; the exact count is flags[0]
  if (raw) {
    if (q == 16) p0_p1_runs<16, true>(c, reads, q, span, key_bits, bits, out, h2, p1, V);
    else p0_p1_runs<0, true>(c, reads, q, span, key_bits, bits, out, h2, p1, V);
  } else if (q == 16) {
    p0_p1_runs<16, false>(c, reads, q, span, key_bits, bits, out, h2, p1, V);
  } else if (q == 12) {
    p0_p1_runs<12, false>(c, reads, q, span, key_bits, bits, out, h2, p1, V);
  } else {
    p0_p1_runs<0, false>(c, reads, q, span, key_bits, bits, out, h2, p1, V);
  }
  out.V = V;
  // P2: refine to the top min(2q, 16) code bits (short reuse distance of the
  // reference-index sectors in the join) and convert to join items. Runs even
  // when P1 already grouped by every key bit (2q <= 8): then it only converts.
  Refine rf;
  rf.shift = shift;
  rf.kshift = 2 * q - key_bits;
  rf.nbins = 1u << bits;
  const unsigned grid2 = unsigned(std::min<uint64_t>(ceil_div(V, kP2Chunk), uint64_t(kSMs) * kP2MinBlocks));
  // h2: P2's per-key cursors, zeroed by P1
  out.pairs.alloc(c, V + 2);  // +2: the join bulk-copies whole 16-byte pairs of items
  const size_t smem2 = kP2Chunk * (2 * sizeof(uint64_t) + sizeof(uint16_t));
  ensure_dynamic_smem(reinterpret_cast<const void*>(k_refine_scatter), size_t(smem2));
  const uint32_t n_chunks2 = uint32_t(ceil_div(V, kP2Chunk));
  DBuf<uint4> chunk_info(c, n_chunks2);
  QGM_KERNEL(c, k_chunk_info, unsigned(ceil_div(n_chunks2, 256)), 256, 0, p1.p, out.flags.p, out.boff.p, rf, sub,
             chunk_info.p);
  {
    KernelScope ks(c, "k_refine_scatter");
    QGM_KERNEL(c, k_refine_scatter, grid2, kP2Threads, smem2, p1.p, out.flags.p, out.boff.p, rf, sub, out.soff.p, h2.p,
               chunk_info.p, out.pairs.p);
  }
}

}  // namespace qgm
