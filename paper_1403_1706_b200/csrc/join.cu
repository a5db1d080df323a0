// join.cu -- stage 2, production path: filtration as a code-ordered join.
//
// Same candidate semantics as filter.cu (Alg. 2; Appendix
// B.1-B.3): a forward candidate (r, +, p - o) for every reference position p
// whose q-gram equals the read q-gram at offset o, a reverse candidate
// (r, -, p + o + q - n) for every p whose reverse-complemented q-gram equals it.
//
// Why a join: streaming the 2L reference q-grams against a 4^q-code read
// index makes every lookup a random probe into a 512 MiB occupancy array
// (q=16); ncu shows each probe costing ~100 B of HBM traffic
// (profiles/r01/README.md). Here the reference side is a q-group index built
// once per reference and q (prepare_ref_index -- the paper's reference index
// with P ordered by q-gram), one per strand, and the batch's read
// q-grams are partitioned by the top 16 bits of their code (partition.cu).
//
// One CTA owns one code sub-bin at a time (2^(2q-16) codes; 2048 group words
// per array at q=16): it stages the sub-bin's occupancy and group-start words
// of both reference strands in shared memory with one coalesced load, so all
// Group-And-Bit / Grouprank lookups of the sub-bin's read q-grams are shared
// memory hits; the S' / O / prev reads that follow fall in the sub-bin's
// contiguous slice of the reference index and are L1/L2 local to the CTA. The
// occupancy/group-start arrays are read from HBM exactly once per batch, in
// order.
//
// Per warp step: up to 4 read q-grams per lane, both strands looked up, then
// the union of the occurrence intervals expanded cooperatively, one
// (reference occurrence, read occurrence) pair per lane. The run-start rule
// uses the base stored next to every reference occurrence (prev_fwd/prev_rc,
// 4 = no predecessor) against the read base at o-1 (forward) or o+q (RC).
#include "internal.hpp"

namespace qgm {
namespace {

constexpr int kJoinThreads = 256;
constexpr int kJoinWarps = kJoinThreads / 32;
constexpr int kItems = 4;                 // read q-grams per lane per step
constexpr int kSlots = 2 * kItems;        // (item, strand) lookups per lane
constexpr int kRanges = 32 * kSlots;
constexpr int kStage = 128;               // staged keys per warp
constexpr uint32_t kInline = 4;           // intervals up to this length are expanded in-lane
constexpr uint32_t kMaxWords = 2048;      // group words per sub-bin and array (q = 16)

struct JoinArgs {
  const uint64_t* items;
  const uint32_t* soff;
  uint32_t n_sub;
  unsigned code_shift;  // sub-bin = code >> code_shift
  uint32_t words;       // group words per sub-bin (>= 1)
  unsigned q;
  const uint32_t *If, *Sf, *S1f, *Of;
  const uint8_t* Xf;
  const uint32_t *Ir, *Sr, *S1r, *Or;
  const uint8_t* Xr;
  const uint64_t* rwords;
  const uint32_t* rlen;
  uint32_t W, m;
  FastDiv by_m;
  const uint64_t* cb;
  const uint64_t* cbp;
  uint32_t n_chrom;
  int strands;
  unsigned diag_bits;
  uint64_t* out;
  uint64_t cap;
  unsigned long long* counter;
  unsigned long long* stats;
};

// One (reference occurrence k, read q-gram pw) pair -> candidate key; false if
// the run-start rule suppresses it (the (q+1)-gram one base to the left on the
// same diagonal also matches).
template <bool kRunStart>
__device__ __forceinline__ bool expand(const JoinArgs& a, unsigned q, uint32_t k, uint32_t pw, uint64_t& key) {
  const bool rev = pw >> 31;
  const uint32_t pp = pw & 0x7FFFFFFFu;
  const uint32_t r = a.by_m.div(pp), o = pp - r * a.m;
  // independent loads: occurrence, its stored predecessor base, the read
  // length and the read word holding the compared base
  const uint32_t cmp = rev ? o + q : (o ? o - 1 : 0);
  const uint32_t x = __ldg((rev ? a.Or : a.Of) + k);
  const uint32_t pv = kRunStart ? uint32_t(__ldg((rev ? a.Xr : a.Xf) + k)) : 4u;
  const uint32_t n = __ldg(a.rlen + r);
  const uint64_t rword = kRunStart ? __ldg(a.rwords + uint64_t(r) * a.W + (cmp >> 5)) : 0ull;
  if (kRunStart && pv != 4 && (rev ? (o + q + 1 <= n) : (o >= 1)) &&
      pv == (uint32_t(rword >> (62 - 2 * (cmp & 31))) & 3u))
    return false;
  uint32_t c = 0, hi = a.n_chrom;  // chromosome of x
  while (hi - c > 1) {
    const uint32_t mid = (c + hi) >> 1;
    if (__ldg(a.cb + mid) <= x) c = mid; else hi = mid;
  }
  const int64_t p = int64_t(x) - int64_t(__ldg(a.cb + c));
  const int64_t d = rev ? p + int64_t(o) + int64_t(q) - int64_t(n) : p - int64_t(o);
  const uint64_t gp = uint64_t(int64_t(__ldg(a.cbp + c)) + d);
  key = (uint64_t(r) << (a.diag_bits + 1)) | (uint64_t(rev) << a.diag_bits) | gp;
  return true;
}

template <bool kRunStart>
__global__ void __launch_bounds__(kJoinThreads, 4) k_join(JoinArgs a) {
  extern __shared__ uint32_t s_words[];  // [I fwd | I rc | S fwd | S rc], a.words each
  uint32_t* sI[2] = {s_words, s_words + a.words};
  uint32_t* sS[2] = {s_words + 2 * a.words, s_words + 3 * a.words};
  __shared__ uint32_t s_k0[kJoinWarps][kRanges];
  __shared__ uint32_t s_pre[kJoinWarps][kRanges + 1];
  __shared__ uint32_t s_pos[kJoinWarps][kRanges];  // read text position | strand << 31
  __shared__ uint64_t s_out[kJoinWarps][kStage];

  const unsigned lane = lane_id(), wid = threadIdx.x >> 5;
  const unsigned q = a.q;
  uint32_t staged = 0;
  unsigned long long n_hit = 0, n_occ = 0;

  auto flush = [&]() {
    unsigned long long base = 0;
    if (lane == 0 && staged) base = atomicAdd(a.counter, (unsigned long long)staged);
    base = __shfl_sync(kFull, base, 0);
    for (uint32_t i = lane; i < staged; i += 32)
      if (base + i < a.cap) a.out[base + i] = s_out[wid][i];
    staged = 0;
    __syncwarp();
  };
  auto stage_key = [&](bool emit, uint64_t key) {  // all lanes call it
    const unsigned m = __ballot_sync(kFull, emit);
    if (emit) s_out[wid][staged + __popc(m & lanemask_lt())] = key;
    staged += __popc(m);
    __syncwarp();
    if (staged > kStage - 32) flush();
  };

  for (uint32_t sb = blockIdx.x; sb < a.n_sub; sb += gridDim.x) {
    const uint32_t b0 = __ldg(a.soff + sb), b1 = __ldg(a.soff + sb + 1);
    if (b0 == b1) continue;  // CTA-uniform
    // first group word of the sub-bin (sub-bins narrower than a word share it)
    const uint32_t w0 = uint32_t((uint64_t(sb) << a.code_shift) >> 5);
    for (uint32_t i = threadIdx.x; i < a.words; i += kJoinThreads) {
      if (a.strands & 1) { sI[0][i] = __ldg(a.If + w0 + i); sS[0][i] = __ldg(a.Sf + w0 + i); }
      if (a.strands & 2) { sI[1][i] = __ldg(a.Ir + w0 + i); sS[1][i] = __ldg(a.Sr + w0 + i); }
    }
    // warm L2 with the next sub-bin's words while this one is processed
    {
      const uint32_t nsb = sb + gridDim.x;
      const uint32_t bytes = a.words * 4u;
      if (nsb < a.n_sub && threadIdx.x * 128u < 4u * bytes) {
        const uint32_t arr = (threadIdx.x * 128u) / bytes, off = (threadIdx.x * 128u) % bytes;
        const uint32_t* src = arr == 0 ? a.If : arr == 1 ? a.Ir : arr == 2 ? a.Sf : a.Sr;
        const char* p = reinterpret_cast<const char*>(src + uint32_t((uint64_t(nsb) << a.code_shift) >> 5)) + off;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
      }
    }
    __syncthreads();
    // the sub-bin's items split evenly over the warps (no warp idles at the
    // end-of-sub-bin barrier while another runs a second full round)
    const uint32_t nitems = b1 - b0;
    const uint32_t my_lo = b0 + uint32_t(uint64_t(nitems) * wid / kJoinWarps);
    const uint32_t my_hi = b0 + uint32_t(uint64_t(nitems) * (wid + 1) / kJoinWarps);
    for (uint32_t base = my_lo; base < my_hi; base += 32 * kItems) {  // warp-uniform bound
      uint32_t cnt = 0, nr = 0, rk0[kSlots], rn[kSlots], rpos[kSlots];
      uint64_t pr[kItems];
#pragma unroll
      for (int u = 0; u < kItems; ++u) {
        const uint32_t it = base + u * 32 + lane;
        pr[u] = it < my_hi ? __ldg(a.items + it) : ~0ull;
      }
#pragma unroll
      for (int s = 0; s < kSlots; ++s) {
        const int u = s >> 1, st = s & 1;
        const bool ok = pr[u] != ~0ull && (a.strands & (1 << st));
        const uint32_t g = uint32_t(pr[u] >> 32);
        const uint32_t wl = (g >> 5) - w0, bit = g & 31u;
        const uint32_t w = ok ? sI[st][wl] : 0u;
        const bool hit = (w >> bit) & 1u;
        const uint32_t b = (hit ? sS[st][wl] : 0u) + __popc(w & ((1u << bit) - 1u));
        const uint32_t* S1 = st ? a.S1r : a.S1f;
        rk0[s] = hit ? __ldg(S1 + b) : 0u;
        rn[s] = hit ? __ldg(S1 + b + 1) : 0u;
        rpos[s] = uint32_t(pr[u]) | (st ? 0x80000000u : 0u);
      }
#pragma unroll
      for (int s = 0; s < kSlots; ++s) {
        rn[s] -= rk0[s];
        cnt += rn[s];
        nr += rn[s] != 0;
      }
      n_hit += nr;
      n_occ += cnt;
      if (__all_sync(kFull, cnt == 0)) continue;
      // compact the non-empty (q-gram, strand) lookups of the warp into a list
      uint32_t nent = 0;
#pragma unroll
      for (int s = 0; s < kSlots; ++s) {
        const bool has = rn[s] != 0;
        const unsigned bm = __ballot_sync(kFull, has);
        if (has) {
          const uint32_t e = nent + __popc(bm & lanemask_lt());
          s_k0[wid][e] = rk0[s];
          s_pre[wid][e] = rn[s];
          s_pos[wid][e] = rpos[s];
        }
        nent += __popc(bm);
      }
      __syncwarp();
      // one list entry per lane per round; intervals of up to kInline
      // occurrences (almost all of them) are expanded in the lane, longer ones
      // (repeats) by the whole warp, one interval at a time
      for (uint32_t e0 = 0; e0 < nent; e0 += 32) {
        const uint32_t e = e0 + lane;
        uint32_t k0 = 0, len = 0, pw = 0;
        if (e < nent) {
          k0 = s_k0[wid][e];
          len = s_pre[wid][e];
          pw = s_pos[wid][e];
        }
        const bool longi = len > kInline;
        const uint32_t nin = longi ? 0u : len;
        const uint32_t rounds = __reduce_max_sync(kFull, nin);
        for (uint32_t t = 0; t < rounds; ++t) {
          uint64_t key = 0;
          const bool emit = t < nin && expand<kRunStart>(a, q, k0 + t, pw, key);
          stage_key(emit, key);
        }
        unsigned lm = __ballot_sync(kFull, longi);
        while (lm) {
          const int src = __ffs(lm) - 1;
          lm &= lm - 1;
          const uint32_t lk0 = __shfl_sync(kFull, k0, src), llen = __shfl_sync(kFull, len, src);
          const uint32_t lpw = __shfl_sync(kFull, pw, src);
          for (uint32_t t0 = 0; t0 < llen; t0 += 32) {
            uint64_t key = 0;
            const bool emit = t0 + lane < llen && expand<kRunStart>(a, q, lk0 + t0 + lane, lpw, key);
            stage_key(emit, key);
          }
        }
      }
      __syncwarp();
    }
    __syncthreads();  // shared words are reloaded for the next sub-bin
  }
  flush();
  n_hit = warp_reduce_sum(n_hit);
  n_occ = warp_reduce_sum(n_occ);
  if (lane == 0 && a.stats && n_hit) {
    atomicAdd(a.stats, n_hit);
    atomicAdd(a.stats + 1, n_occ);
  }
}

}  // namespace

uint64_t join_filter(Ctx& c, const Partitioned& rp, const Reads& reads, const Ref& ref, int strands, int mode,
                     unsigned read_bits, DBuf<uint64_t>& keys, uint64_t* fstats) {
  if (read_bits + 1 + ref.diag_bits > 64) throw InputError("read batch too large for the 64-bit candidate key");
  if (reads.max_len + 64 > ref.gap) throw InputError("reads longer than the reference padding supports");
  prepare_ref_index(c, ref, rp.q);
  const RefQIndex& X = ref.qidx;
  JoinArgs a;
  a.items = rp.pairs.p;
  a.soff = rp.soff.p;
  a.n_sub = 1u << rp.sub_bits;
  a.code_shift = 2 * rp.q - rp.sub_bits;
  a.words = std::max<uint32_t>(1, (1u << a.code_shift) / 32);
  if (a.words > kMaxWords) throw InternalError("join: sub-bin wider than the shared staging");
  a.q = rp.q;
  a.If = reinterpret_cast<const uint32_t*>(X.fwd.I.p);
  a.Sf = X.fwd.S.p;
  a.S1f = X.fwd.S1.p;
  a.Of = X.fwd.O.p;
  a.Xf = X.prev_fwd.p;
  a.Ir = reinterpret_cast<const uint32_t*>(X.rc.I.p);
  a.Sr = X.rc.S.p;
  a.S1r = X.rc.S1.p;
  a.Or = X.rc.O.p;
  a.Xr = X.prev_rc.p;
  a.rwords = reads.words.p;
  a.rlen = reads.lengths.p;
  a.W = reads.W;
  a.m = reads.stride;
  a.by_m = FastDiv(std::max<uint32_t>(reads.stride, 1));
  a.cb = ref.d_cb.p;
  a.cbp = ref.d_cbp.p;
  a.n_chrom = ref.n_chrom;
  a.strands = strands;
  a.diag_bits = ref.diag_bits;
  DBuf<unsigned long long> counter(c, 3);
  a.counter = counter.p;
  a.stats = counter.p + 1;
  if (keys.n == 0) keys.alloc(c, std::max<uint64_t>(1 << 20, uint64_t(reads.n) * 16));
  const void* kfn = mode == 1 ? (const void*)k_join<true> : (const void*)k_join<false>;
  const size_t smem = size_t(4) * a.words * sizeof(uint32_t);
  QGM_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const unsigned grid = std::min<unsigned>(a.n_sub, resident_grid(kfn, kJoinThreads, smem));
  for (int attempt = 0; attempt < 2; ++attempt) {
    counter.zero();
    a.out = keys.p;
    a.cap = keys.n;
    if (rp.V > 0) {
      KernelScope ks(c, "k_join");
      if (mode == 1) QGM_KERNEL(c, k_join<true>, grid, kJoinThreads, smem, a);
      else QGM_KERNEL(c, k_join<false>, grid, kJoinThreads, smem, a);
    }
    unsigned long long h[3] = {0, 0, 0};
    QGM_CUDA(cudaMemcpyAsync(h, counter.p, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    QGM_CUDA(cudaStreamSynchronize(c.stream));
    if (fstats) {
      fstats[0] = h[1];
      fstats[1] = h[2];
    }
    if (h[0] <= keys.n) return h[0];
    keys.alloc(c, h[0] + h[0] / 8);
  }
  throw InternalError("join filtration: candidate buffer overflow after resize");
}

}  // namespace qgm
