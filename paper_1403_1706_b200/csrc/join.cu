// join.cu -- stage 2, production path: filtration as a bucket-ordered join.
//
// Same candidate semantics as filter.cu (Alg. 2; Appendix
// B.1-B.3): a forward candidate (r, +, p - o) for every reference position p
// whose q-gram equals the read q-gram at offset o, a reverse candidate
// (r, -, p + o + q - n) for every p whose reverse-complemented q-gram equals it.
//
// Why a join: streaming 2L reference q-grams against a 4^q-code read index
// makes every lookup a random 32-byte probe into a 512 MiB occupancy array
// (q=16); ncu shows each probe costing ~100 B of HBM traffic (profiles/
// r01_filter_stream.md). Here the reference side is a q-group index built once
// per reference and q (prepare_ref_index; the paper's reference index with P
// ordered by q-gram), one per strand, and the per-batch read
// q-grams are only bucket-sorted by code (bucket_reads). One CTA per code
// bucket (8192 codes) stages the bucket's 256 occupancy words and group
// starts of both reference strands in shared memory (coalesced), looks up the
// bucket's read q-grams there, and reads S'/O of the reference index in
// (nearly) increasing order. Every HBM stream is sequential.
//
// The run-start rule needs ref[p-1] (forward) or its complement (RC): stored
// per occurrence next to O (prev_fwd / prev_rc, 4 = no predecessor) so the
// check costs one byte read from the same, sequentially read, region.
#include "internal.hpp"

namespace qgm {
namespace {

constexpr int kJoinThreads = 256;
constexpr int kJoinWarps = kJoinThreads / 32;
constexpr int kStage = 512;
constexpr int kMaxGpb = 256;  // w = 32, 13 low bits per bucket

struct JoinArgs {
  const uint64_t* rpairs;
  const uint32_t* rboff;
  uint64_t buckets;
  uint32_t gpb;
  unsigned q;
  const uint32_t *If, *Sf, *S1f, *Of;
  const uint8_t* Xf;
  const uint32_t *Ir, *Sr, *S1r, *Or;
  const uint8_t* Xr;
  const uint64_t* rwords;
  const uint32_t* rlen;
  uint32_t W, m;
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

template <bool kRunStart>
__global__ void __launch_bounds__(kJoinThreads) k_join(JoinArgs a) {
  __shared__ uint32_t sIf[kMaxGpb], sSf[kMaxGpb], sIr[kMaxGpb], sSr[kMaxGpb];
  __shared__ uint32_t s_k0[kJoinWarps][64];
  __shared__ uint32_t s_pre[kJoinWarps][65];
  __shared__ uint32_t s_pos[kJoinWarps][64];  // read text position p' | strand << 31 kept apart:
  __shared__ uint8_t s_rev[kJoinWarps][64];
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

  for (uint64_t bk = blockIdx.x; bk < a.buckets; bk += gridDim.x) {
    const uint32_t b0 = __ldg(a.rboff + bk), b1 = __ldg(a.rboff + bk + 1);
    if (b0 == b1) continue;  // block-uniform: no read q-gram in this bucket
    for (uint32_t i = threadIdx.x; i < a.gpb; i += kJoinThreads) {
      const uint64_t gi = bk * a.gpb + i;
      if (a.strands & 1) { sIf[i] = __ldg(a.If + gi); sSf[i] = __ldg(a.Sf + gi); }
      if (a.strands & 2) { sIr[i] = __ldg(a.Ir + gi); sSr[i] = __ldg(a.Sr + gi); }
    }
    __syncthreads();
    const uint32_t rounds = (b1 - b0 + kJoinThreads - 1) / kJoinThreads;
    for (uint32_t rd = 0; rd < rounds; ++rd) {
      const uint32_t it = b0 + rd * kJoinThreads + wid * 32 + lane;
      uint32_t nr = 0, cnt = 0, rk0[2], rn[2];
      uint8_t rrev[2];
      uint32_t pos = 0;
      if (it < b1) {
        const uint64_t pr = __ldg(a.rpairs + it);
        const uint32_t gl = uint32_t(pr >> 32) & 8191u;
        pos = uint32_t(pr);
        const uint32_t wi = gl >> 5, bit = gl & 31;
        if (a.strands & 1) {
          const uint32_t w = sIf[wi];
          if ((w >> bit) & 1u) {
            const uint32_t b = sSf[wi] + __popc(w & ((1u << bit) - 1u));
            const uint32_t k0 = __ldg(a.S1f + b), k1 = __ldg(a.S1f + b + 1);
            rk0[nr] = k0; rn[nr] = k1 - k0; rrev[nr] = 0; cnt += k1 - k0; ++nr;
          }
        }
        if (a.strands & 2) {
          const uint32_t w = sIr[wi];
          if ((w >> bit) & 1u) {
            const uint32_t b = sSr[wi] + __popc(w & ((1u << bit) - 1u));
            const uint32_t k0 = __ldg(a.S1r + b), k1 = __ldg(a.S1r + b + 1);
            rk0[nr] = k0; rn[nr] = k1 - k0; rrev[nr] = 1; cnt += k1 - k0; ++nr;
          }
        }
      }
      n_hit += nr;
      n_occ += cnt;
      const uint32_t r_off = warp_inclusive_scan(nr) - nr;
      const uint32_t o_inc = warp_inclusive_scan(cnt);
      const uint32_t R = __shfl_sync(kFull, r_off + nr, 31);
      const uint32_t T = __shfl_sync(kFull, o_inc, 31);
      if (T == 0) continue;
      uint32_t run = o_inc - cnt;
      for (uint32_t i = 0; i < nr; ++i) {
        s_k0[wid][r_off + i] = rk0[i];
        s_pre[wid][r_off + i] = run;
        s_pos[wid][r_off + i] = pos;
        s_rev[wid][r_off + i] = rrev[i];
        run += rn[i];
      }
      if (lane == 0) s_pre[wid][R] = T;
      __syncwarp();
      for (uint32_t j0 = 0; j0 < T; j0 += 32) {
        const uint32_t j = j0 + lane;
        bool emit = false;
        uint64_t key = 0;
        if (j < T) {
          uint32_t lo = 0, hi = R;  // largest e with s_pre[e] <= j
          while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (s_pre[wid][mid] <= j) lo = mid; else hi = mid;
          }
          const bool rev = s_rev[wid][lo];
          const uint32_t k = s_k0[wid][lo] + (j - s_pre[wid][lo]);
          const uint32_t x = __ldg((rev ? a.Or : a.Of) + k);
          const uint32_t pp = s_pos[wid][lo];
          const uint32_t r = pp / a.m, o = pp - r * a.m;
          const uint64_t* rw = a.rwords + uint64_t(r) * a.W;
          emit = true;
          uint32_t c = 0, hi2 = a.n_chrom;  // chromosome of x
          while (hi2 - c > 1) {
            const uint32_t mid = (c + hi2) >> 1;
            if (__ldg(a.cb + mid) <= x) c = mid; else hi2 = mid;
          }
          const int64_t p = int64_t(x) - int64_t(__ldg(a.cb + c));
          int64_t d;
          if (!rev) {
            d = p - int64_t(o);
            if (kRunStart && o >= 1) {
              const uint32_t pv = __ldg(a.Xf + k);
              if (pv != 4 && pv == base_at(rw, o - 1)) emit = false;
            }
          } else {
            const uint32_t n = __ldg(a.rlen + r);
            d = p + int64_t(o) + int64_t(q) - int64_t(n);
            if (kRunStart && o + q + 1 <= n) {
              const uint32_t pv = __ldg(a.Xr + k);
              if (pv != 4 && pv == base_at(rw, o + q)) emit = false;
            }
          }
          const uint64_t gp = uint64_t(int64_t(__ldg(a.cbp + c)) + d);
          key = (uint64_t(r) << (a.diag_bits + 1)) | (uint64_t(rev) << a.diag_bits) | gp;
        }
        const unsigned m = __ballot_sync(kFull, emit);
        if (emit) s_out[wid][staged + __popc(m & lanemask_lt())] = key;
        staged += __popc(m);
        __syncwarp();
        if (staged > kStage - 32) flush();
      }
    }
    __syncthreads();  // shared words are reloaded for the next bucket
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

uint64_t join_filter(Ctx& c, const Buckets& rb, const Reads& reads, const Ref& ref, int strands, int mode,
                     unsigned read_bits, DBuf<uint64_t>& keys, uint64_t* fstats) {
  if (read_bits + 1 + ref.diag_bits > 64) throw InputError("read batch too large for the 64-bit candidate key");
  if (reads.max_len + 64 > ref.gap) throw InputError("reads longer than the reference padding supports");
  if (rb.w != 32 || rb.gpb > kMaxGpb) throw InternalError("join: read buckets must use 32-bit groups");
  prepare_ref_index(c, ref, rb.q);
  const RefQIndex& X = ref.qidx;
  JoinArgs a;
  a.rpairs = rb.pairs.p;
  a.rboff = rb.boff.p;
  a.buckets = rb.buckets;
  a.gpb = uint32_t(rb.gpb);
  a.q = rb.q;
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
  a.cb = ref.d_cb.p;
  a.cbp = ref.d_cbp.p;
  a.n_chrom = ref.n_chrom;
  a.strands = strands;
  a.diag_bits = ref.diag_bits;
  DBuf<unsigned long long> counter(c, 3);
  a.counter = counter.p;
  a.stats = counter.p + 1;
  if (keys.n == 0) keys.alloc(c, std::max<uint64_t>(1 << 20, uint64_t(reads.n) * 16));
  const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>(rb.buckets, uint64_t(kSMs) * 8)));
  for (int attempt = 0; attempt < 2; ++attempt) {
    counter.zero();
    a.out = keys.p;
    a.cap = keys.n;
    if (rb.V > 0) {
      KernelScope ks(c, "k_join");
      if (mode == 1) QGM_KERNEL(c, k_join<true>, grid, kJoinThreads, 0, a);
      else QGM_KERNEL(c, k_join<false>, grid, kJoinThreads, 0, a);
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
