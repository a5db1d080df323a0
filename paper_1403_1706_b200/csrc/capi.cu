// capi.cu -- the extern "C" boundary (include/qgm_c.h): context and object
// lifetime, host<->device staging, and the orchestration of the five stages
// for qgm_map. No exception crosses this file's exported functions.
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>

#include "../../include/qgm_c.h"
#include "internal.hpp"

struct qgm_ctx {
  qgm::Ctx c;
};
struct qgm_reads {
  qgm_ctx* owner;
  qgm::Reads r;
};
struct qgm_ref {
  qgm_ctx* owner;
  qgm::Ref r;
};
struct qgm_index {
  qgm_ctx* owner;
  qgm::Index i;
};
struct qgm_cands {
  qgm_ctx* owner;
  qgm::Cands c;
};
struct qgm_hits {
  qgm_ctx* owner;
  qgm::HitsObj h;
};

namespace qgm {

// ------------------------------------------------------------------ Ctx
cudaEvent_t Ctx::take_event() {
  if (!ev_pool.empty()) {
    cudaEvent_t e = ev_pool.back();
    ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  QGM_CUDA(cudaEventCreate(&e));
  return e;
}

void* Ctx::block_alloc(size_t bytes, size_t& cls) {
  cls = size_class(bytes);
  // best fit among cached blocks no larger than 1.5x the request's class
  size_t best = free_blocks.size();
  for (size_t i = 0; i < free_blocks.size(); ++i) {
    const size_t c = free_blocks[i].first;
    if (c >= cls && c <= cls + cls / 2 && (best == free_blocks.size() || c < free_blocks[best].first)) best = i;
  }
  if (best < free_blocks.size()) {
    void* p = free_blocks[best].second;
    cls = free_blocks[best].first;
    free_blocks[best] = free_blocks.back();
    free_blocks.pop_back();
    cached_bytes -= cls;
    live_bytes += cls;
    return p;
  }
  // no size cap: the cache is trimmed only when the pool is out of memory
  // (a cap made repeat-heavy batches -- tens of GB of cached candidate
  // buffers -- trim and synchronise on almost every allocation)
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, cls, stream);
  if (e == cudaErrorMemoryAllocation && !free_blocks.empty()) {
    cudaGetLastError();
    block_trim();  // give cached blocks of other sizes back, then retry once
    e = cudaMallocAsync(&p, cls, stream);
  }
  if (e != cudaSuccess)
    throw CudaError(std::string("device allocation of ") + std::to_string(cls) + " bytes failed: " +
                    cudaGetErrorString(e));
  live_bytes += cls;
  return p;
}

void Ctx::block_free(void* p, size_t cls) {
  free_blocks.push_back({cls, p});
  live_bytes -= cls;
  cached_bytes += cls;
}

void Ctx::block_trim() {
  for (auto& b : free_blocks) cudaFreeAsync(b.second, stream);
  free_blocks.clear();
  cached_bytes = 0;
  cudaStreamSynchronize(stream);
}

void Ctx::stage_begin(int s) {
  if (!profile || cur_stage >= 0) return;  // nested stages are folded into the outer one
  cur_stage = s;
  cur_host = std::chrono::steady_clock::now();
  cur_a = take_event();
  QGM_CUDA(cudaEventRecord(cur_a, stream));
}

void Ctx::stage_end() {
  if (!profile || cur_stage < 0) return;
  cudaEvent_t b = take_event();
  QGM_CUDA(cudaEventRecord(b, stream));
  marks.push_back({cur_stage, cur_a, b});
  host_ms[cur_stage] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - cur_host).count();
  cur_stage = -1;
  cur_a = nullptr;
}

void Ctx::fold_marks() {
  for (auto& m : marks) {
    QGM_CUDA(cudaEventSynchronize(m.b));
    float ms = 0;
    QGM_CUDA(cudaEventElapsedTime(&ms, m.a, m.b));
    stage_ms[m.stage] += ms;
    ev_pool.push_back(m.a);
    ev_pool.push_back(m.b);
  }
  marks.clear();
  for (auto& m : kmarks) {
    QGM_CUDA(cudaEventSynchronize(m.b));
    float ms = 0;
    QGM_CUDA(cudaEventElapsedTime(&ms, m.a, m.b));
    auto it = std::find_if(kernel_ms.begin(), kernel_ms.end(), [&](auto& e) { return e.first == m.name; });
    if (it == kernel_ms.end()) kernel_ms.push_back({m.name, {ms, 1}});
    else { it->second.first += ms; it->second.second += 1; }
    ev_pool.push_back(m.a);
    ev_pool.push_back(m.b);
  }
  kmarks.clear();
}

namespace {

// ------------------------------------------------------------------ planes
__device__ __forceinline__ uint32_t compress_even(uint64_t x) {  // bit 2i -> bit i
  x &= 0x5555555555555555ull;
  x = (x | (x >> 1)) & 0x3333333333333333ull;
  x = (x | (x >> 2)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x >> 4)) & 0x00FF00FF00FF00FFull;
  x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
  x = (x | (x >> 16)) & 0x00000000FFFFFFFFull;
  return uint32_t(x);
}

// 2-bit word (32 bases, MSB-first) -> {lo bits, hi bits}, bit 31-j = base j.
__device__ __forceinline__ uint2 to_planes(uint64_t w) { return make_uint2(compress_even(w), compress_even(w >> 1)); }

__global__ void k_read_planes(const uint64_t* __restrict__ words, uint32_t n_reads, uint32_t W, uint32_t Wp,
                              uint2* __restrict__ planes) {
  QGM_GRID_DEP();
  const uint64_t total = uint64_t(n_reads) * Wp;
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < total; t += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = t / Wp;
    const uint32_t c = uint32_t(t - r * Wp);
    planes[t] = (c >= 1 && c <= W) ? to_planes(words[r * W + c - 1]) : make_uint2(0u, 0u);
  }
}

// dense 2-bit stream (read r = bases [r*stride, (r+1)*stride)) -> W words per read
__global__ void k_unpack_dense(const uint64_t* __restrict__ dense, uint32_t n_reads, uint32_t stride, uint32_t W,
                               uint64_t* __restrict__ words) {
  QGM_GRID_DEP();
  const uint64_t total = uint64_t(n_reads) * W;
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < total; t += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = t / W;
    const uint32_t k = uint32_t(t - r * W);
    const uint64_t b0 = r * stride + 32ull * k;  // first base of this word in the stream
    const uint64_t i = b0 >> 5;
    const unsigned sh = unsigned(b0 & 31) * 2;
    uint64_t w = __ldg(dense + i) << sh;
    if (sh) w |= __ldg(dense + i + 1) >> (64 - sh);
    const uint32_t nb = min(32u, stride - 32 * k);  // bases of this read in the word
    if (nb < 32) w &= ~(~0ull >> (2 * nb));         // zero padding past the read
    words[t] = w;
  }
}

__global__ void k_fill_u32(uint32_t* __restrict__ p, uint64_t n, uint32_t v) {
  QGM_GRID_DEP();
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < n; t += uint64_t(gridDim.x) * blockDim.x) p[t] = v;
}

__global__ void k_ref_planes(const uint64_t* __restrict__ words, uint64_t nw, uint2* __restrict__ planes) {
  QGM_GRID_DEP();
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < nw; k += uint64_t(gridDim.x) * blockDim.x)
    planes[k + 2] = to_planes(words[k]);
}

// out[0] = max, out[1] = ~min (both folded with atomicMax; out zeroed)
__global__ void k_minmax_u32(const uint32_t* __restrict__ v, uint64_t n, uint32_t* __restrict__ out) {
  QGM_GRID_DEP();
  uint32_t m = 0, nm = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    m = max(m, v[i]);
    nm = max(nm, ~v[i]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    m = max(m, __shfl_xor_sync(kFull, m, o));
    nm = max(nm, __shfl_xor_sync(kFull, nm, o));
  }
  // one atomic pair per CTA (per warp, ~5k same-address atomics cost ~10 us
  // for a 1M-read batch)
  __shared__ uint32_t s_m[32], s_nm[32];
  const unsigned wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane_id() == 0) {
    s_m[wid] = m;
    s_nm[wid] = nm;
  }
  __syncthreads();
  if (wid == 0) {
    m = lane_id() < nw ? s_m[lane_id()] : 0u;
    nm = lane_id() < nw ? s_nm[lane_id()] : 0u;
    for (int o = 16; o > 0; o >>= 1) {
      m = max(m, __shfl_xor_sync(kFull, m, o));
      nm = max(nm, __shfl_xor_sync(kFull, nm, o));
    }
    if (lane_id() == 0) {
      atomicMax(out, m);
      atomicMax(out + 1, nm);
    }
  }
}

unsigned read_bits_for(uint32_t n_reads) { return std::max(1u, bit_width_u64(n_reads ? n_reads - 1 : 0)); }

}  // namespace

void make_read_planes(Ctx& c, Reads& r) {
  r.Wp = r.W + 2;
  r.planes.alloc(c, std::max<uint64_t>(uint64_t(r.n) * r.Wp, 1));
  const uint64_t total = uint64_t(r.n) * r.Wp;
  if (!total) return;
  // on the side stream, after everything the compute stream has queued (the
  // words, and any earlier user of the planes block); consumers wait on
  // planes_ev (Ctx::wait_planes)
  if (!c.side_stream) {
    QGM_CUDA(cudaStreamCreateWithFlags(&c.side_stream, cudaStreamNonBlocking));
    QGM_CUDA(cudaEventCreateWithFlags(&c.side_ev, cudaEventDisableTiming));
    QGM_CUDA(cudaEventCreateWithFlags(&c.planes_ev, cudaEventDisableTiming));
  }
  QGM_CUDA(cudaEventRecord(c.side_ev, c.stream));
  QGM_CUDA(cudaStreamWaitEvent(c.side_stream, c.side_ev, 0));
  k_read_planes<<<unsigned(std::min<uint64_t>(ceil_div(total, 256), kSMs * 16)), 256, 0, c.side_stream>>>(
      r.words.p, r.n, r.W, r.Wp, r.planes.p);
  ++c.launches;
  QGM_LAUNCH_CHECK();
  QGM_CUDA(cudaEventRecord(c.planes_ev, c.side_stream));
}

void make_ref_planes(Ctx& c, Ref& ref) {
  const uint64_t nw = ceil_div(ref.total, 32);
  ref.planes.alloc(c, nw + 4);
  ref.planes.zero();
  if (nw)
    QGM_KERNEL(c, k_ref_planes, unsigned(std::min<uint64_t>(ceil_div(nw, 256), kSMs * 16)), 256, 0, ref.words.p, nw,
               ref.planes.p);
}

// ------------------------------------------------------------------ pipeline
static void finish_reads(Ctx& c, Reads& r) {
  make_read_planes(c, r);
  r.lens.alloc(c, 2);
  r.lens.zero();
  if (r.n)
    QGM_KERNEL(c, k_minmax_u32, unsigned(std::min<uint64_t>(ceil_div(r.n, 256), kSMs * 4)), 256, 0, r.lengths.p,
               uint64_t(r.n), r.lens.p);
}

static void check_reads_shape(uint32_t n_reads, uint32_t stride) {
  if (uint64_t(n_reads) * stride > 0xFFFFFFFFull) throw InputError("read text exceeds 2^32 positions");
  if (n_reads > (1u << 27)) throw InputError("at most 2^27 reads per batch");
}

// after_filter: called (host side) once the candidate dedup is enqueued --
// qgm_map_host_batches enqueues its copies there, so they overlap the
// compute-bound validation (and the strata) rather than the L2-sensitive
// partition and join (QGM_HOOK=0/1/2: after the join / the dedup / the
// validation, measured within noise of each other).
constexpr uint64_t kDedupDirectMax = uint64_t(10) << 20;  // raw keys whose hash table (<= 16M slots) stays L2-resident

static int hook_point() {  // experiment knob: 0 after the join, 1 after dedup, 2 after validation, 3 first
  static const int h = [] {
    const char* e = std::getenv("QGM_HOOK");
    return e ? std::atoi(e) : 1;
  }();
  return h;
}

static uint64_t dedup_direct_max() {
  const char* e = std::getenv("QGM_DEDUP_DIRECT_MAX");  // tests
  if (e && e[0]) return std::strtoull(e, nullptr, 10);
  return kDedupDirectMax;
}

// The batch without a host round trip before its end: partition, join,
// dedup, validation and strata all sized by the candidate-buffer capacity
// (the larger of 16 per read and 1.125x the context's last count) and run on
// the device counts; one read-back at the end returns every count. Taken
// when that capacity is within the always-deduplicated range, so no decision
// needs the count on the host. Returns false when the join's count exceeded
// the capacity (keys truncated): the caller maps the batch again with the
// round-trip path, which sizes the buffer from the count.
static bool map_reads_async(Ctx& c, const Reads& reads, const Ref& ref, const qgm_map_params& P, int strands,
                            unsigned rb, uint64_t cap, const std::function<void()>& after_filter, HitsObj& out) {
  prepare_ref_index(c, ref, P.q);
  if (after_filter && hook_point() == 3) after_filter();
  Partitioned rbk;
  {
    StageScope s(c, kStageIndex);
    partition_reads(c, reads, P.q, rbk);
  }
  DBuf<uint64_t> keys(c, cap), alt;
  DBuf<unsigned long long> jc(c, 3);  // candidates, lookups that hit, occurrences
  {
    StageScope s(c, kStageFilter);
    join_filter(c, rbk, reads, ref, strands, QGM_FILTER_RUN_START, rb, keys, nullptr, jc.p);
  }
  if (after_filter && hook_point() == 0) after_filter();
  DBuf<unsigned long long> cnt(c, 3);  // validated hits, unique candidates, reads with > 32 hits
  cnt.zero();
  {
    StageScope s(c, kStageSort);
    dedup_keys_dev(c, keys.p, cap, jc.p, alt, cnt.p + 1);
  }
  if (after_filter && hook_point() == 1) after_filter();
  DBuf<uint64_t> hkeys(c, cap);
  DBuf<uint32_t> hvals(c, cap);
  DBuf<uint32_t> per_read(c, uint64_t(reads.n) + 1), kept_total(c, 1);  // hits per read, counted by validation
  per_read.zero();
  {
    StageScope s(c, kStageValidate);
    validate_candidates(c, reads, ref, alt.p, cap, rb, P.band_width, P.pct_identity, 0, hkeys.p, hvals.p, cnt.p,
                        nullptr, cnt.p + 1, P.q, per_read.p, cnt.p + 2);
  }
  if (after_filter && hook_point() == 2) after_filter();
  unsigned long long jh[3] = {0, 0, 0}, h[3] = {0, 0, 0};
  uint32_t fl[4] = {0, 0, 0, 0}, kept = 0;
  {
    StageScope s(c, kStageStrata);
    stratify_unsorted_dev(c, ref, hkeys.p, hvals.p, cnt.p, cap, reads.n, int(P.mode), per_read, cnt.p + 2, out.hits,
                          kept_total.p);
    // the batch's one host round trip
    read_back(c, {{jc.p, jh, sizeof(jh)}, {rbk.flags.p, fl, sizeof(fl)}, {cnt.p, h, sizeof(h)},
                  {kept_total.p, &kept, 4}});
  }
  if (fl[2]) throw InputError("read longer than the stride");
  c.last_raw_candidates = jh[0];
  if (jh[0] > cap) return false;
  const uint64_t n_val = h[0];
  out.n = kept;
  if (h[2] != 0) {  // a read with > 32 hits: the radix-sorted strata on the known count
    StageScope s(c, kStageStrata);
    out.n = stratify_unsorted(c, ref, hkeys, hvals, n_val, reads.n, int(P.mode), per_read, true, out.hits);
  }
  out.n_reads = reads.n;
  out.stats[0] = jh[0];
  out.stats[1] = h[1];
  out.stats[2] = n_val;
  out.stats[3] = out.n;
  out.stats[5] = fl[0];
  out.stats[6] = jh[1];
  out.stats[7] = jh[2];
  return true;
}

static HitsObj map_reads(Ctx& c, const Reads& reads, const Ref& ref, const qgm_map_params& P,
                         const std::function<void()>& after_filter_once = {}) {
  bool hooked = false;  // the hook runs once even when the batch is mapped twice
  const std::function<void()> after_filter = [&] {
    if (after_filter_once && !hooked) {
      hooked = true;
      after_filter_once();
    }
  };
  if (P.q == 0 || P.q > 16) throw InputError("q must be in [1, 16]");
  if (P.band_width == 0 || P.band_width > 64) throw InputError("band width must be in [1, 64]");
  if (P.pct_identity > 100) throw InputError("percent identity must be in [0, 100]");
  if (P.mode > 1) throw InputError("mode must be best-stratum (0) or all (1)");
  const int strands = P.strands ? int(P.strands) : 3;
  if (P.group_width && P.group_width != 32 && P.group_width != 64) throw InputError("group width must be 32 or 64");
  if (ref.padded_total < (uint64_t(1) << 32)) {
    // candidate capacity: 1.25x the context's last batch once there is one
    // (a larger count re-maps the batch through the round-trip path), else
    // 16 per read
    uint64_t cap = c.last_raw_candidates ? c.last_raw_candidates + c.last_raw_candidates / 4
                                         : uint64_t(reads.n) * 16;
    cap = std::max<uint64_t>(cap, 1 << 20);
    const char* ce = std::getenv("QGM_MAP_ASYNC_CAP");  // tests
    if (ce && ce[0]) cap = std::max<uint64_t>(1, std::strtoull(ce, nullptr, 10));
    const char* ae = std::getenv("QGM_MAP_ASYNC");  // A/B and test knob: 0 = always the round-trip path
    const bool async_off = ae && ae[0] == '0';
    if (!async_off && cap <= dedup_direct_max()) {
      HitsObj out;
      if (map_reads_async(c, reads, ref, P, strands, read_bits_for(reads.n), cap, after_filter, out)) return out;
      // truncated candidate set: map again below (the hook has run)
    }
  }
  const unsigned rb = read_bits_for(reads.n);
  HitsObj out;
  DBuf<uint64_t> keys, alt;
  uint64_t n_raw, n_u;
  uint64_t fst[3] = {0, 0, 0};
  if (ref.padded_total < (uint64_t(1) << 32)) {
    // production path: read q-grams bucket-sorted by code, joined with the
    // per-strand reference q-group indexes (join.cu). group_width / sampled
    // only change the layout of an index that is never materialised here.
    prepare_ref_index(c, ref, P.q);  // once per reference and q (cached)
    Partitioned rbk;
    {
      StageScope s(c, kStageIndex);
      partition_reads(c, reads, P.q, rbk);
    }
    {
      StageScope s(c, kStageFilter);
      n_raw = join_filter(c, rbk, reads, ref, strands, QGM_FILTER_RUN_START, rb, keys, fst);
    }
    out.stats[5] = fst[2];  // exact read q-gram count, read back with the candidate count
  } else {
    // references beyond 2^32 bases: stream the reference against the read index (filter.cu)
    Index idx;
    {
      StageScope s(c, kStageIndex);
      build_index(c, reads, P.q, P.group_width ? P.group_width : 32, P.sampled != 0, idx);
    }
    out.stats[4] = idx.distinct;
    out.stats[5] = idx.occ;
    StageScope s(c, kStageFilter);
    n_raw = filter_reference(c, idx, reads, ref, strands, QGM_FILTER_RUN_START, rb, keys, fst);
  }
  out.stats[6] = fst[0];
  out.stats[7] = fst[1];
  const int hook_at = hook_point();
  if (after_filter && hook_at == 0) after_filter();
  // cnt[0]: validated hits, cnt[1]: unique candidates, cnt[2]: reads with
  // more than 32 hits -- read back together after validation (no host round
  // trip between dedup, validation and the strata's per-read counts)
  DBuf<unsigned long long> cnt(c, 3);
  cnt.zero();
  // Candidate dedup only pays when the set has duplicates to remove: above
  // ~10M keys the hash table leaves L2 (C3: 7.6 ms of atomics in DRAM for 1%
  // duplicates), so a large set is first sampled and deduplicated only if
  // more than 10% of it repeats. Skipping it cannot change a hit: validation
  // is a pure function of the key and the strata keep one hit per (read,
  // chromosome, start, strand). unique_candidates then reports the raw count.
  bool dedup = true;
  if (n_raw > dedup_direct_max()) {
    StageScope s(c, kStageSort);
    dedup = estimate_dup_fraction(c, keys.p, n_raw, ref.diag_bits + 1) > 0.10;
  }
  {
    StageScope s(c, kStageSort);
    if (dedup && (n_raw <= dedup_direct_max() || n_raw > 0xFFFFFFFFull)) {  // radix pass offsets are u32
      dedup_keys_async(c, keys.p, n_raw, alt, cnt.p + 1);  // unique candidates, any order (validation is per key)
    } else if (dedup) {
      // one table for all keys would leave L2 (C5: 752M keys, a 16 GB table,
      // 48 ms of random DRAM read-modify-writes): partitioned on 8 key bits,
      // each partition's table stays L2-resident
      dedup_keys_partitioned(c, keys.p, n_raw, alt, cnt.p + 1);
    } else {
      alt.swap(keys);
      const unsigned long long nr = n_raw;
      QGM_CUDA(cudaMemcpyAsync(cnt.p + 1, &nr, sizeof(nr), cudaMemcpyHostToDevice, c.stream));
    }
  }
  if (after_filter && hook_at == 1) after_filter();
  const uint64_t n_bound = std::max<uint64_t>(n_raw, 1);
  DBuf<uint64_t> hkeys(c, n_bound), hkeys_alt;
  DBuf<uint32_t> hvals(c, n_bound), hvals_alt;
  uint64_t n_val = 0;
  DBuf<uint32_t> per_read(c, uint64_t(reads.n) + 1);  // hits per read, counted by validation
  per_read.zero();
  {
    StageScope s(c, kStageValidate);
    validate_candidates(c, reads, ref, alt.p, n_raw, rb, P.band_width, P.pct_identity, 0, hkeys.p, hvals.p, cnt.p,
                        nullptr, cnt.p + 1, P.q, per_read.p, cnt.p + 2);
  }
  if (after_filter && hook_at == 2) after_filter();
  bool big = false, speculative_done = false;
  {
    StageScope s(c, kStageStrata);
    // The per-read counting-sort strata run on the device counts (output sized
    // for n_raw records) so that one read-back after them returns every count;
    // a batch with a read of > 32 hits (repeats) then takes the radix path.
    // Above 1 GiB of bound-sized output the counts are read back first.
    const bool speculative = n_bound <= (uint64_t(1) << 26);
    DBuf<uint32_t> kept_total(c, 1);
    if (speculative)
      stratify_unsorted_dev(c, ref, hkeys.p, hvals.p, cnt.p, n_bound, reads.n, int(P.mode), per_read, cnt.p + 2,
                            out.hits, kept_total.p);
    unsigned long long h[3] = {0, 0, 0};
    uint32_t kept = 0;
    if (speculative)
      read_back(c, {{cnt.p, h, sizeof(h)}, {kept_total.p, &kept, 4}});
    else
      read_back(c, {{cnt.p, h, sizeof(h)}});
    n_val = h[0];
    n_u = h[1];
    big = h[2] != 0;
    if (speculative && !big) {
      out.n = kept;
      speculative_done = true;
    }
  }
  keys.release();
  alt.release();
  if (!speculative_done) {
    StageScope s(c, kStageStrata);
    out.n = stratify_unsorted(c, ref, hkeys, hvals, n_val, reads.n, int(P.mode), per_read, big, out.hits);
  }
  out.n_reads = reads.n;
  out.stats[0] = n_raw;
  out.stats[1] = n_u;
  out.stats[2] = n_val;
  out.stats[3] = out.n;
  return out;
}

}  // namespace qgm

// ===================================================================== C ABI
namespace {

template <class Fn>
int guard(qgm_ctx* ctx, Fn&& fn) {
  try {
    fn();
    return QGM_OK;
  } catch (const qgm::InputError& e) {
    if (ctx) ctx->c.err = e.what();
    return QGM_ERR_INPUT;
  } catch (const qgm::InternalError& e) {
    if (ctx) ctx->c.err = e.what();
    return QGM_ERR_INTERNAL;
  } catch (const qgm::CudaError& e) {
    if (ctx) ctx->c.err = e.what();
    return QGM_ERR_CUDA;
  } catch (const std::bad_alloc& e) {
    if (ctx) ctx->c.err = std::string("host allocation failed: ") + e.what();
    return QGM_ERR_INTERNAL;
  } catch (const std::exception& e) {
    if (ctx) ctx->c.err = e.what();
    return QGM_ERR_INTERNAL;
  }
}

void require(bool ok, const char* what) {
  if (!ok) throw qgm::InputError(what);
}

void activate(qgm_ctx* ctx) { QGM_CUDA(cudaSetDevice(ctx->c.device)); }

}  // namespace

extern "C" {

int qgm_ctx_create(int device, qgm_ctx** out) {
  if (!out) return QGM_ERR_INPUT;
  *out = nullptr;
  auto ctx = std::make_unique<qgm_ctx>();
  int rc = guard(ctx.get(), [&] {
    int n = 0;
    QGM_CUDA(cudaGetDeviceCount(&n));
    require(device >= 0 && device < n, "no such CUDA device");
    ctx->c.device = device;
    QGM_CUDA(cudaSetDevice(device));
    QGM_CUDA(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
    ctx->c.own_stream = true;
    cudaMemPool_t pool;
    QGM_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = ~uint64_t(0);
    QGM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  });
  if (rc == QGM_OK) *out = ctx.release();
  return rc;
}

int qgm_ctx_set_stream(qgm_ctx* ctx, void* stream) {
  if (!ctx) return QGM_ERR_INPUT;
  return guard(ctx, [&] {
    activate(ctx);
    QGM_CUDA(cudaStreamSynchronize(ctx->c.stream));
    if (stream) {
      if (ctx->c.own_stream) QGM_CUDA(cudaStreamDestroy(ctx->c.stream));
      ctx->c.stream = static_cast<cudaStream_t>(stream);
      ctx->c.own_stream = false;
    } else if (!ctx->c.own_stream) {
      QGM_CUDA(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
      ctx->c.own_stream = true;
    }
  });
}

void* qgm_ctx_stream(qgm_ctx* ctx) { return ctx ? ctx->c.stream : nullptr; }

void qgm_ctx_destroy(qgm_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->c.device);
  cudaStreamSynchronize(ctx->c.stream);
  ctx->c.block_trim();
  if (ctx->c.tail_h) cudaFreeHost(ctx->c.tail_h);
  for (auto& m : ctx->c.marks) { cudaEventDestroy(m.a); cudaEventDestroy(m.b); }
  for (auto e : ctx->c.ev_pool) cudaEventDestroy(e);
  if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.stream);
  if (ctx->c.copy_stream) cudaStreamDestroy(ctx->c.copy_stream);
  if (ctx->c.d2h_stream) cudaStreamDestroy(ctx->c.d2h_stream);
  if (ctx->c.side_stream) {
    cudaStreamSynchronize(ctx->c.side_stream);
    cudaStreamDestroy(ctx->c.side_stream);
    cudaEventDestroy(ctx->c.side_ev);
    cudaEventDestroy(ctx->c.planes_ev);
  }
  delete ctx;
}

const char* qgm_last_error(const qgm_ctx* ctx) { return ctx ? ctx->c.err.c_str() : "null context"; }

int qgm_ctx_synchronize(qgm_ctx* ctx) {
  if (!ctx) return QGM_ERR_INPUT;
  return guard(ctx, [&] { QGM_CUDA(cudaStreamSynchronize(ctx->c.stream)); });
}

int qgm_ctx_profile(qgm_ctx* ctx, int enable) {
  if (!ctx) return QGM_ERR_INPUT;
  ctx->c.profile = enable != 0;
  return QGM_OK;
}

int qgm_ctx_stage_times(qgm_ctx* ctx, double* ms, int n, int reset) {
  if (!ctx) return QGM_ERR_INPUT;
  return guard(ctx, [&] {
    ctx->c.fold_marks();
    for (int i = 0; i < n && i < qgm::kNumStages; ++i) ms[i] = ctx->c.stage_ms[i];
    for (int i = qgm::kNumStages; i < n && i < 2 * qgm::kNumStages; ++i) ms[i] = ctx->c.host_ms[i - qgm::kNumStages];
    if (reset) {
      for (double& v : ctx->c.stage_ms) v = 0;
      for (double& v : ctx->c.host_ms) v = 0;
    }
  });
}

int qgm_ctx_kernel_times(qgm_ctx* ctx, char* buf, uint64_t cap, int reset) {
  if (!ctx || (!buf && cap)) return QGM_ERR_INPUT;
  return guard(ctx, [&] {
    ctx->c.fold_marks();
    std::string s;
    for (auto& e : ctx->c.kernel_ms)
      s += e.first + "\t" + std::to_string(e.second.first) + "\t" + std::to_string(e.second.second) + "\n";
    if (cap) {
      const size_t n = std::min<size_t>(s.size(), cap - 1);
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
    if (reset) ctx->c.kernel_ms.clear();
  });
}

uint64_t qgm_ctx_launches(qgm_ctx* ctx, int reset) {
  if (!ctx) return 0;
  const uint64_t n = ctx->c.launches;
  if (reset) ctx->c.launches = 0;
  return n;
}

int qgm_pack_codes(const uint8_t* codes, uint64_t n, uint64_t* words) {
  if ((!codes && n) || (!words && n)) return QGM_ERR_INPUT;
  const uint64_t nw = (n + 31) / 32;
  for (uint64_t k = 0; k < nw; ++k) {
    uint64_t w = 0;
    const uint64_t b = k * 32, e = std::min<uint64_t>(n, b + 32);
    for (uint64_t j = b; j < e; ++j) {
      if (codes[j] > 3) return QGM_ERR_INPUT;
      w |= uint64_t(codes[j]) << (62 - 2 * (j - b));
    }
    words[k] = w;
  }
  return QGM_OK;
}

int qgm_pack_reads(const uint8_t* codes, uint32_t stride, uint32_t n_reads, uint64_t* words) {
  const uint32_t W = (stride + 31) / 32;
  for (uint32_t r = 0; r < n_reads; ++r) {
    int rc = qgm_pack_codes(codes + uint64_t(r) * stride, stride, words + uint64_t(r) * W);
    if (rc) return rc;
  }
  return QGM_OK;
}

static int reads_common(qgm_ctx* ctx, const uint64_t* w, const uint32_t* len, uint32_t n_reads, uint32_t stride,
                        qgm_reads** out, cudaMemcpyKind kind) {
  if (!ctx || !out) return QGM_ERR_INPUT;
  *out = nullptr;
  auto rd = std::make_unique<qgm_reads>();
  rd->owner = ctx;
  int rc = guard(ctx, [&] {
    activate(ctx);
    qgm::Ctx& c = ctx->c;
    qgm::check_reads_shape(n_reads, stride);
    require(n_reads == 0 || (w && len), "null read buffers");
    qgm::StageScope s(c, qgm::kStageReads);
    auto& r = rd->r;
    r.n = n_reads;
    r.stride = stride;
    r.W = (stride + 31) / 32;
    const uint64_t nw = uint64_t(n_reads) * r.W;
    r.words.alloc(c, nw + 2);  // 2 guard words: the partition bulk-copies whole 16-byte pairs
    r.lengths.alloc(c, std::max<uint32_t>(n_reads, 1));
    if (nw) QGM_CUDA(cudaMemcpyAsync(r.words.p, w, nw * 8, kind, c.stream));
    fill_bytes(c, r.words.p + nw, 0, 16);
    if (n_reads) QGM_CUDA(cudaMemcpyAsync(r.lengths.p, len, uint64_t(n_reads) * 4, kind, c.stream));
    qgm::finish_reads(c, r);
  });
  if (rc == QGM_OK) *out = rd.release();
  return rc;
}

int qgm_reads_upload(qgm_ctx* ctx, const uint64_t* w, const uint32_t* len, uint32_t n_reads, uint32_t stride,
                     qgm_reads** out) {
  return reads_common(ctx, w, len, n_reads, stride, out, cudaMemcpyHostToDevice);
}

int qgm_reads_from_device(qgm_ctx* ctx, const uint64_t* w, const uint32_t* len, uint32_t n_reads, uint32_t stride,
                          qgm_reads** out) {
  return reads_common(ctx, w, len, n_reads, stride, out, cudaMemcpyDeviceToDevice);
}

void qgm_reads_destroy(qgm_reads* r) {
  if (!r) return;
  cudaSetDevice(r->owner->c.device);
  r->owner->c.wait_planes();  // the planes block goes back to the stream-ordered cache
  delete r;
}

int qgm_index_build(qgm_ctx* ctx, const qgm_reads* reads, uint32_t q, uint32_t w, int sampled, qgm_index** out) {
  if (!ctx || !reads || !out) return QGM_ERR_INPUT;
  *out = nullptr;
  auto ix = std::make_unique<qgm_index>();
  ix->owner = ctx;
  int rc = guard(ctx, [&] {
    activate(ctx);
    qgm::StageScope s(ctx->c, qgm::kStageIndex);
    qgm::build_index(ctx->c, reads->r, q, w, sampled != 0, ix->i);
  });
  if (rc == QGM_OK) *out = ix.release();
  return rc;
}

int qgm_index_sample(qgm_ctx* ctx, const qgm_index* in, qgm_index** out) {
  if (!ctx || !in || !out) return QGM_ERR_INPUT;
  *out = nullptr;
  auto ix = std::make_unique<qgm_index>();
  ix->owner = ctx;
  int rc = guard(ctx, [&] {
    activate(ctx);
    qgm::sample_index(ctx->c, in->i, ix->i);
  });
  if (rc == QGM_OK) *out = ix.release();
  return rc;
}

int qgm_index_normalize(qgm_ctx* ctx, qgm_index* idx) {
  if (!ctx || !idx) return QGM_ERR_INPUT;
  return guard(ctx, [&] {
    activate(ctx);
    qgm::normalize_index(ctx->c, idx->i);
  });
}

int qgm_index_info_get(const qgm_index* idx, qgm_index_info* o) {
  if (!idx || !o) return QGM_ERR_INPUT;
  const auto& i = idx->i;
  o->q = i.q;
  o->group_width = i.w;
  o->sampled = i.sampled;
  o->reserved = 0;
  o->group_count = i.groups;
  o->group_starts_len = i.gs_len;
  o->distinct = i.distinct;
  o->occurrences = i.occ;
  return QGM_OK;
}

int qgm_index_download(qgm_ctx* ctx, const qgm_index* idx, void* I, uint32_t* S, uint32_t* S1, uint32_t* O) {
  if (!ctx || !idx) return QGM_ERR_INPUT;
  return guard(ctx, [&] {
    activate(ctx);
    const auto& i = idx->i;
    cudaStream_t st = ctx->c.stream;
    if (I && i.groups) QGM_CUDA(cudaMemcpyAsync(I, i.I.p, i.groups * (i.w / 8), cudaMemcpyDeviceToHost, st));
    if (S) QGM_CUDA(cudaMemcpyAsync(S, i.S.p, i.gs_len * 4, cudaMemcpyDeviceToHost, st));
    if (S1) QGM_CUDA(cudaMemcpyAsync(S1, i.S1.p, (i.distinct + 1) * 4, cudaMemcpyDeviceToHost, st));
    if (O && i.occ) QGM_CUDA(cudaMemcpyAsync(O, i.O.p, i.occ * 4, cudaMemcpyDeviceToHost, st));
    QGM_CUDA(cudaStreamSynchronize(st));
  });
}

int qgm_index_lookup(qgm_ctx* ctx, const qgm_index* idx, const uint32_t* codes, uint64_t n, uint32_t* begin,
                     uint32_t* end) {
  if (!ctx || !idx) return QGM_ERR_INPUT;
  return guard(ctx, [&] {
    activate(ctx);
    qgm::Ctx& c = ctx->c;
    const uint64_t space = uint64_t(1) << (2 * idx->i.q);
    for (uint64_t t = 0; t < n; ++t) require(codes[t] < space, "q-gram code out of range");
    qgm::DBuf<uint32_t> dc(c, std::max<uint64_t>(n, 1)), db(c, std::max<uint64_t>(n, 1)),
        de(c, std::max<uint64_t>(n, 1));
    if (n) QGM_CUDA(cudaMemcpyAsync(dc.p, codes, n * 4, cudaMemcpyHostToDevice, c.stream));
    qgm::lookup_index(c, idx->i, dc.p, n, db.p, de.p);
    if (n) {
      QGM_CUDA(cudaMemcpyAsync(begin, db.p, n * 4, cudaMemcpyDeviceToHost, c.stream));
      QGM_CUDA(cudaMemcpyAsync(end, de.p, n * 4, cudaMemcpyDeviceToHost, c.stream));
    }
    QGM_CUDA(cudaStreamSynchronize(c.stream));
  });
}

void qgm_index_destroy(qgm_index* idx) {
  if (!idx) return;
  cudaSetDevice(idx->owner->c.device);
  delete idx;
}

int qgm_ref_upload(qgm_ctx* ctx, const uint64_t* ref2bit, const uint64_t* chrom_begin, uint32_t n_chrom,
                   const uint64_t* mask_bits, qgm_ref** out) {
  if (!ctx || !out) return QGM_ERR_INPUT;
  *out = nullptr;
  auto rf = std::make_unique<qgm_ref>();
  rf->owner = ctx;
  int rc = guard(ctx, [&] {
    activate(ctx);
    qgm::Ctx& c = ctx->c;
    require(n_chrom >= 1 && chrom_begin, "need at least one chromosome");
    require(chrom_begin[0] == 0, "chrom_begin[0] must be 0");
    for (uint32_t k = 0; k < n_chrom; ++k) {
      require(chrom_begin[k + 1] >= chrom_begin[k], "chrom_begin must be non-decreasing");
      require(chrom_begin[k + 1] - chrom_begin[k] < 0xFFFFFFFFull, "chromosome longer than 2^32-1 bases");
    }
    auto& r = rf->r;
    r.n_chrom = n_chrom;
    r.total = chrom_begin[n_chrom];
    require(r.total == 0 || ref2bit, "null reference buffer");
    r.gap = uint64_t(1) << 16;
    r.cb.assign(chrom_begin, chrom_begin + n_chrom + 1);
    r.cbp.resize(n_chrom + 1);
    for (uint32_t k = 0; k <= n_chrom; ++k) r.cbp[k] = r.cb[k] + uint64_t(k + 1) * r.gap;
    r.padded_total = r.total + uint64_t(n_chrom + 1) * r.gap;
    r.diag_bits = qgm::bit_width_u64(r.padded_total);
    require(r.diag_bits <= 40, "reference too large");
    const uint64_t nw = qgm::ceil_div(r.total, 32);
    r.words.alloc(c, nw + 1);
    if (nw) QGM_CUDA(cudaMemcpyAsync(r.words.p, ref2bit, nw * 8, cudaMemcpyDefault, c.stream));  // host or device
    fill_bytes(c, r.words.p + nw, 0, 8);
    r.d_cb.alloc(c, n_chrom + 1);
    r.d_cbp.alloc(c, n_chrom + 1);
    QGM_CUDA(cudaMemcpyAsync(r.d_cb.p, r.cb.data(), (n_chrom + 1) * 8, cudaMemcpyHostToDevice, c.stream));
    QGM_CUDA(cudaMemcpyAsync(r.d_cbp.p, r.cbp.data(), (n_chrom + 1) * 8, cudaMemcpyHostToDevice, c.stream));
    if (mask_bits) {
      const uint64_t mw = qgm::ceil_div(r.total, 64);
      r.mask.alloc(c, std::max<uint64_t>(mw, 1));
      if (mw) QGM_CUDA(cudaMemcpyAsync(r.mask.p, mask_bits, mw * 8, cudaMemcpyDefault, c.stream));
    }
    qgm::make_ref_planes(c, r);
    QGM_CUDA(cudaStreamSynchronize(c.stream));
  });
  if (rc == QGM_OK) *out = rf.release();
  return rc;
}

int qgm_ref_prepare(qgm_ctx* ctx, qgm_ref* ref, uint32_t q) {
  if (!ctx || !ref) return QGM_ERR_INPUT;
  return guard(ctx, [&] {
    activate(ctx);
    require(q >= 1 && q <= 16, "q must be in [1, 16]");
    require(ref->r.padded_total < (uint64_t(1) << 32), "reference index: more than 2^32-1 padded bases");
    qgm::prepare_ref_index(ctx->c, ref->r, q);
    QGM_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int qgm_ref_mask_repeats(qgm_ctx* ctx, qgm_ref* ref, uint32_t q, uint64_t threshold) {
  if (!ctx || !ref) return QGM_ERR_INPUT;
  return guard(ctx, [&] {
    activate(ctx);
    require(q >= 1 && q <= 16, "q must be in [1, 16]");
    qgm::mask_repeats(ctx->c, ref->r, q, threshold);
    QGM_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int qgm_ref_mask_download(qgm_ctx* ctx, const qgm_ref* ref, uint64_t* mask_bits) {
  if (!ctx || !ref || !mask_bits) return QGM_ERR_INPUT;
  return guard(ctx, [&] {
    activate(ctx);
    const uint64_t mw = qgm::ceil_div(ref->r.total, 64);
    if (!ref->r.mask.p) {
      std::fill(mask_bits, mask_bits + mw, 0ull);
      return;
    }
    if (mw) QGM_CUDA(cudaMemcpyAsync(mask_bits, ref->r.mask.p, mw * 8, cudaMemcpyDeviceToHost, ctx->c.stream));
    QGM_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

void qgm_ref_destroy(qgm_ref* r) {
  if (!r) return;
  cudaSetDevice(r->owner->c.device);
  delete r;
}

int qgm_filter(qgm_ctx* ctx, const qgm_index* idx, const qgm_reads* reads, const qgm_ref* ref, int strands, int mode,
               qgm_cands** out) {
  if (!ctx || !idx || !reads || !ref || !out) return QGM_ERR_INPUT;
  *out = nullptr;
  auto cd = std::make_unique<qgm_cands>();
  cd->owner = ctx;
  int rc = guard(ctx, [&] {
    activate(ctx);
    require(strands >= 1 && strands <= 3, "strands must be 1, 2 or 3");
    const int base_mode = mode & ~(QGM_FILTER_JOIN | QGM_FILTER_STREAM);
    require(base_mode == QGM_FILTER_FULL || base_mode == QGM_FILTER_RUN_START, "unknown filter mode");
    require(!((mode & QGM_FILTER_JOIN) && (mode & QGM_FILTER_STREAM)), "QGM_FILTER_JOIN and QGM_FILTER_STREAM exclude each other");
    const bool join = (mode & QGM_FILTER_JOIN) ||
                      (!(mode & QGM_FILTER_STREAM) && ref->r.padded_total < (uint64_t(1) << 32));
    qgm::Ctx& c = ctx->c;
    auto& C = cd->c;
    C.read_bits = qgm::read_bits_for(reads->r.n);
    C.diag_bits = ref->r.diag_bits;
    C.cbp = ref->r.cbp;
    if (idx->i.stride != reads->r.stride || idx->i.n_reads != reads->r.n)
      throw qgm::InputError("index was built over a different read buffer");
    if (join) {
      qgm::Partitioned rbk;
      qgm::partition_reads(c, reads->r, idx->i.q, rbk);
      qgm::StageScope s(c, qgm::kStageFilter);
      C.n = qgm::join_filter(c, rbk, reads->r, ref->r, strands, base_mode, C.read_bits, C.keys);
    } else {
      qgm::StageScope s(c, qgm::kStageFilter);
      C.n = qgm::filter_reference(c, idx->i, reads->r, ref->r, strands, base_mode, C.read_bits, C.keys);
    }
    qgm::StageScope s(c, qgm::kStageSort);
    qgm::DBuf<uint64_t> alt;
    qgm::radix_sort(c, C.keys, alt, nullptr, nullptr, C.n, 0, int(C.read_bits + 1 + C.diag_bits));
  });
  if (rc == QGM_OK) *out = cd.release();
  return rc;
}

int qgm_cands_count(const qgm_cands* c, uint64_t* n) {
  if (!c || !n) return QGM_ERR_INPUT;
  *n = c->c.n;
  return QGM_OK;
}

int qgm_cands_unique(qgm_ctx* ctx, qgm_cands* cd) {
  if (!ctx || !cd) return QGM_ERR_INPUT;
  return guard(ctx, [&] {
    activate(ctx);
    qgm::Ctx& c = ctx->c;
    auto& C = cd->c;
    qgm::DBuf<uint64_t> u(c, std::max<uint64_t>(C.n, 1));
    C.n = qgm::select_u64(c, C.keys.p, nullptr, nullptr, C.n, u.p, nullptr);
    C.keys.swap(u);
  });
}

int qgm_cands_download(qgm_ctx* ctx, const qgm_cands* cd, qgm_candidate* out) {
  if (!ctx || !cd || (!out && cd->c.n)) return QGM_ERR_INPUT;
  return guard(ctx, [&] {
    activate(ctx);
    const auto& C = cd->c;
    std::vector<uint64_t> k(C.n);
    if (C.n) QGM_CUDA(cudaMemcpyAsync(k.data(), C.keys.p, C.n * 8, cudaMemcpyDeviceToHost, ctx->c.stream));
    QGM_CUDA(cudaStreamSynchronize(ctx->c.stream));
    const uint64_t dmask = (uint64_t(1) << C.diag_bits) - 1;
    const uint64_t gap = C.cbp.size() >= 2 ? (C.cbp[0]) : 0;  // cbp[0] = gap
    for (uint64_t i = 0; i < C.n; ++i) {
      const uint64_t key = k[i];
      const uint64_t gp = key & dmask;
      // largest c with cbp[c] - gap <= gp
      size_t lo = 0, hi = C.cbp.size() - 1;
      while (hi - lo > 1) {
        size_t mid = (lo + hi) / 2;
        if (C.cbp[mid] - gap <= gp) lo = mid; else hi = mid;
      }
      out[i].diagonal = int64_t(gp) - int64_t(C.cbp[lo]);
      out[i].read_id = uint32_t(key >> (C.diag_bits + 1));
      out[i].chrom = uint32_t(lo);
      out[i].strand = uint32_t((key >> C.diag_bits) & 1);
      out[i].reserved = 0;
    }
  });
}

void qgm_cands_destroy(qgm_cands* c) {
  if (!c) return;
  cudaSetDevice(c->owner->c.device);
  delete c;
}

int qgm_validate(qgm_ctx* ctx, const qgm_reads* reads, const qgm_ref* ref, const qgm_candidate* cands, uint64_t n,
                 uint32_t band, uint32_t pct, qgm_validated* out) {
  if (!ctx || !reads || !ref || ((!cands || !out) && n)) return QGM_ERR_INPUT;
  return guard(ctx, [&] {
    activate(ctx);
    qgm::Ctx& c = ctx->c;
    const auto& R = ref->r;
    const unsigned rb = qgm::read_bits_for(reads->r.n);
    require(rb + 1 + R.diag_bits <= 64, "read batch too large for the 64-bit key");
    std::vector<uint64_t> keys(n);
    for (uint64_t i = 0; i < n; ++i) {
      const auto& cd = cands[i];
      require(cd.read_id < reads->r.n, "candidate read id out of range");
      require(cd.chrom < R.n_chrom, "candidate chromosome out of range");
      require(cd.strand <= 1, "candidate strand must be 0 or 1");
      const int64_t Lc = int64_t(R.cb[cd.chrom + 1] - R.cb[cd.chrom]);
      require(cd.diagonal > -int64_t(R.gap) + 64 && cd.diagonal < Lc, "candidate diagonal out of range");
      keys[i] = (uint64_t(cd.read_id) << (R.diag_bits + 1)) | (uint64_t(cd.strand) << R.diag_bits) |
                uint64_t(int64_t(R.cbp[cd.chrom]) + cd.diagonal);
    }
    qgm::StageScope s(c, qgm::kStageValidate);
    qgm::DBuf<uint64_t> dk(c, std::max<uint64_t>(n, 1));
    qgm::DBuf<uint8_t> dv(c, std::max<uint64_t>(n * 20, 20));
    if (n) QGM_CUDA(cudaMemcpyAsync(dk.p, keys.data(), n * 8, cudaMemcpyHostToDevice, c.stream));
    qgm::validate_candidates(c, reads->r, R, dk.p, n, rb, band, pct, 1, nullptr, nullptr, nullptr, dv.p);
    std::vector<uint32_t> raw(n * 5);
    if (n) QGM_CUDA(cudaMemcpyAsync(raw.data(), dv.p, n * 20, cudaMemcpyDeviceToHost, c.stream));
    QGM_CUDA(cudaStreamSynchronize(c.stream));
    for (uint64_t i = 0; i < n; ++i) {
      out[i].edits = int32_t(raw[i * 5]);
      out[i].start = raw[i * 5 + 1];
      out[i].ref_start = raw[i * 5 + 2];
      out[i].kept = uint8_t(raw[i * 5 + 3] & 0xFF);
      out[i].in_range = uint8_t((raw[i * 5 + 3] >> 8) & 0xFF);
      out[i].reserved0 = out[i].reserved1 = 0;
      out[i].reserved2 = 0;
    }
  });
}

int qgm_map(qgm_ctx* ctx, const qgm_reads* reads, const qgm_ref* ref, const qgm_map_params* P, qgm_hits** out) {
  if (!ctx || !reads || !ref || !P || !out) return QGM_ERR_INPUT;
  *out = nullptr;
  auto h = std::make_unique<qgm_hits>();
  h->owner = ctx;
  int rc = guard(ctx, [&] {
    activate(ctx);
    h->h = qgm::map_reads(ctx->c, reads->r, ref->r, *P);
  });
  if (rc == QGM_OK) *out = h.release();
  return rc;
}

int qgm_hits_count(const qgm_hits* h, uint64_t* n) {
  if (!h || !n) return QGM_ERR_INPUT;
  *n = h->h.n;
  return QGM_OK;
}

int qgm_hits_stats(const qgm_hits* h, qgm_map_stats* o) {
  if (!h || !o) return QGM_ERR_INPUT;
  o->raw_candidates = h->h.stats[0];
  o->unique_candidates = h->h.stats[1];
  o->validated = h->h.stats[2];
  o->hits = h->h.stats[3];
  o->index_distinct = h->h.stats[4];
  o->index_occurrences = h->h.stats[5];
  o->lookups_hit = h->h.stats[6];
  o->occurrences = h->h.stats[7];
  return QGM_OK;
}

int qgm_hits_download(qgm_ctx* ctx, const qgm_hits* h, qgm_hit* out) {
  if (!ctx || !h || (!out && h->h.n)) return QGM_ERR_INPUT;
  return guard(ctx, [&] {
    activate(ctx);
    qgm::StageScope s(ctx->c, qgm::kStageD2H);
    if (h->h.n)  // host or device destination (unified addressing)
      QGM_CUDA(cudaMemcpyAsync(out, h->h.hits.p, h->h.n * 16, cudaMemcpyDefault, ctx->c.stream));
    QGM_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int qgm_hits_ranks(qgm_ctx* ctx, const qgm_hits* h, uint32_t* rank) {
  if (!ctx || !h || (!rank && h->h.n)) return QGM_ERR_INPUT;
  return guard(ctx, [&] {
    activate(ctx);
    qgm::DBuf<uint32_t> r;
    qgm::hit_ranks(ctx->c, h->h.hits, h->h.n, h->h.n_reads, r);
    if (h->h.n) QGM_CUDA(cudaMemcpyAsync(rank, r.p, h->h.n * 4, cudaMemcpyDeviceToHost, ctx->c.stream));
    QGM_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

namespace {
int cigar_impl(qgm_ctx* ctx, const qgm::DBuf<uint8_t>* dev_hits, const qgm_hit* host_hits, uint64_t n,
               const qgm_reads* reads, const qgm_ref* ref, uint32_t band_width, uint32_t max_ops, uint32_t* ops,
               qgm_cigar_info* out) {
  if (!ctx || !reads || !ref || (n && (!ops || !out))) return QGM_ERR_INPUT;
  return guard(ctx, [&] {
    activate(ctx);
    require(band_width >= 1 && band_width <= 64, "band_width must be in [1, 64]");
    require(max_ops >= 1, "max_ops must be positive");
    qgm::DBuf<uint8_t> up;
    if (!dev_hits) {
      up.alloc(ctx->c, std::max<uint64_t>(n, 1) * 16);
      if (n) QGM_CUDA(cudaMemcpyAsync(up.p, host_hits, n * 16, cudaMemcpyHostToDevice, ctx->c.stream));
      dev_hits = &up;
    }
    qgm::DBuf<uint32_t> d_ops;
    qgm::DBuf<uint2> d_info;
    qgm::hits_cigar(ctx->c, *dev_hits, n, reads->r, ref->r, band_width, max_ops, d_ops, d_info);
    if (n) {
      QGM_CUDA(cudaMemcpyAsync(ops, d_ops.p, n * max_ops * 4, cudaMemcpyDeviceToHost, ctx->c.stream));
      QGM_CUDA(cudaMemcpyAsync(out, d_info.p, n * 8, cudaMemcpyDeviceToHost, ctx->c.stream));
    }
    QGM_CUDA(cudaStreamSynchronize(ctx->c.stream));
    uint32_t need = 0;
    for (uint64_t i = 0; i < n; ++i) need = std::max<uint32_t>(need, out[i].n_ops);
    if (need > max_ops)
      throw qgm::InputError("cigar: a record needs " + std::to_string(need) + " operations, max_ops is " +
                            std::to_string(max_ops));
  });
}
}  // namespace

int qgm_hits_cigar(qgm_ctx* ctx, const qgm_hits* h, const qgm_reads* reads, const qgm_ref* ref,
                   uint32_t band_width, uint32_t max_ops, uint32_t* ops, qgm_cigar_info* out) {
  if (!h) return QGM_ERR_INPUT;
  return cigar_impl(ctx, &h->h.hits, nullptr, h->h.n, reads, ref, band_width, max_ops, ops, out);
}

int qgm_cigar_records(qgm_ctx* ctx, const qgm_reads* reads, const qgm_ref* ref, const qgm_hit* hits, uint64_t n,
                      uint32_t band_width, uint32_t max_ops, uint32_t* ops, qgm_cigar_info* out) {
  if (!hits && n) return QGM_ERR_INPUT;
  return cigar_impl(ctx, nullptr, hits, n, reads, ref, band_width, max_ops, ops, out);
}

int qgm_ref_positions(qgm_ctx* ctx, qgm_ref* ref, uint32_t q, uint64_t* positions) {
  if (!ctx || !ref || !positions) return QGM_ERR_INPUT;
  return guard(ctx, [&] {
    activate(ctx);
    require(q >= 1 && q <= 16, "q must be in [1, 16]");
    require(ref->r.padded_total < (uint64_t(1) << 32), "reference index: more than 2^32-1 padded bases");
    qgm::prepare_ref_index(ctx->c, ref->r, q);
    QGM_CUDA(cudaStreamSynchronize(ctx->c.stream));
    *positions = ref->r.qidx.positions;
  });
}

void qgm_hits_destroy(qgm_hits* h) {
  if (!h) return;
  cudaSetDevice(h->owner->c.device);
  delete h;
}

int qgm_map_host(qgm_ctx* ctx, const uint64_t* reads2bit, const uint32_t* lengths, uint32_t n_reads, uint32_t stride,
                 const qgm_ref* ref, const qgm_map_params* P, qgm_hit* out, uint64_t cap, uint64_t* n_out,
                 qgm_map_stats* stats) {
  if (!ctx || !ref || !P || !n_out) return QGM_ERR_INPUT;
  qgm_reads* rd = nullptr;
  int rc = qgm_reads_upload(ctx, reads2bit, lengths, n_reads, stride, &rd);
  if (rc) return rc;
  qgm_hits* h = nullptr;
  rc = qgm_map(ctx, rd, ref, P, &h);
  if (rc == QGM_OK) {
    *n_out = h->h.n;
    if (stats) qgm_hits_stats(h, stats);
    if (h->h.n > cap) {
      ctx->c.err = "output capacity too small";
      rc = QGM_ERR_INPUT;
    } else {
      rc = qgm_hits_download(ctx, h, out);
    }
  }
  qgm_hits_destroy(h);
  qgm_reads_destroy(rd);
  return rc;
}

// Streamed batches (the paper's overlapped pipeline): the
// reads of batch i+1 are copied in on the context's copy stream while batch i
// is mapped on the compute stream, and the hits of batch i are copied out
// while batch i+1 is mapped. Two device input slots; a batch's hit buffer is
// released only after its D2H completed (the block cache hands blocks out in
// compute-stream order only).
int qgm_map_host_batches(qgm_ctx* ctx, qgm_batch* batches, uint32_t n_batches, const qgm_ref* ref,
                         const qgm_map_params* P) {
  if (!ctx || !ref || !P || (n_batches && !batches)) return QGM_ERR_INPUT;
  struct Slot {
    qgm::DBuf<uint64_t> words;
    qgm::DBuf<uint32_t> lens;
    qgm::DBuf<uint64_t> dense;  // staging of a QGM_READS_DENSE batch
    cudaEvent_t h2d = nullptr;
  };
  struct Pending {
    qgm::HitsObj h;
    cudaEvent_t comp = nullptr, done = nullptr;
    bool live = false;
  };
  Slot slot[2];
  Pending pend[2];
  int overflow = 0;
  int rc = guard(ctx, [&] {
    activate(ctx);
    qgm::Ctx& c = ctx->c;
    if (!c.copy_stream) QGM_CUDA(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
    if (!c.d2h_stream) QGM_CUDA(cudaStreamCreateWithFlags(&c.d2h_stream, cudaStreamNonBlocking));
    const cudaStream_t cs = c.copy_stream, ds = c.d2h_stream;
    for (auto& s : slot) QGM_CUDA(cudaEventCreateWithFlags(&s.h2d, cudaEventDisableTiming));
    for (auto& p : pend) {
      QGM_CUDA(cudaEventCreateWithFlags(&p.comp, cudaEventDisableTiming));
      QGM_CUDA(cudaEventCreateWithFlags(&p.done, cudaEventDisableTiming));
    }
    // both slots sized for the largest batch up front (allocated on the
    // compute stream's block cache, released after both streams are idle)
    uint64_t max_w = 1, max_n = 1, max_d = 1;
    for (uint32_t i = 0; i < n_batches; ++i) {
      const qgm_batch& b = batches[i];
      qgm::check_reads_shape(b.n_reads, b.stride);
      require(b.n_reads == 0 || b.reads2bit, "null read buffers");
      require(b.layout == QGM_READS_PADDED || b.layout == QGM_READS_DENSE, "unknown read layout");
      max_w = std::max<uint64_t>(max_w, uint64_t(b.n_reads) * ((b.stride + 31) / 32) + 2);
      max_n = std::max<uint64_t>(max_n, b.n_reads);
      if (b.layout == QGM_READS_DENSE) max_d = std::max<uint64_t>(max_d, qgm::ceil_div(uint64_t(b.n_reads) * b.stride, 32) + 1);
    }
    for (auto& s : slot) {
      s.words.alloc(c, max_w);
      s.lens.alloc(c, max_n);
      s.dense.alloc(c, max_d);
    }
    QGM_CUDA(cudaStreamSynchronize(c.stream));  // allocations visible before the copy stream writes
    auto h2d = [&](uint32_t i) {
      const qgm_batch& b = batches[i];
      Slot& s = slot[i & 1];
      if (b.layout == QGM_READS_DENSE) {
        const uint64_t nd = qgm::ceil_div(uint64_t(b.n_reads) * b.stride, 32);
        if (nd) QGM_CUDA(cudaMemcpyAsync(s.dense.p, b.reads2bit, nd * 8, cudaMemcpyHostToDevice, cs));
        QGM_CUDA(cudaMemsetAsync(s.dense.p + nd, 0, 8, cs));
      } else {
        const uint64_t nw = uint64_t(b.n_reads) * ((b.stride + 31) / 32);
        if (nw) QGM_CUDA(cudaMemcpyAsync(s.words.p, b.reads2bit, nw * 8, cudaMemcpyHostToDevice, cs));
        QGM_CUDA(cudaMemsetAsync(s.words.p + nw, 0, 16, cs));
      }
      if (b.n_reads && b.lengths)
        QGM_CUDA(cudaMemcpyAsync(s.lens.p, b.lengths, uint64_t(b.n_reads) * 4, cudaMemcpyHostToDevice, cs));
      QGM_CUDA(cudaEventRecord(s.h2d, cs));
    };
    auto d2h = [&](uint32_t i) {  // batch i's hits, after its mapping (comp event)
      qgm_batch& b = batches[i];
      Pending& p = pend[i & 1];
      if (p.h.n > b.cap) {
        overflow = 1;
      } else if (p.h.n) {
        QGM_CUDA(cudaStreamWaitEvent(ds, p.comp, 0));
        QGM_CUDA(cudaMemcpyAsync(b.out, p.h.hits.p, p.h.n * 16, cudaMemcpyDeviceToHost, ds));
      }
      QGM_CUDA(cudaEventRecord(p.done, ds));
    };
    if (n_batches) h2d(0);
    for (uint32_t i = 0; i < n_batches; ++i) {
      qgm_batch& b = batches[i];
      Slot& s = slot[i & 1];
      QGM_CUDA(cudaStreamWaitEvent(c.stream, s.h2d, 0));
      qgm::Reads r;
      r.n = b.n_reads;
      r.stride = b.stride;
      r.W = (b.stride + 31) / 32;
      {  // expand a dense batch / fill uniform lengths on the compute stream
        const unsigned g = unsigned(std::min<uint64_t>(qgm::ceil_div(std::max<uint64_t>(uint64_t(r.n) * r.W, 1), 256),
                                                       qgm::kSMs * 16));
        if (b.layout == QGM_READS_DENSE && r.n) {
          QGM_KERNEL(c, qgm::k_unpack_dense, g, 256, 0, s.dense.p, r.n, r.stride, r.W, s.words.p);
          fill_bytes(c, s.words.p + uint64_t(r.n) * r.W, 0, 16);
        }
        if (!b.lengths && r.n) QGM_KERNEL(c, qgm::k_fill_u32, g, 256, 0, s.lens.p, uint64_t(r.n), r.stride);
      }
      r.words.swap(s.words);
      r.lengths.swap(s.lens);
      struct Back {  // the slot keeps its buffers whatever happens; the planes
                     // block returns to the cache only after its side-stream build
        qgm::Ctx& c;
        qgm::Reads& r;
        Slot& s;
        ~Back() { r.words.swap(s.words); r.lengths.swap(s.lens); c.wait_planes(); }
      } back{c, r, s};
      {
        qgm::StageScope st(c, qgm::kStageReads);
        qgm::finish_reads(c, r);
      }
      Pending& p = pend[i & 1];
      if (p.live) {  // batch i-2's hits must be downloaded before its buffer goes back to the cache
        QGM_CUDA(cudaEventSynchronize(p.done));
        p.h = qgm::HitsObj();
        p.live = false;
      }
      // the copies run while the compute-bound validation of batch i runs:
      // batch i-1's hits out, batch i+1's reads in (slot (i+1)&1 was last read
      // by batch i-1, finished)
      p.h = qgm::map_reads(c, r, ref->r, *P, [&] {
        if (i >= 1) d2h(i - 1);
        if (i + 1 < n_batches) h2d(i + 1);
      });
      QGM_CUDA(cudaEventRecord(p.comp, c.stream));
      p.live = true;
      b.n_out = p.h.n;
      std::memset(&b.stats, 0, sizeof(b.stats));
      b.stats.raw_candidates = p.h.stats[0];
      b.stats.unique_candidates = p.h.stats[1];
      b.stats.validated = p.h.stats[2];
      b.stats.hits = p.h.stats[3];
      b.stats.index_distinct = p.h.stats[4];
      b.stats.index_occurrences = p.h.stats[5];
      b.stats.lookups_hit = p.h.stats[6];
      b.stats.occurrences = p.h.stats[7];
    }
    if (n_batches) d2h(n_batches - 1);
    QGM_CUDA(cudaStreamSynchronize(cs));
    QGM_CUDA(cudaStreamSynchronize(ds));
    QGM_CUDA(cudaStreamSynchronize(c.stream));
  });
  if (ctx->c.copy_stream) cudaStreamSynchronize(ctx->c.copy_stream);
  if (ctx->c.d2h_stream) cudaStreamSynchronize(ctx->c.d2h_stream);
  cudaStreamSynchronize(ctx->c.stream);
  for (auto& p : pend) {
    p.h = qgm::HitsObj();
    if (p.comp) cudaEventDestroy(p.comp);
    if (p.done) cudaEventDestroy(p.done);
  }
  for (auto& s : slot)
    if (s.h2d) cudaEventDestroy(s.h2d);
  if (rc == QGM_OK && overflow) {
    ctx->c.err = "output capacity too small (see qgm_batch.n_out)";
    return QGM_ERR_INPUT;
  }
  return rc;
}

int qgm_exclusive_scan_u32(qgm_ctx* ctx, const uint32_t* in, uint64_t n, uint32_t* out, uint32_t* total) {
  if (!ctx || ((!in || !out) && n)) return QGM_ERR_INPUT;
  return guard(ctx, [&] {
    activate(ctx);
    qgm::Ctx& c = ctx->c;
    qgm::DBuf<uint32_t> d(c, std::max<uint64_t>(n, 1));
    qgm::DBuf<uint32_t> t(c, 1);
    qgm::DBuf<int> ov(c, 1);
    if (n) QGM_CUDA(cudaMemcpyAsync(d.p, in, n * 4, cudaMemcpyHostToDevice, c.stream));
    qgm::exclusive_scan_u32(c, d.p, d.p, n, t.p, ov.p);
    int o = 0;
    uint32_t tot = 0;
    QGM_CUDA(cudaMemcpyAsync(&o, ov.p, 4, cudaMemcpyDeviceToHost, c.stream));
    QGM_CUDA(cudaMemcpyAsync(&tot, t.p, 4, cudaMemcpyDeviceToHost, c.stream));
    if (n) QGM_CUDA(cudaMemcpyAsync(out, d.p, n * 4, cudaMemcpyDeviceToHost, c.stream));
    QGM_CUDA(cudaStreamSynchronize(c.stream));
    if (o) throw qgm::InputError("prefix sum overflows the index word");
    if (total) *total = tot;
  });
}

}  // extern "C"
