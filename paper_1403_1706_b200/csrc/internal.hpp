// internal.hpp -- host-side objects behind the C ABI and the launcher API of
// the kernel files. Not installed; include/qgm_c.h is the public surface.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <initializer_list>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace qgm {

// --------------------------------------------------------------- context
enum Stage { kStageReads = 0, kStageIndex, kStageFilter, kStageSort, kStageValidate, kStageStrata, kStageD2H,
             kStageOther, kNumStages };

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t copy_stream = nullptr;  // H2D of qgm_map_host_batches (created on first use)
  cudaStream_t d2h_stream = nullptr;   // its D2H: a second stream, so uploads and downloads
                                       // use separate copy engines and overlap each other
  // side stream: the reads' bit planes (validation input) are built there,
  // concurrently with the partition and the join; planes_ev marks the last
  // planes build and every planes consumer / release waits for it
  cudaStream_t side_stream = nullptr;
  cudaEvent_t side_ev = nullptr, planes_ev = nullptr;
  void wait_planes() {
    if (planes_ev) cudaStreamWaitEvent(stream, planes_ev, 0);
  }
  uint64_t last_raw_candidates = 0;    // sizes the next batch's candidate buffer
  uint32_t* tail_h = nullptr;          // mapped pinned page of read_back (host / device view)
  uint32_t* tail_d = nullptr;
  std::string err;
  uint64_t launches = 0;
  bool profile = false;
  struct Mark { int stage; cudaEvent_t a, b; };
  std::vector<Mark> marks;          // recorded, not yet folded into stage_ms
  std::vector<cudaEvent_t> ev_pool; // reusable events
  double stage_ms[kNumStages] = {0};
  double host_ms[kNumStages] = {0};  // host wall time spent inside each stage
  std::chrono::steady_clock::time_point cur_host;
  int cur_stage = -1;
  cudaEvent_t cur_a = nullptr;
  // per-kernel timing of the hot kernels (name -> total ms, launches)
  struct KMark { const char* name; cudaEvent_t a, b; };
  std::vector<KMark> kmarks;
  std::vector<std::pair<std::string, std::pair<double, uint64_t>>> kernel_ms;

  // Block cache: every device buffer of this context comes from here. Blocks
  // are rounded up to size classes (<= 25% slack) and return to a free list
  // on release; all work of a context runs on its one stream, so a released
  // block can be handed out again without synchronisation (stream order).
  // Steady-state batches therefore never call the driver allocator.
  std::vector<std::pair<size_t, void*>> free_blocks;
  size_t cached_bytes = 0, live_bytes = 0;

  cudaEvent_t take_event();
  void stage_begin(int s);
  void stage_end();
  void fold_marks();  // synchronises the recorded events
  void* block_alloc(size_t bytes, size_t& cls);
  void block_free(void* p, size_t cls);
  void block_trim();  // frees every cached block (synchronises the stream)
};

// Size class of an allocation: 1/4-octave granularity above 4 KiB.
inline size_t size_class(size_t bytes) {
  if (bytes <= 4096) return 4096;
  size_t top = size_t(1) << (63 - __builtin_clzll(bytes - 1));  // largest power of two < bytes
  const size_t step = top / 4;
  return (bytes + step - 1) / step * step;
}

struct StageScope {
  Ctx& c;
  StageScope(Ctx& ctx, int s) : c(ctx) { c.stage_begin(s); }
  ~StageScope() { c.stage_end(); }
};

// CUDA-event timing of one kernel launch (profile mode only).
struct KernelScope {
  Ctx& c;
  const char* name;
  cudaEvent_t a = nullptr;
  KernelScope(Ctx& ctx, const char* n) : c(ctx), name(n) {
    if (c.profile) {
      a = c.take_event();
      QGM_CUDA(cudaEventRecord(a, c.stream));
    }
  }
  ~KernelScope() {
    if (!a) return;
    cudaEvent_t b = c.take_event();
    cudaEventRecord(b, c.stream);
    c.kmarks.push_back({name, a, b});
  }
};

// Programmatic dependent launch. Every kernel of the library starts with
// QGM_GRID_DEP(): wait until the grids it depends on have completed and
// their writes are visible, then allow the next kernel of the stream to be
// scheduled. Launched with programmatic stream serialization, a kernel's
// CTAs are placed while its predecessor's last CTAs still run and start
// the moment it completes, instead of the GPU draining at every boundary
// (a batch is ~35 dependent launches; C1 is bound by those boundaries).
// tests/test_capi_symbols.py checks that every __global__ begins with it.
#define QGM_GRID_DEP() asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")

bool pdl_enabled();  // QGM_PDL=0: plain stream serialization (A/B)

inline cudaLaunchConfig_t launch_config(Ctx& c, dim3 grid, dim3 block, size_t smem, cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cfg;
}

// Launch on the context stream (programmatic serialization), count it,
// surface launch errors.
#define QGM_KERNEL(ctx, kernel, grid, block, smem, ...)                          \
  do {                                                                         \
    cudaLaunchAttribute qgm_attr_[1];                                          \
    const cudaLaunchConfig_t qgm_cfg_ =                                        \
        ::qgm::launch_config((ctx), dim3(grid), dim3(block), size_t(smem), qgm_attr_); \
    QGM_CUDA(cudaLaunchKernelEx(&qgm_cfg_, kernel, __VA_ARGS__));              \
    ++(ctx).launches;                                                          \
    QGM_LAUNCH_CHECK();                                                        \
  } while (0)

// cudaMemsetAsync as a kernel of the stream: a memset node between two
// kernels would end their programmatic overlap. value is a byte.
void fill_bytes(Ctx& c, void* p, int value, size_t bytes);

// Small device counters to host variables: one gather kernel into the
// context's mapped pinned page and one stream synchronisation (instead of a
// pageable cudaMemcpyAsync per counter, each a blocking round trip, and a
// copy node that ends the programmatic overlap of the kernels before it).
struct ReadSeg {
  const void* src;  // device, 4-byte aligned
  void* dst;        // host
  size_t bytes;     // multiple of 4
};
constexpr int kMaxReadSegs = 8;
constexpr size_t kReadBackBytes = 4096;
void read_back(Ctx& c, std::initializer_list<ReadSeg> segs);

// --------------------------------------------------------------- memory
// Device buffer from the context's block cache (Ctx::block_alloc).
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  size_t cls = 0;
  Ctx* ctx = nullptr;
  DBuf() = default;
  DBuf(Ctx& c, size_t count) { alloc(c, count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { *this = std::move(o); }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; cls = o.cls; ctx = o.ctx;
      o.p = nullptr; o.n = 0; o.cls = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(Ctx& c, size_t count) {
    release();
    ctx = &c;
    n = count;
    if (count) p = static_cast<T*>(c.block_alloc(count * sizeof(T), cls));
  }
  void release() {
    if (p) ctx->block_free(p, cls);
    p = nullptr;
    n = 0;
    cls = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
  void zero() {
    if (n) fill_bytes(*ctx, p, 0, bytes());
  }
  void swap(DBuf& o) {
    std::swap(p, o.p); std::swap(n, o.n); std::swap(cls, o.cls); std::swap(ctx, o.ctx);
  }
};

// --------------------------------------------------------------- objects
// One read buffer (PackedReadText, seq.hpp:98-115) in the 2-bit layout, plus
// per-read bit planes (lo/hi bit of every base, MSB-first, one guard word in
// front) for the validation kernel.
struct Reads {
  uint32_t n = 0, stride = 0, W = 0, Wp = 0;
  DBuf<uint32_t> lens;     // device: {max length, ~min length} (no host round trip at upload;
                           // the first synchronising stage checks max <= stride)
  DBuf<uint64_t> words;    // n * W
  DBuf<uint32_t> lengths;  // n
  DBuf<uint2> planes;      // n * Wp, word 0 of every read is a zero guard
};

// q-group index (QGroupIndex<W>, qgroup_index.hpp:28-104) in device memory.
struct Index {
  unsigned q = 0, w = 32;
  bool sampled = false;
  uint64_t groups = 0, gs_len = 0, distinct = 0, occ = 0;
  uint32_t stride = 0, n_reads = 0;
  DBuf<uint8_t> I;        // groups words of w bits
  DBuf<uint32_t> S;       // gs_len
  DBuf<uint32_t> S1;      // distinct + 1
  DBuf<uint32_t> O;       // occ
};

// Items bucketed by the top 2q-lb bits of their q-gram code (the first half
// of the index build, index_build.cu). pairs[i] = extra << 48 | (code & (2^lb
// - 1)) << 32 | position (or, join_items, a raw-code partition's items);
// bucket k holds pairs[boff[k], boff[k+1]).
struct Buckets {
  unsigned q = 0, w = 32, lb = 0, hb = 0;
  uint64_t groups = 0, buckets = 0, gpb = 0;
  uint32_t V = 0;
  bool join_items = false;  // pairs are join items of a raw-code partition (partition.cu), lb = 16
  DBuf<uint32_t> boff;
  DBuf<uint64_t> pairs;
};

// q-group index over the reference itself, keyed by CANONICAL q-gram codes
// (canon_code: one fixed member of {code, rc(code)}; SPEC.md:262-316's precomputed reference index with P
// ordered by q-gram as in PAPER.md:344, both strands in one index). Every
// position x is listed under the canonical code of its forward window with
// flag = (forward code != canonical); a position whose q-gram is its own
// reverse complement (even q only) is listed twice, with flag 0 and 1. A read
// q-gram with code g looks up canon(g) once: an occurrence matches the
// forward strand iff flag == (g != canon(g)), else the reverse strand.
// Per occurrence: O = padded coordinate cbp[c] + p (the candidate diagonal is
// O - offset, no chromosome search) and extra = b | flag << 3 with b =
// ref[x-1] (4 = none: chromosome start or masked), the base the run-start
// rule compares. When the padded reference is < 2^28, extra is packed into
// O's top 4 bits (packed = true, `extra` empty).
struct RefQIndex {
  unsigned q = 0;
  bool packed = false;
  bool ex_sorted = false;  // packed O sorted inside every interval: grouped by (strand flag, compare base)
  uint64_t palindromes = 0;  // positions listed twice
  Index can;
  DBuf<uint8_t> extra;
  // per join sub-bin s (the 2^sub_bits prefixes of the partition, sub_bits =
  // min(2q, 16)): its distinct-code range [sb_d[s], sb_d[s+1]) of S' and
  // occurrence range [sb_o[s], sb_o[s+1]) of O; built when a sub-bin spans
  // >= 8 group words (the join stages these slices with bulk copies)
  uint64_t positions = 0;  // reference positions in P (|P| of mapping_quality)
  unsigned sub_bits = ~0u;
  DBuf<uint32_t> sb_d, sb_o;
  DBuf<uint16_t> r16;  // per group word: S[w] - sb_d[sub-bin of w] (group start inside its sub-bin)
};
constexpr unsigned kPackedPosBits = 28;

// Reference sequences (ReferenceIndex): the concatenated
// chromosomes in 2-bit (+1 guard word) and as lo/hi bit planes (2 guard words
// on both sides). Diagonals are keyed in a padded coordinate space where
// chromosome c starts at cbp[c] = cb[c] + (c+1)*gap, so (chrom, diagonal)
// round-trips through one unsigned integer.
struct Ref {
  uint32_t n_chrom = 0;
  uint64_t total = 0;
  uint64_t gap = 0;
  uint64_t padded_total = 0;
  unsigned diag_bits = 0;
  std::vector<uint64_t> cb;   // host copy, n_chrom+1
  std::vector<uint64_t> cbp;  // host copy, n_chrom+1 (padded begins)
  DBuf<uint64_t> words;       // ceil(total/32)+1
  DBuf<uint2> planes;         // ceil(total/32)+4 (lo, hi)
  DBuf<uint64_t> mask;        // nullable: bit x = masked
  DBuf<uint64_t> d_cb, d_cbp; // n_chrom+1 each
  mutable RefQIndex qidx;     // cache, built lazily per q (prepare_ref_index)
};

struct Cands {
  uint64_t n = 0;
  unsigned read_bits = 0, diag_bits = 0;
  std::vector<uint64_t> cbp;  // decode: padded chromosome begins
  DBuf<uint64_t> keys;        // (read, strand, padded diagonal), sorted
};

struct HitsObj {
  uint64_t n = 0;
  uint32_t n_reads = 0;
  // raw, unique, validated, hits, index distinct, index occurrences,
  // filtration lookups with the occupancy bit set, occurrences visited
  uint64_t stats[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  DBuf<uint8_t> hits;  // n * 16-byte qgm_hit
};

// --------------------------------------------------------------- launchers
// scan.cu -- exclusive scan of u32 values (u64 running sums). d_total and
// d_overflow (set to 1 when the total exceeds 2^32-1) are optional device
// outputs. in may equal out.
void exclusive_scan_u32(Ctx& c, const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* d_total,
                        int* d_overflow);
// Order-preserving selection of keys[i] with flag[i] != 0 (or, if flags is
// null, keys that differ from their predecessor: unique of a sorted array).
// Returns the count (host sync).
uint64_t select_u64(Ctx& c, const uint64_t* keys, const uint32_t* vals, const uint32_t* flags, uint64_t n,
                    uint64_t* out_keys, uint32_t* out_vals);

// dedup.cu -- unique keys (any order) of keys[0, n) into `out` (grown as
// needed); returns their count.
uint64_t dedup_keys(Ctx& c, const uint64_t* keys, uint64_t n, DBuf<uint64_t>& out);
// Same without a host round trip: `out` is sized n (the bound) and the unique
// count lands in d_count (device).
void dedup_keys_async(Ctx& c, const uint64_t* keys, uint64_t n, DBuf<uint64_t>& out, unsigned long long* d_count);
// The same with the key count on the device (*d_n, clamped to n_max): the
// table is allocated for n_max and sized for *d_n by the kernels themselves.
void dedup_keys_dev(Ctx& c, const uint64_t* keys, uint64_t n_max, const unsigned long long* d_n,
                    DBuf<uint64_t>& out, unsigned long long* d_count);
// Above the L2-resident size: one radix pass splits the keys into 256
// partitions on their low 8 bits (equal keys share every bit), then each
// partition is deduplicated in its own L2-sized hash table; unique keys in
// any order to out, their count to *d_count.
void dedup_keys_partitioned(Ctx& c, const uint64_t* keys, uint64_t n, DBuf<uint64_t>& out,
                            unsigned long long* d_count);
// Estimated duplicate fraction of a candidate set (keys of every 64th read).
double estimate_dup_fraction(Ctx& c, const uint64_t* keys, uint64_t n, unsigned rshift);

// radix_sort.cu -- stable LSD radix sort of u64 keys (+ optional u32 values)
// on bits [begin_bit, end_bit). Sorted data ends up in keys/vals (buffers may
// be swapped with the alternates).
// One stable 8-bit digit pass (bits [shift, shift + 8)) of u64 keys from in
// to out; digit d's keys land at [starts[d], starts[d+1]) (257 u32, device).
void radix_digit_pass(Ctx& c, const uint64_t* in, uint64_t* out, uint64_t n, int shift, uint32_t* starts);
void radix_sort(Ctx& c, DBuf<uint64_t>& keys, DBuf<uint64_t>& keys_alt, DBuf<uint32_t>* vals,
                DBuf<uint32_t>* vals_alt, uint64_t n, int begin_bit, int end_bit);

// reads / ref preparation (capi.cu)
void make_read_planes(Ctx& c, Reads& r);
void make_ref_planes(Ctx& c, Ref& ref);

// index_build.cu
void bucket_reads(Ctx& c, const Reads& reads, unsigned q, unsigned w, Buckets& out, unsigned lb_max = 13);
void bucket_ref(Ctx& c, const Ref& ref, unsigned q, bool packed, Buckets& out, uint64_t* n_pal);
// Repeat mask on the device: set the mask bit of every
// position whose forward q-gram occurs more than `threshold` times among the
// windows of its chromosome; drops the cached reference index.
void mask_repeats(Ctx& c, Ref& ref, unsigned q, uint64_t threshold);
// (Re)build the per-sub-bin tables of the cached reference index for sub-bins
// of 2^sub_bits code prefixes (no-op when they already match).
void subbin_tables(Ctx& c, const Ref& ref, unsigned sub_bits);
void index_from_buckets(Ctx& c, const Buckets& B, bool sampled, Index& out, DBuf<uint8_t>* extra);
void build_index(Ctx& c, const Reads& reads, unsigned q, unsigned w, bool sampled, Index& out);
void prepare_ref_index(Ctx& c, const Ref& ref, unsigned q);
void sample_index(Ctx& c, const Index& in, Index& out);
void normalize_index(Ctx& c, Index& idx);
void lookup_index(Ctx& c, const Index& idx, const uint32_t* d_codes, uint64_t n, uint32_t* d_begin,
                  uint32_t* d_end);

// filter.cu -- raw candidate keys (unsorted) appended to `keys` (grown and
// re-run on overflow). Returns the count.
// fstats (optional, host): {lookups with the occupancy bit set, occurrences visited}.
uint64_t filter_reference(Ctx& c, const Index& idx, const Reads& reads, const Ref& ref, int strands, int mode,
                          unsigned read_bits, DBuf<uint64_t>& keys, uint64_t* fstats = nullptr);

// partition.cu -- the batch's read q-grams grouped by the top min(2q,16)
// bits of their CANONICAL code (sub-bins), one 64-bit join item each:
//   bits  0..31  read text position pp = r * stride + o
//   bits 33..35  read base at o - 1 (forward run-start compare), 4 = none
//   bits 36..38  complement of the read base at o + q (reverse run-start
//                compare), 4 = none
//   bit  39      fr = (read code != canonical code)
//   bits 40..63  the canonical code bits below the first pass's 8-bit bin
//                (the join ORs them with its sub-bin prefix; the bits the
//                refinement grouped by are implied by the sub-bin)
// The first pass writes the item in its final form; the refinement only
// permutes items.
constexpr unsigned kItemFbShift = 33, kItemRbShift = 36, kItemFrShift = 39, kItemCodeShift = 40;
struct Partitioned {
  unsigned q = 0;
  uint32_t bins = 0, V = 0;
  unsigned sub_bits = 0;  // sub-bin = code >> (2q - sub_bits); sub_bits = min(2q, 16)
  // V above is the host-side bound n_reads * (stride - q + 1) (exact for
  // uniform batches); the exact values stay on the device, read back with the
  // join's candidate count (no host round trip inside the partition):
  // flags[0] = V, flags[1] = every read has length `stride` (n - q - o from pp
  // alone), flags[2] = a read is longer than the stride (input error)
  DBuf<uint32_t> flags;
  DBuf<uint32_t> boff;    // 8-bit bin offsets (first pass)
  DBuf<uint32_t> soff;    // sub-bin offsets, 2^sub_bits + 1 entries
  DBuf<uint64_t> pairs;
};
// raw: group by the q-grams' own codes (the read index of qgm_index_build)
// instead of canonical codes; force_key_bits (0 = adaptive): the sub-bin width.
void partition_reads(Ctx& c, const Reads& reads, unsigned q, Partitioned& out, bool raw = false,
                     unsigned force_key_bits = 0);

// join.cu -- the same candidates as filter_reference, from a code-ordered
// join of the partitioned read q-grams with the reference q-group indexes.
uint64_t join_filter(Ctx& c, const Partitioned& rp, const Reads& reads, const Ref& ref, int strands, int mode,
                     unsigned read_bits, DBuf<uint64_t>& keys, uint64_t* fstats = nullptr,
                     unsigned long long* dev_counter = nullptr);
// dev_counter (nullable): launch only, no host round trip -- the candidate
// count, join statistics and partition flags are the caller's to read back
// (keys.n is the capacity; a count above it means the keys were truncated).

// validate.cu
// mode 0: append kept hits as (hit key, k) to hit_keys/hit_vals (counter in
//         *d_count); mode 1: write one qgm_validated per candidate.
// d_n (nullable): the exact candidate count in device memory, n then only
// bounds it (no host round trip between dedup and validation). seed_q: the
// filtration's q (every candidate has a q-row exact seed; it places the map
// path's phase split).
void validate_candidates(Ctx& c, const Reads& reads, const Ref& ref, const uint64_t* cand_keys, uint64_t n,
                         unsigned read_bits, unsigned band, unsigned pct, int mode, uint64_t* hit_keys,
                         uint32_t* hit_vals, unsigned long long* d_count, void* d_validated,
                         const unsigned long long* d_n = nullptr, unsigned seed_q = 0,
                         uint32_t* per_read = nullptr, unsigned long long* d_big = nullptr);
// per_read (nullable, n_reads + 1 zeroed u32): the map path's hits per read,
// counted as they are emitted; *d_big += reads passing kSmallSeg hits (the
// strata's radix path) -- counted while the hits are emitted (no pass over them).
constexpr uint32_t kSmallSeg = 32;

// strata.cu -- dedup (read, chrom, ref_start, strand) keeping min k, then
// best-stratum / all; writes qgm_hit records, returns their count.
// Same output from hits in any order (map path): validation counts the hits
// per read as it emits them (per_read, *d_big += reads with more than
// kSmallSeg hits); stratify_unsorted then uses a per-read counting sort, or --
// when big -- the radix-sorted path.
uint64_t stratify_unsorted(Ctx& c, const Ref& ref, DBuf<uint64_t>& hit_keys, DBuf<uint32_t>& hit_vals, uint64_t n,
                           uint32_t n_reads, int mode, DBuf<uint32_t>& cnt, bool big, DBuf<uint8_t>& out);
// The per-read counting-sort path of stratify_unsorted with the hit count and
// the big flag left on the device (no host round trip before the output is
// written): every kernel reads *d_n and does nothing when *d_big != 0 (the
// caller then runs stratify_unsorted's radix path); `out` is sized for n_max
// records; *d_kept receives the record count.
void stratify_unsorted_dev(Ctx& c, const Ref& ref, const uint64_t* hit_keys, const uint32_t* hit_vals,
                           const unsigned long long* d_n, uint64_t n_max, uint32_t n_reads, int mode,
                           DBuf<uint32_t>& cnt, const unsigned long long* d_big, DBuf<uint8_t>& out,
                           uint32_t* d_kept);
// hit-rank of every output record: #records of its read
// whose identity is >= its own (edits <= its edits).
void hit_ranks(Ctx& c, const DBuf<uint8_t>& hits, uint64_t n, uint32_t n_reads, DBuf<uint32_t>& rank);
// cigar.cu -- traceback_cigar (DESIGN.md section 2 item 9) of every hit record: ops (n *
// max_ops BAM-style u32) and info {ref_start, n_ops | edits << 16}.
void hits_cigar(Ctx& c, const DBuf<uint8_t>& hits, uint64_t n, const Reads& reads, const Ref& ref, unsigned band,
                uint32_t max_ops, DBuf<uint32_t>& ops, DBuf<uint2>& info);
uint64_t stratify_hits(Ctx& c, const Ref& ref, const uint64_t* hit_keys, const uint32_t* hit_vals, uint64_t n,
                       uint32_t n_reads, unsigned read_bits, int mode, DBuf<uint8_t>& out);

// Per-process memo of launch configuration queries (they cost host time on
// every batch otherwise: small batches are bound by the host's enqueue rate).
struct LaunchMemo {
  std::mutex m;
  std::map<std::tuple<int, const void*, int, size_t>, unsigned> grid;
  std::map<std::pair<int, const void*>, size_t> smem;
  std::map<std::pair<int, const void*>, cudaFuncAttributes> attrs;
  static LaunchMemo& get() {
    static LaunchMemo memo;
    return memo;
  }
};

inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

// Persistent-grid size: SMs x resident CTAs per SM for this kernel/config
// (one full wave; grid-stride kernels then never run a partial second wave).
inline unsigned resident_grid(const void* kernel, int threads, size_t smem) {
  const int dev = current_device();
  LaunchMemo& M = LaunchMemo::get();
  std::lock_guard<std::mutex> lk(M.m);
  auto it = M.grid.find({dev, kernel, threads, smem});
  if (it != M.grid.end()) return it->second;
  int sms = kSMs, per = 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem);
  const unsigned g = unsigned(std::max(1, sms * std::max(1, per)));
  M.grid[{dev, kernel, threads, smem}] = g;
  return g;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when a kernel needs
// more dynamic shared memory than it was last configured for on this device.
inline void ensure_dynamic_smem(const void* kernel, size_t smem) {
  const int dev = current_device();
  LaunchMemo& M = LaunchMemo::get();
  std::lock_guard<std::mutex> lk(M.m);
  size_t& have = M.smem[{dev, kernel}];
  if (smem <= have) return;
  QGM_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  have = smem;
}

inline cudaFuncAttributes func_attributes(const void* kernel) {
  const int dev = current_device();
  LaunchMemo& M = LaunchMemo::get();
  std::lock_guard<std::mutex> lk(M.m);
  auto it = M.attrs.find({dev, kernel});
  if (it != M.attrs.end()) return it->second;
  cudaFuncAttributes fa;
  QGM_CUDA(cudaFuncGetAttributes(&fa, kernel));
  M.attrs[{dev, kernel}] = fa;
  return fa;
}

inline unsigned bit_width_u64(uint64_t x) {
  unsigned b = 0;
  while (x) { ++b; x >>= 1; }
  return b;
}

}  // namespace qgm
