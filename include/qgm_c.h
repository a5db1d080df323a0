/* qgm_c.h -- C ABI of the B200-native read-mapping hot path (libqgm_b200.so).
 *
 * The drop-in boundary for PEANUT's (arXiv 1403.1706) q-group-index mapper:
 * plain pointers and sizes, no C++ or torch types, no exceptions. Every entry
 * point names the reference interface it replaces (paths relative to the
 * reference checkout, proj/include/qgmap/... ; SPEC.md for the spec-only
 * stages). The C++ mirror of the reference API (the include/qgmap headers) and the
 * python binding (paper_1403_1706_b200/__init__.py) are thin layers over it.
 *
 * Sequence format ("2-bit MSB-first"): base j of a sequence lives in 64-bit
 * word j/32 at bits [62-2(j%32), 63-2(j%32)], codes A=0 C=1 G=2 T=3
 * (seq.hpp:18-19). Read r of a batch occupies words [r*W, (r+1)*W) with
 * W = ceil(stride/32); bases past the read length are ignored. N bases must be
 * replaced on the host before packing (seq.hpp:39; qgm_pack_codes does not
 * touch them).
 *
 * Status codes: 0 ok; 1 input error (qgmap::input_error, seq.hpp:13-16);
 * 2 internal/capacity (std::logic_error, parallel.hpp:176,181); 3 CUDA error.
 * qgm_last_error(ctx) returns the message of the last failure on ctx.
 *
 * Threading: one ctx per device; calls on a ctx are serialised on its stream
 * and are not re-entrant. Host buffers are caller-owned; device objects are
 * owned by their handle and released by the matching *_destroy.
 */
#ifndef QGM_C_H
#define QGM_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QGM_OK 0
#define QGM_ERR_INPUT 1
#define QGM_ERR_INTERNAL 2
#define QGM_ERR_CUDA 3

#define QGM_MODE_BEST_STRATUM 0
#define QGM_MODE_ALL 1

#define QGM_STRAND_FWD 1
#define QGM_STRAND_REV 2
#define QGM_STRAND_BOTH 3

#define QGM_FILTER_FULL 0      /* Alg. 2 multiset */
#define QGM_FILTER_RUN_START 1 /* leftmost q-gram of each run per diagonal (same set) */
#define QGM_FILTER_JOIN 2      /* flag: bucket-ordered join with the reference q-group index */
#define QGM_FILTER_STREAM 4    /* flag: stream every reference position against the read index */
/* Neither flag: the join when the reference is below 2^32 padded bases (the
 * production filtration), else the streaming kernel. */

typedef struct qgm_ctx qgm_ctx;
typedef struct qgm_reads qgm_reads;
typedef struct qgm_ref qgm_ref;
typedef struct qgm_index qgm_index;
typedef struct qgm_cands qgm_cands;
typedef struct qgm_hits qgm_hits;

/* Candidate (Hit{d, r} of SPEC.md:323-327 / oracle::HitKey oracles.hpp:29-33,
 * plus strand and chromosome). diagonal is chromosome-relative; strand 1 means
 * reverse_complement(read) aligns forward at `diagonal`. 24 bytes. */
typedef struct qgm_candidate {
  int64_t diagonal;
  uint32_t read_id;
  uint32_t chrom;
  uint32_t strand;
  uint32_t reserved;
} qgm_candidate;

/* Validation result of one candidate (ValidatedHit). 20 bytes. */
typedef struct qgm_validated {
  int32_t edits;       /* k: banded semi-global edit distance */
  uint32_t start;      /* window column of the smallest optimal start */
  uint32_t ref_start;  /* chromosome-relative alignment start (clamped) */
  uint8_t kept;        /* 100*(n-k) >= pct*n */
  uint8_t in_range;    /* window overlaps its chromosome */
  uint8_t reserved0, reserved1;
  uint32_t reserved2;
} qgm_validated;

/* Mapped hit after dedup + strata. 16 bytes. */
typedef struct qgm_hit {
  uint32_t read_id;
  uint32_t chrom;
  uint32_t ref_start;
  uint16_t edits;
  uint8_t strand;
  uint8_t reserved;
} qgm_hit;

typedef struct qgm_map_params {
  uint32_t q;            /* q-gram length, 1..16 (seq.hpp:27); default 16 */
  uint32_t group_width;  /* 32 or 64 (QGroupIndex<GroupWord>, qgroup_index.hpp:28) */
  uint32_t sampled;      /* sample_group_starts (qgroup_index.hpp:185) */
  uint32_t band_width;   /* B, 1..64; default 32 */
  uint32_t pct_identity; /* 0..100; default 80 */
  uint32_t mode;         /* QGM_MODE_* */
  uint32_t strands;      /* QGM_STRAND_*; default both */
  uint32_t reserved;
} qgm_map_params;

typedef struct qgm_index_info {
  uint32_t q, group_width, sampled, reserved;
  uint64_t group_count;        /* QGroupIndex::group_count()          :38 */
  uint64_t group_starts_len;   /* group_starts().size() (sentinel incl.) */
  uint64_t distinct;           /* distinct_qgram_count()              :40 */
  uint64_t occurrences;        /* occurrence_count() = |O|            :39 */
} qgm_index_info;

typedef struct qgm_map_stats {
  uint64_t raw_candidates;    /* filtration emissions (RUN_START mode) */
  uint64_t unique_candidates; /* after radix sort + unique */
  uint64_t validated;         /* candidates passing the identity threshold */
  uint64_t hits;              /* after dedup + strata */
  uint64_t index_distinct;    /* distinct read q-grams (|S'|-1) */
  uint64_t index_occurrences; /* indexed read q-grams (|O|) */
  uint64_t lookups_hit;       /* reference lookups whose occupancy bit was set */
  uint64_t occurrences;       /* (position, occurrence) pairs visited by filtration */
} qgm_map_stats;

/* ---- context ------------------------------------------------------------ */
int qgm_ctx_create(int device, qgm_ctx** out);
/* Run subsequent work on an existing cudaStream_t (NULL = ctx-owned stream). */
int qgm_ctx_set_stream(qgm_ctx* ctx, void* cuda_stream);
void* qgm_ctx_stream(qgm_ctx* ctx);
void qgm_ctx_destroy(qgm_ctx* ctx);
const char* qgm_last_error(const qgm_ctx* ctx);
int qgm_ctx_synchronize(qgm_ctx* ctx);
/* Per-stage CUDA-event timing (ms, accumulated until reset). Stage ids:
 * 0 reads prep, 1 index build, 2 filtration, 3 candidate sort+unique,
 * 4 validation, 5 strata, 6 hit D2H; entries 8..15 (if n > 8) are the host
 * wall-clock ms spent inside the same stages. */
#define QGM_NUM_STAGES 8
int qgm_ctx_profile(qgm_ctx* ctx, int enable);
int qgm_ctx_stage_times(qgm_ctx* ctx, double* ms, int n, int reset);
/* Per-kernel CUDA-event times of the hot kernels (profile mode): writes
 * "name<TAB>total_ms<TAB>launches\n" lines into buf (NUL-terminated). */
int qgm_ctx_kernel_times(qgm_ctx* ctx, char* buf, uint64_t cap, int reset);
/* Kernels launched on ctx since the last reset. */
uint64_t qgm_ctx_launches(qgm_ctx* ctx, int reset);

/* ---- host codec helpers (seq.hpp:33-56, 80-84) --------------------------- */
/* codes (1 byte per base, values 0..3) -> 2-bit MSB-first words. */
int qgm_pack_codes(const uint8_t* codes, uint64_t n, uint64_t* words);
/* n_reads reads at `stride` codes each -> n_reads*ceil(stride/32) words. */
int qgm_pack_reads(const uint8_t* codes, uint32_t stride, uint32_t n_reads, uint64_t* words);

/* ---- read batch: PackedReadText (seq.hpp:98-140) ------------------------- */
int qgm_reads_upload(qgm_ctx* ctx, const uint64_t* reads2bit, const uint32_t* lengths, uint32_t n_reads,
                     uint32_t stride, qgm_reads** out);
/* Same, from device-resident buffers (copied device-to-device). */
int qgm_reads_from_device(qgm_ctx* ctx, const uint64_t* d_reads2bit, const uint32_t* d_lengths,
                          uint32_t n_reads, uint32_t stride, qgm_reads** out);
void qgm_reads_destroy(qgm_reads* reads);

/* ---- q-group index: build_qgroup_index<W> (qgroup_index.hpp:124-180) ------ */
int qgm_index_build(qgm_ctx* ctx, const qgm_reads* reads, uint32_t q, uint32_t group_width, int sampled,
                    qgm_index** out);
/* sample_group_starts (qgroup_index.hpp:185-196): new index with halved S. */
int qgm_index_sample(qgm_ctx* ctx, const qgm_index* idx, qgm_index** out);
/* Sort positions within every occurrence interval (the normalisation of
 * test_parallel.cpp:121-122); makes O byte-reproducible. */
int qgm_index_normalize(qgm_ctx* ctx, qgm_index* idx);
int qgm_index_info_get(const qgm_index* idx, qgm_index_info* out);
/* Copy the four arrays to host (occupancy/group_starts/occ_starts/positions,
 * qgroup_index.hpp:42-45). Any pointer may be NULL. occupancy holds
 * group_count words of group_width bits. */
int qgm_index_download(qgm_ctx* ctx, const qgm_index* idx, void* occupancy, uint32_t* group_starts,
                       uint32_t* occ_starts, uint32_t* positions);
/* index_pair (qgroup_index.hpp:50-57) for n codes: [begin,end) or
 * begin=end=0xFFFFFFFF when absent. Host buffers. */
int qgm_index_lookup(qgm_ctx* ctx, const qgm_index* idx, const uint32_t* codes, uint64_t n, uint32_t* begin,
                     uint32_t* end);
void qgm_index_destroy(qgm_index* idx);

/* ---- reference: ReferenceIndex sequences ---------------- */
/* ref2bit: the concatenated chromosomes in the 2-bit format; chrom_begin:
 * n_chrom+1 base offsets (host); mask_bits (nullable): bit x of word x/64 set =
 * position x excluded from P (repeat mask). ref2bit and
 * mask_bits may be host or device pointers (unified addressing): a multi-GPU
 * run uploads the reference once and broadcasts the 2-bit words over NVLink,
 * then every rank calls this with its device copy. */
int qgm_ref_upload(qgm_ctx* ctx, const uint64_t* ref2bit, const uint64_t* chrom_begin, uint32_t n_chrom,
                   const uint64_t* mask_bits, qgm_ref** out);
/* Build (and cache on ref) the reference-side q-group indexes for q, one per
 * strand: the precomputed reference index of SPEC.md:262-316 with P ordered by
 * q-gram. qgm_map does this lazily on first use of a q; call it
 * ahead of time to keep it out of the first batch. References < 2^32 bases. */
int qgm_ref_prepare(qgm_ctx* ctx, qgm_ref* ref, uint32_t q);
/* Repeat mask on the device (build_reference_index's masking, SPEC.md:270,
 * 302; default threshold 1000): every position whose forward q-gram occurs
 * more than `threshold` times among the windows of its own chromosome is
 * removed from P (ORed into the upload mask). Drops the cached reference
 * index; call before qgm_ref_prepare / qgm_map. */
int qgm_ref_mask_repeats(qgm_ctx* ctx, qgm_ref* ref, uint32_t q, uint64_t threshold);
/* The current mask, ceil(total/64) words (all zero when there is none). */
int qgm_ref_mask_download(qgm_ctx* ctx, const qgm_ref* ref, uint64_t* mask_bits);
/* |P|: reference positions in P for q (windows inside a chromosome, not
 * masked) -- the P_size of mapping_quality. */
int qgm_ref_positions(qgm_ctx* ctx, qgm_ref* ref, uint32_t q, uint64_t* positions);
void qgm_ref_destroy(qgm_ref* ref);

/* ---- filtration: Alg. 2 -------------- */
/* Candidates over every chromosome, sorted by (read, strand, chrom, diagonal).
 * mode QGM_FILTER_FULL keeps the multiset (one per (p, p') pair, like
 * oracle::filter_hits, oracles.hpp:37-51); QGM_FILTER_RUN_START keeps the
 * leftmost q-gram of each run on a diagonal (identical candidate set). */
int qgm_filter(qgm_ctx* ctx, const qgm_index* idx, const qgm_reads* reads, const qgm_ref* ref, int strands,
               int mode, qgm_cands** out);
int qgm_cands_count(const qgm_cands* c, uint64_t* n);
int qgm_cands_download(qgm_ctx* ctx, const qgm_cands* c, qgm_candidate* out);
/* Unique candidates (dedup on (read, strand, chrom, diagonal)). */
int qgm_cands_unique(qgm_ctx* ctx, qgm_cands* c);
void qgm_cands_destroy(qgm_cands* c);

/* ---- validation: myers_banded / validate_hits ---------- */
/* One result per host candidate, in input order. */
int qgm_validate(qgm_ctx* ctx, const qgm_reads* reads, const qgm_ref* ref, const qgm_candidate* cands,
                 uint64_t n, uint32_t band_width, uint32_t pct_identity, qgm_validated* out);

/* ---- map: run_map core for one read buffer ------------- */
int qgm_map(qgm_ctx* ctx, const qgm_reads* reads, const qgm_ref* ref, const qgm_map_params* params,
            qgm_hits** out);
int qgm_hits_count(const qgm_hits* h, uint64_t* n);
int qgm_hits_stats(const qgm_hits* h, qgm_map_stats* out);
/* out: n records, host or device memory (a device destination keeps the
 * hits on the GPU, e.g. for the reference-sharded exchange over NCCL). */
int qgm_hits_download(qgm_ctx* ctx, const qgm_hits* h, qgm_hit* out);
/* hit_rank of every record, in download order: the number
 * of the read's records whose identity is >= the record's (edits <=). In
 * best-stratum mode that is the size of the read's best stratum. */
int qgm_hits_ranks(qgm_ctx* ctx, const qgm_hits* h, uint32_t* rank);
/* traceback_cigar (DESIGN.md section 2 item 9) of every record,
 * in download order: the oriented read against its chromosome from ref_start,
 * anchored start, free end, band |j - i| <= band_width - 1. ops[i * max_ops
 * + x] are BAM-style (length << 4 | op, M = 0, I = 1, D = 2). Fails with
 * QGM_ERR_INPUT if a record needs more than max_ops operations (out[].n_ops
 * then holds the counts). reads/ref must be the ones the hits were mapped
 * from. */
typedef struct qgm_cigar_info {
  uint32_t ref_start; /* alignment start; > the hit's ref_start when leading deletions were dropped */
  uint16_t n_ops;     /* CIGAR operations */
  uint16_t edits;     /* I + D + mismatched M columns (<= the hit's edits when its alignment is in the band) */
} qgm_cigar_info;
int qgm_hits_cigar(qgm_ctx* ctx, const qgm_hits* h, const qgm_reads* reads, const qgm_ref* ref,
                   uint32_t band_width, uint32_t max_ops, uint32_t* ops, qgm_cigar_info* out);
/* The same for host hit records (e.g. from qgm_map_host). */
int qgm_cigar_records(qgm_ctx* ctx, const qgm_reads* reads, const qgm_ref* ref, const qgm_hit* hits, uint64_t n,
                      uint32_t band_width, uint32_t max_ops, uint32_t* ops, qgm_cigar_info* out);
void qgm_hits_destroy(qgm_hits* h);
/* One call from host buffers to host hits: upload reads, build the index,
 * map, download (the e2e path). *n_out = hit count; if it exceeds cap the
 * call fails with QGM_ERR_INPUT and *n_out holds the required capacity. */
int qgm_map_host(qgm_ctx* ctx, const uint64_t* reads2bit, const uint32_t* lengths, uint32_t n_reads,
                 uint32_t stride, const qgm_ref* ref, const qgm_map_params* params, qgm_hit* out, uint64_t cap,
                 uint64_t* n_out, qgm_map_stats* stats);

/* One read buffer of a streamed run (run_map's bounded-queue pipeline,
 * SPEC.md:521-528 / PAPER.md:238-262). Host buffers; pinned memory lets the
 * copies overlap the mapping. */
#define QGM_READS_PADDED 0u /* qgm_pack_reads: ceil(stride/32) words per read */
#define QGM_READS_DENSE 1u  /* one 2-bit stream, read r = bases [r*stride, (r+1)*stride) (qgm_pack_codes) */
typedef struct qgm_batch {
  const uint64_t* reads2bit; /* layout below */
  const uint32_t* lengths;   /* NULL: every read has length `stride` */
  uint32_t n_reads;
  uint32_t stride;
  qgm_hit* out;              /* capacity `cap` records */
  uint64_t cap;
  uint64_t n_out;            /* out: hit count (the required capacity when it exceeds cap) */
  qgm_map_stats stats;       /* out */
  uint32_t layout;           /* QGM_READS_PADDED or QGM_READS_DENSE */
  uint32_t reserved;
} qgm_batch;
/* Maps the batches in order, same results as qgm_map_host per batch: the
 * reads of batch i+1 are uploaded on a second stream while batch i is
 * mapped, the hits of batch i are downloaded while batch i+1 is mapped.
 * Fails with QGM_ERR_INPUT if any batch's hits exceed its cap (every n_out is
 * still set). */
int qgm_map_host_batches(qgm_ctx* ctx, qgm_batch* batches, uint32_t n_batches, const qgm_ref* ref,
                         const qgm_map_params* params);

/* ---- data-parallel primitive: par::exclusive_scan (parallel.hpp:64-121) --- */
/* Device exclusive scan of host u32 values; QGM_ERR_INPUT on u32 overflow. */
int qgm_exclusive_scan_u32(qgm_ctx* ctx, const uint32_t* in, uint64_t n, uint32_t* out, uint32_t* total);

#ifdef __cplusplus
}
#endif
#endif /* QGM_C_H */
