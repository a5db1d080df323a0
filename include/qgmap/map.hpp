// qgmap/map.hpp -- filter / validate / map entry points of the B200 mapper
// (the spec-only modules of SPEC.md: filtration :318-361, validation
// :363-420, postprocess strata :422-472, run_map core :531-539), as thin
// C++ wrappers of include/qgm_c.h.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "qgmap/packed_words.hpp"
#include "qgmap/qgroup_index.hpp"
#include "qgmap/reference.hpp"

namespace qgmap {

// ------------------------------------------------------------- filtration
// Hit extended with the strand and chromosome of the
// streamed reference q-gram. d = p - (p' mod m) on the forward strand
// (Alg. 2 line 12); d = p + o + q - n for a reverse-complement match.
struct Hit {
  std::int64_t d;
  std::uint32_t r;
  std::uint32_t chrom;
  std::uint8_t strand;
  auto operator<=>(const Hit&) const = default;
};

// full / run_start: stream the reference against the read index (filter.cu);
// *_join: bucket-ordered join of the read q-grams with the reference q-group
// indexes (join.cu, the path qgm_map uses). All four give the same candidate set.
// full / run_start: the join below 2^32 padded reference bases, else the
// streaming kernel; *_join / *_stream force either (same candidates).
enum class FilterMode {
  full = QGM_FILTER_FULL,
  run_start = QGM_FILTER_RUN_START,
  full_join = QGM_FILTER_FULL | QGM_FILTER_JOIN,
  run_start_join = QGM_FILTER_RUN_START | QGM_FILTER_JOIN,
  full_stream = QGM_FILTER_FULL | QGM_FILTER_STREAM,
  run_start_stream = QGM_FILTER_RUN_START | QGM_FILTER_STREAM
};

// filter_reference over every unmasked reference position of
// every chromosome, both strands by default. Sorted by (r, strand, chrom, d).
template <class W>
std::vector<Hit> filter_reference(const DeviceReference& ref, const QGroupIndex<W>& index,
                                  FilterMode mode = FilterMode::full, int strands = QGM_STRAND_BOTH,
                                  bool unique = false) {
  auto ctx = index.device_index().ctx;
  qgm_cands* c = nullptr;
  ctx->check(qgm_filter(ctx->get(), index.device_index().get(), index.device_reads().get(), ref.get(), strands,
                        int(mode), &c));
  std::unique_ptr<qgm_cands, void (*)(qgm_cands*)> guard(c, qgm_cands_destroy);
  if (unique) ctx->check(qgm_cands_unique(ctx->get(), c));
  std::uint64_t n = 0;
  ctx->check(qgm_cands_count(c, &n));
  std::vector<qgm_candidate> raw(n);
  ctx->check(qgm_cands_download(ctx->get(), c, raw.data()));
  std::vector<Hit> out(n);
  for (std::uint64_t i = 0; i < n; ++i)
    out[i] = {raw[i].diagonal, raw[i].read_id, raw[i].chrom, std::uint8_t(raw[i].strand)};
  return out;
}

// ------------------------------------------------------------- validation
struct BandConfig {
  unsigned band_width = 32;
  double identity_threshold = 0.80;
  unsigned percent() const { return unsigned(std::lround(identity_threshold * 100.0)); }
};

struct ValidatedHit {
  std::uint32_t r;
  std::uint32_t chrom;
  std::uint32_t ref_start;
  int k;
  double identity;
  std::int64_t d;
  std::uint8_t strand;
};

// validate_hits: one ValidatedHit per input hit whose
// identity (n-k)/n reaches the threshold (integer test 100(n-k) >= pct*n).
template <class W>
std::vector<ValidatedHit> validate_hits(const std::vector<Hit>& hits, const QGroupIndex<W>& index,
                                        const PackedReadText& text, const DeviceReference& ref,
                                        BandConfig band = {}) {
  auto ctx = index.device_index().ctx;
  std::vector<qgm_candidate> in(hits.size());
  for (std::size_t i = 0; i < hits.size(); ++i) in[i] = {hits[i].d, hits[i].r, hits[i].chrom, hits[i].strand, 0};
  std::vector<qgm_validated> res(hits.size());
  ctx->check(qgm_validate(ctx->get(), index.device_reads().get(), ref.get(), in.data(), in.size(), band.band_width,
                          band.percent(), res.data()));
  std::vector<ValidatedHit> out;
  for (std::size_t i = 0; i < hits.size(); ++i) {
    if (!res[i].kept || !res[i].in_range) continue;
    const double n = double(text.read_lengths[hits[i].r]);
    out.push_back({hits[i].r, hits[i].chrom, res[i].ref_start, res[i].edits, (n - res[i].edits) / n, hits[i].d,
                   hits[i].strand});
  }
  return out;
}

struct MyersResult {
  int k;
  unsigned start_offset;
};

// myers_banded for one read and one window; the band width
// is implied by the window: B = |window| - |read| + 1 (1..64).
inline MyersResult myers_banded(std::span<const base_code> read, std::span<const base_code> window,
                                std::shared_ptr<device::Context> ctx = device::Context::default_context()) {
  if (read.empty() || window.size() < read.size() || window.size() - read.size() + 1 > 64)
    throw input_error("myers_banded: need 1 <= |window| - |read| + 1 <= 64");
  const unsigned B = unsigned(window.size() - read.size() + 1);
  Reference R;
  R.names = {"window"};
  R.codes.assign(window.begin(), window.end());
  R.chrom_begin = {0, window.size()};
  DeviceReference dref(R, ctx);
  std::vector<std::vector<base_code>> one{std::vector<base_code>(read.begin(), read.end())};
  auto text = pack_encoded_reads(one, std::uint32_t(read.size()), 1);
  auto reads = device::upload_reads(text, ctx);
  const qgm_candidate c{std::int64_t((B - 1) / 2), 0, 0, 0, 0};
  qgm_validated v{};
  ctx->check(qgm_validate(ctx->get(), reads.get(), dref.get(), &c, 1, B, 0, &v));
  return {v.edits, v.start};
}

// ------------------------------------------------------------- map
enum class StratumMode { best_stratum = QGM_MODE_BEST_STRATUM, all = QGM_MODE_ALL };

struct MapParams {
  unsigned q = 16;
  unsigned group_width = 32;
  bool sampled = false;
  BandConfig band{};
  StratumMode mode = StratumMode::best_stratum;
  int strands = QGM_STRAND_BOTH;
};

struct MappedHit {
  std::uint32_t read_id, chrom, ref_start;
  std::uint16_t edits;
  std::uint8_t strand;
  auto operator<=>(const MappedHit&) const = default;
};

// mapping_quality: min{-10 log10((R-1)/|P|),
// 255}, R = 1 -> 255, rounded half up, floored at 0. Host floating point: the
// quality is reported, never compared bit-exactly.
inline unsigned mapping_quality(std::uint32_t rank, std::uint64_t p_size) {
  if (rank <= 1) return 255;
  const double q = -10.0 * std::log10(double(rank - 1) / double(p_size ? p_size : 1));
  const double r = std::floor(std::min(q, 255.0) + 0.5);
  return r < 0 ? 0u : unsigned(r);
}

// traceback_cigar (DESIGN.md section 2 item 9) of one record:
// the alignment's start (leading deletions dropped), its edits and the CIGAR
// as BAM-style ops (length << 4 | op, M = 0, I = 1, D = 2).
struct Alignment {
  std::uint32_t ref_start = 0;
  std::uint16_t edits = 0;
  std::vector<std::uint32_t> ops;
  std::string cigar() const {
    std::string o;
    for (std::uint32_t x : ops) o += std::to_string(x >> 4) + "MID"[x & 15];
    return o.empty() ? "*" : o;
  }
  std::uint32_t ref_span() const {  // reference bases consumed (M and D)
    std::uint32_t s = 0;
    for (std::uint32_t x : ops) s += (x & 15) != 1 ? x >> 4 : 0;
    return s;
  }
};

namespace detail {
inline std::vector<Alignment> unpack_alignments(const std::vector<std::uint32_t>& ops,
                                                const std::vector<qgm_cigar_info>& info, std::uint32_t max_ops) {
  std::vector<Alignment> out(info.size());
  for (std::size_t i = 0; i < info.size(); ++i) {
    out[i].ref_start = info[i].ref_start;
    out[i].edits = info[i].edits;
    out[i].ops.assign(ops.begin() + std::ptrdiff_t(i * max_ops), ops.begin() + std::ptrdiff_t(i * max_ops + info[i].n_ops));
  }
  return out;
}
// Calls fn(max_ops, ops, info) until every record fits: the first try
// assumes 2 * band + 16 operations (any hit the validation keeps at 80%
// identity), a record needing more is retried once with enough.
template <class Fn>
std::vector<Alignment> run_cigar(const device::Context& ctx, std::uint64_t n, unsigned band, Fn&& fn) {
  std::uint32_t max_ops = 2 * band + 16;
  for (int attempt = 0;; ++attempt) {
    std::vector<std::uint32_t> ops(std::max<std::uint64_t>(n * max_ops, 1));
    std::vector<qgm_cigar_info> info(n);
    const int st = fn(max_ops, ops.data(), info.data());
    if (st == QGM_OK) return unpack_alignments(ops, info, max_ops);
    std::uint32_t need = 0;
    for (const auto& x : info) need = std::max<std::uint32_t>(need, x.n_ops);
    if (st != QGM_ERR_INPUT || need <= max_ops || attempt > 0) ctx.check(st);
    max_ops = need;
  }
}
}  // namespace detail

// One read buffer against the whole reference: index build, filtration,
// candidate dedup, validation, dedup + strata -- all on the device. Output
// sorted by (read, chrom, ref_start, strand); with `ranks`, also the
// hit_rank R of every record.
namespace detail {
inline std::vector<MappedHit> map_uploaded(const DeviceReference& ref, const device::ReadsHandle& reads,
                                           const MapParams& p, qgm_map_stats* stats,
                                           std::vector<std::uint32_t>* ranks, std::vector<Alignment>* aligns) {
  auto ctx = ref.context();
  const qgm_map_params mp{p.q, p.group_width, p.sampled ? 1u : 0u, p.band.band_width, p.band.percent(),
                          unsigned(p.mode), unsigned(p.strands), 0};
  qgm_hits* h = nullptr;
  ctx->check(qgm_map(ctx->get(), reads.get(), ref.get(), &mp, &h));
  std::unique_ptr<qgm_hits, void (*)(qgm_hits*)> guard(h, qgm_hits_destroy);
  std::uint64_t n = 0;
  ctx->check(qgm_hits_count(h, &n));
  if (stats) ctx->check(qgm_hits_stats(h, stats));
  std::vector<qgm_hit> raw(n);
  ctx->check(qgm_hits_download(ctx->get(), h, raw.data()));
  std::vector<MappedHit> out(n);
  for (std::uint64_t i = 0; i < n; ++i)
    out[i] = {raw[i].read_id, raw[i].chrom, raw[i].ref_start, raw[i].edits, raw[i].strand};
  if (ranks) {
    ranks->assign(n, 0);
    ctx->check(qgm_hits_ranks(ctx->get(), h, ranks->data()));
  }
  if (aligns) {  // CIGAR of every record while the reads are on the device
    *aligns = run_cigar(*ctx, n, p.band.band_width,
                        [&](std::uint32_t max_ops, std::uint32_t* ops, qgm_cigar_info* info) {
                          return qgm_hits_cigar(ctx->get(), h, reads.get(), ref.get(), p.band.band_width, max_ops,
                                                ops, info);
                        });
  }
  return out;
}
}  // namespace detail

inline std::vector<MappedHit> map_reads_ranked(const DeviceReference& ref, const PackedReadText& text,
                                               const MapParams& p, qgm_map_stats* stats,
                                               std::vector<std::uint32_t>* ranks,
                                               std::vector<Alignment>* aligns = nullptr) {
  return detail::map_uploaded(ref, device::upload_reads(text, ref.context()), p, stats, ranks, aligns);
}

// The same for reads already in the device's 2-bit layout (pack_words): no
// 1-byte codes or position list on the host.
inline std::vector<MappedHit> map_packed_reads(const DeviceReference& ref, const PackedWords& pw, const MapParams& p,
                                               qgm_map_stats* stats = nullptr,
                                               std::vector<std::uint32_t>* ranks = nullptr,
                                               std::vector<Alignment>* aligns = nullptr) {
  auto ctx = ref.context();
  qgm_reads* r = nullptr;
  ctx->check(qgm_reads_upload(ctx->get(), pw.words.data(), pw.lengths.data(), std::uint32_t(pw.lengths.size()),
                              pw.stride, &r));
  return detail::map_uploaded(ref, device::ReadsHandle(ctx, r), p, stats, ranks, aligns);
}

inline std::vector<MappedHit> map_reads(const DeviceReference& ref, const PackedReadText& text,
                                        const MapParams& p = {}, qgm_map_stats* stats = nullptr) {
  return map_reads_ranked(ref, text, p, stats, nullptr);
}

}  // namespace qgmap
