// qgmap/qgroup_index.hpp -- the q-group index, built on the B200.
//
// Source-compatible with the reference's proj/include/qgmap/qgroup_index.hpp
// (QGroupIndex<GroupWord>, build_qgroup_index, sample_group_starts,
// group_and_bit, grouprank, index_size_words; qgroup_index.hpp:28-213).
// build_qgroup_index runs the sm_100a build (index_build.cu) through
// qgm_index_build; the four arrays stay in HBM for filtration and are mirrored
// to host vectors lazily, on first use of an accessor, so code written against
// the reference's host vectors keeps working. The `threads` argument is
// accepted for source compatibility and ignored. Position order inside one
// occurrence interval is unspecified, as in the reference (:120-123).
#pragma once

#include <bit>
#include <cstdint>
#include <limits>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <sstream>
#include <string>
#include <vector>

#include "qgmap/device.hpp"
#include "qgmap/parallel.hpp"
#include "qgmap/seq.hpp"

namespace qgmap {

template <class GroupWord = std::uint32_t>
class QGroupIndex {
  static_assert(std::is_same_v<GroupWord, std::uint32_t> || std::is_same_v<GroupWord, std::uint64_t>,
                "group words are 32 or 64 bits");

 public:
  using group_word = GroupWord;
  static constexpr unsigned group_width = std::numeric_limits<GroupWord>::digits;

  QGroupIndex() = default;

  unsigned q() const { return info_.q; }
  bool sampled() const { return info_.sampled != 0; }
  std::size_t group_count() const { return info_.group_count; }
  std::size_t occurrence_count() const { return info_.occurrences; }
  std::size_t distinct_qgram_count() const { return info_.group_count ? info_.distinct : 0; }

  const std::vector<GroupWord>& occupancy() const { return mirror().I; }
  const std::vector<std::uint32_t>& group_starts() const { return mirror().S; }
  const std::vector<std::uint32_t>& occ_starts() const { return mirror().S1; }
  const std::vector<std::uint32_t>& positions() const { return mirror().O; }

  // Indexpair (qgroup_index.hpp:50-57): half-open interval of positions of g.
  std::optional<std::pair<std::uint32_t, std::uint32_t>> index_pair(qgram_code g) const {
    const auto& m = mirror();
    const std::size_t i = g / group_width;
    const unsigned j = g % group_width;
    const GroupWord word = m.I[i];
    if (word == 0 || !((word >> j) & GroupWord(1))) return std::nullopt;
    const std::uint32_t base = group_base(i) + rank_below(word, j);
    return std::make_pair(m.S1[base], m.S1[base + 1]);
  }

  std::span<const std::uint32_t> occurrences(qgram_code g) const {
    const auto p = index_pair(g);
    if (!p) return {};
    return {mirror().O.data() + p->first, p->second - p->first};
  }

  // Same text and FNV-1a checksums as the reference's debug_summary (:66-78).
  std::string debug_summary() const {
    auto fold = [](auto const& v) {
      std::uint64_t h = 1469598103934665603ull;
      for (auto x : v) { h ^= std::uint64_t(x); h *= 1099511628211ull; }
      return h;
    };
    const auto& m = mirror();
    std::ostringstream os;
    os << "occupancy len=" << m.I.size() << " sum=" << fold(m.I) << '\n'
       << "group_starts len=" << m.S.size() << " sum=" << fold(m.S) << '\n'
       << "occ_starts len=" << m.S1.size() << " sum=" << fold(m.S1) << '\n'
       << "positions len=" << m.O.size() << " sum=" << fold(m.O) << '\n';
    return os.str();
  }

  static std::uint32_t rank_below(GroupWord word, unsigned j) {
    const GroupWord mask = j == 0 ? GroupWord(0) : GroupWord(~GroupWord(0) >> (group_width - j));
    return std::uint32_t(std::popcount(GroupWord(word & mask)));
  }

  // Sort positions inside every interval on the device (byte-reproducible O).
  void normalize() {
    dev_.ctx->check(qgm_index_normalize(dev_.ctx->get(), dev_.get()));
    mirror_.reset();
    once_ = std::make_shared<std::once_flag>();
  }

  const device::IndexHandle& device_index() const { return dev_; }
  const device::ReadsHandle& device_reads() const { return reads_; }

  template <class W>
  friend QGroupIndex<W> build_qgroup_index(const PackedReadText&, unsigned);
  template <class W>
  friend QGroupIndex<W> sample_group_starts(const QGroupIndex<W>&);

 private:
  struct Mirror {
    std::vector<GroupWord> I;
    std::vector<std::uint32_t> S, S1, O;
  };

  const Mirror& mirror() const {
    std::call_once(*once_, [this] {
      auto m = std::make_shared<Mirror>();
      if (dev_) {
        m->I.resize(info_.group_count);
        m->S.resize(info_.group_starts_len);
        m->S1.resize(info_.distinct + 1);
        m->O.resize(info_.occurrences);
        dev_.ctx->check(qgm_index_download(dev_.ctx->get(), dev_.get(), m->I.data(), m->S.data(), m->S1.data(),
                                           m->O.data()));
      }
      mirror_ = m;
    });
    return *mirror_;
  }

  std::uint32_t group_base(std::size_t i) const {
    const auto& m = mirror();
    if (!sampled()) return m.S[i];
    const std::uint32_t even = m.S[i / 2];
    return (i & 1) ? even + std::uint32_t(std::popcount(m.I[i - 1])) : even;
  }

  void attach(device::IndexHandle h, device::ReadsHandle reads) {
    dev_ = std::move(h);
    reads_ = std::move(reads);
    dev_.ctx->check(qgm_index_info_get(dev_.get(), &info_));
  }

  device::IndexHandle dev_;
  device::ReadsHandle reads_;
  qgm_index_info info_{};
  mutable std::shared_ptr<std::once_flag> once_ = std::make_shared<std::once_flag>();
  mutable std::shared_ptr<Mirror> mirror_;
};

struct GroupCoords {
  std::size_t group;
  unsigned bit;
};

inline GroupCoords group_and_bit(qgram_code g, unsigned width) { return {g / width, unsigned(g % width)}; }

template <class GroupWord>
std::uint32_t grouprank(std::span<const GroupWord> occupancy, std::size_t group, unsigned bit) {
  return QGroupIndex<GroupWord>::rank_below(occupancy[group], bit);
}

// Alg. 1 on the device (index_build.cu). `threads` is ignored.
template <class GroupWord = std::uint32_t>
QGroupIndex<GroupWord> build_qgroup_index(const PackedReadText& text, unsigned threads = 1) {
  (void)threads;
  if (text.q == 0 || text.q > max_qgram_length)
    throw input_error("q must be in [1, " + std::to_string(max_qgram_length) + "]");
  auto ctx = device::Context::default_context();
  auto reads = device::upload_reads(text, ctx);
  qgm_index* ix = nullptr;
  ctx->check(qgm_index_build(ctx->get(), reads.get(), text.q, QGroupIndex<GroupWord>::group_width, 0, &ix));
  QGroupIndex<GroupWord> out;
  out.attach(device::IndexHandle(ctx, ix), reads);
  return out;
}

// sample_group_starts (qgroup_index.hpp:185-196): halved S; every lookup result
// is unchanged.
template <class GroupWord>
QGroupIndex<GroupWord> sample_group_starts(const QGroupIndex<GroupWord>& index) {
  if (!index.dev_ || index.sampled()) return index;
  auto ctx = index.dev_.ctx;
  qgm_index* ix = nullptr;
  ctx->check(qgm_index_sample(ctx->get(), index.dev_.get(), &ix));
  QGroupIndex<GroupWord> out;
  out.attach(device::IndexHandle(ctx, ix), index.reads_);
  return out;
}

struct IndexSize {
  std::uint64_t qgroup_words;
  std::uint64_t classic_words;
  double ratio;
};

// Word budget vs a flat q-gram index: 2/w*4^q +
// min(4^q,|T|) + |T| against 4^q + |T|.
inline IndexSize index_size_words(unsigned q, std::uint64_t text_len, unsigned width) {
  const std::uint64_t space = std::uint64_t(1) << (2 * q);
  const std::uint64_t qg = (2 * space + width - 1) / width + std::min(space, text_len) + text_len;
  const std::uint64_t cl = space + text_len;
  return {qg, cl, double(qg) / double(cl)};
}

}  // namespace qgmap
