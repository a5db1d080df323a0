// qgmap/reference.hpp -- reference sequences for the device path: the sequence
// part of SPEC's ReferenceIndex (per-chromosome 2-bit
// sequences + the repeat mask). The q-gram-sorted P list of the spec is built
// on the device by Reference::prepare (qgm_ref_prepare): one canonical q-group
// index over the unmasked positions of both strands, which the production
// filtration joins against the batch's code-sorted read q-grams (join.cu).
// Only references beyond 2^32 padded bases take the streaming k_filter path.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "qgmap/device.hpp"
#include "qgmap/seq.hpp"

namespace qgmap {

struct Reference {
  std::vector<std::string> names;
  std::vector<base_code> codes;            // concatenated chromosomes
  std::vector<std::uint64_t> chrom_begin;  // names.size()+1 offsets
  std::vector<std::uint8_t> mask;          // empty, or 1 byte per base (1 = not in P)

  std::uint32_t chromosome_count() const { return std::uint32_t(names.size()); }
  std::uint64_t length(std::uint32_t c) const { return chrom_begin[c + 1] - chrom_begin[c]; }

  void add_chromosome(std::string name, std::string_view seq, rng_engine& rng) {
    if (chrom_begin.empty()) chrom_begin.push_back(0);
    names.push_back(std::move(name));
    auto enc = encode_sequence(seq, rng);
    codes.insert(codes.end(), enc.begin(), enc.end());
    chrom_begin.push_back(codes.size());
    if (!mask.empty()) mask.resize(codes.size(), 0);
  }

  // The repeat mask is computed on the device:
  // DeviceReference::mask_repeats.
};

class DeviceReference {
 public:
  DeviceReference() = default;
  explicit DeviceReference(const Reference& ref,
                           std::shared_ptr<device::Context> ctx = device::Context::default_context())
      : chrom_begin_(ref.chrom_begin) {
    if (ref.chrom_begin.size() < 2) throw input_error("reference has no chromosome");
    std::vector<std::uint64_t> words((ref.codes.size() + 31) / 32 + 1, 0);
    pack_2bit(ref.codes, words.data());
    std::vector<std::uint64_t> mbits;
    if (!ref.mask.empty()) {
      mbits.assign((ref.codes.size() + 63) / 64 + 1, 0);
      for (std::size_t x = 0; x < ref.mask.size(); ++x)
        if (ref.mask[x]) mbits[x >> 6] |= std::uint64_t(1) << (x & 63);
    }
    qgm_ref* r = nullptr;
    ctx->check(qgm_ref_upload(ctx->get(), words.data(), ref.chrom_begin.data(),
                              std::uint32_t(ref.chrom_begin.size() - 1), mbits.empty() ? nullptr : mbits.data(), &r));
    h_ = device::RefHandle(ctx, r);
  }
  // Repeat mask on the device (qgm_ref_mask_repeats): positions whose forward
  // q-gram occurs more than `threshold` times in their chromosome leave P.
  void mask_repeats(unsigned q, std::uint64_t threshold = 1000) {
    context()->check(qgm_ref_mask_repeats(context()->get(), get(), q, threshold));
  }
  // |P| for q-grams of length q: unmasked positions of both strands (the
  // P_size of mapping_quality).
  std::uint64_t positions(unsigned q) const {
    std::uint64_t n = 0;
    context()->check(qgm_ref_positions(context()->get(), get(), q, &n));
    return n;
  }
  // The current mask, one byte per base (1 = not in P).
  std::vector<std::uint8_t> mask() const {
    const std::uint64_t total = chrom_begin_.back();
    std::vector<std::uint64_t> w((total + 63) / 64 + 1, 0);
    context()->check(qgm_ref_mask_download(context()->get(), get(), w.data()));
    std::vector<std::uint8_t> m(total);
    for (std::uint64_t x = 0; x < total; ++x) m[x] = std::uint8_t((w[x >> 6] >> (x & 63)) & 1u);
    return m;
  }
  qgm_ref* get() const { return h_.get(); }
  const std::shared_ptr<device::Context>& context() const { return h_.ctx; }
  const std::vector<std::uint64_t>& chrom_begin() const { return chrom_begin_; }

 private:
  device::RefHandle h_;
  std::vector<std::uint64_t> chrom_begin_;
};

}  // namespace qgmap
