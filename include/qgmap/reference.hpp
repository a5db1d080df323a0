// qgmap/reference.hpp -- reference sequences for the device path: the sequence
// part of SPEC's ReferenceIndex (per-chromosome 2-bit
// sequences + the repeat mask). The q-gram-sorted P list of the spec is not
// needed: filtration streams every unmasked position of the packed reference.
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

  // Repeat mask: drop positions whose forward q-gram occurs
  // more than `threshold` times in its own chromosome.
  void mask_repeats(unsigned q, std::uint64_t threshold) {
    mask.assign(codes.size(), 0);
    for (std::uint32_t c = 0; c < chromosome_count(); ++c) {
      const std::uint64_t b = chrom_begin[c], L = length(c);
      if (L < q) continue;
      std::map<qgram_code, std::uint64_t> freq;
      for (std::uint64_t p = 0; p + q <= L; ++p) ++freq[encode_qgram({codes.data() + b + p, q})];
      for (std::uint64_t p = 0; p + q <= L; ++p)
        if (freq[encode_qgram({codes.data() + b + p, q})] > threshold) mask[b + p] = 1;
    }
  }
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
  qgm_ref* get() const { return h_.get(); }
  const std::shared_ptr<device::Context>& context() const { return h_.ctx; }
  const std::vector<std::uint64_t>& chrom_begin() const { return chrom_begin_; }

 private:
  device::RefHandle h_;
  std::vector<std::uint64_t> chrom_begin_;
};

}  // namespace qgmap
