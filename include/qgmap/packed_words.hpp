// packed_words.hpp -- host encoding of read sequences straight into the
// device's 2-bit read layout (the run_map ingestion path).
#pragma once

#include <array>
#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "qgmap/parallel.hpp"
#include "qgmap/seq.hpp"

namespace qgmap {

// Reads straight into the device's 2-bit layout (PackedReadText::pack():
// ceil(stride/32) MSB-first words per read) with encode_base's semantics --
// N (either case) becomes rng() & 3, drawn in read order exactly as
// pack_reads draws them, any other symbol is an input_error -- without the
// 1-byte code text and the valid-position list. Encoded in parallel over
// reads; the N bases are filled afterwards in order.
struct PackedWords {
  std::vector<std::uint64_t> words;
  std::vector<std::uint32_t> lengths;
  std::uint32_t stride = 0, W = 0;
};

inline PackedWords pack_words(const std::vector<std::string>& reads, std::uint32_t stride, rng_engine& rng,
                              unsigned threads = 0) {
  PackedWords pw;
  pw.stride = stride;
  pw.W = (stride + 31) / 32;
  const std::size_t n = reads.size();
  pw.words.assign(std::max<std::size_t>(1, n * pw.W), 0);
  pw.lengths.resize(n);
  static const auto table = [] {
    std::array<signed char, 256> t{};
    t.fill(-1);
    const char* sym = "ACGTN";
    for (int i = 0; i < 5; ++i) {
      t[static_cast<unsigned char>(sym[i])] = static_cast<signed char>(i);
      t[static_cast<unsigned char>(sym[i] - 'A' + 'a')] = static_cast<signed char>(i);
    }
    return t;
  }();
  std::vector<char> has_n(n, 0);
  std::atomic<std::size_t> bad{SIZE_MAX};
  par::parallel_for(n, threads, [&](std::size_t b, std::size_t e) {
    for (std::size_t r = b; r < e; ++r) {
      const std::string& s = reads[r];
      if (s.size() > stride) {
        std::size_t cur = bad.load();
        while (r < cur && !bad.compare_exchange_weak(cur, r)) {}
        continue;
      }
      pw.lengths[r] = std::uint32_t(s.size());
      std::uint64_t* w = pw.words.data() + r * pw.W;
      for (std::size_t j = 0; j < s.size(); ++j) {
        const int v = table[static_cast<unsigned char>(s[j])];
        if (v < 0) {
          std::size_t cur = bad.load();
          while (r < cur && !bad.compare_exchange_weak(cur, r)) {}
          break;
        }
        if (v == 4) has_n[r] = 1;
        else w[j >> 5] |= std::uint64_t(v) << (62 - 2 * (j & 31));
      }
    }
  });
  if (bad.load() != SIZE_MAX) {
    const std::string& s = reads[bad.load()];
    if (s.size() > stride)
      throw input_error("read of length " + std::to_string(s.size()) + " exceeds stride " + std::to_string(stride));
    for (char c : s)
      if (table[static_cast<unsigned char>(c)] < 0) throw input_error(std::string("unsupported base symbol '") + c + "'");
  }
  for (std::size_t r = 0; r < n; ++r) {  // N bases, in read order (pack_reads' rng order)
    if (!has_n[r]) continue;
    std::uint64_t* w = pw.words.data() + r * pw.W;
    const std::string& s = reads[r];
    for (std::size_t j = 0; j < s.size(); ++j)
      if (s[j] == 'N' || s[j] == 'n') w[j >> 5] |= std::uint64_t(random_base(rng)) << (62 - 2 * (j & 31));
  }
  return pw;
}

}  // namespace qgmap
