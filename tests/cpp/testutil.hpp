// Shared helpers of the C++ parity tests: seeded synthetic inputs and
// conversions between the B200 API (include/qgmap) and the CPU oracle
// (oracle/qgm_oracle.hpp, test infrastructure).
#pragma once

#include <algorithm>
#include <random>
#include <string>
#include <vector>

#include "qgm_oracle.hpp"
#include "qgmap/map.hpp"

namespace tu {

using qgmap::base_code;

inline std::vector<base_code> random_codes(std::size_t n, std::mt19937_64& g) {
  std::vector<base_code> v(n);
  for (auto& c : v) c = base_code(g() & 3u);
  return v;
}

// Read sampled from `src` at `pos` with ~err edits per base (sub/ins/del),
// optionally reverse complemented; exactly `len` bases.
inline std::vector<base_code> sample_read(const std::vector<base_code>& src, std::size_t pos, std::size_t len,
                                          double err, bool rc, std::mt19937_64& g) {
  std::uniform_real_distribution<double> U(0, 1);
  std::vector<base_code> out;
  std::size_t p = pos;
  while (out.size() < len) {
    const double u = U(g);
    const base_code b = p < src.size() ? src[p] : base_code(g() & 3u);
    if (u < err * 0.8) { out.push_back(base_code((b + 1 + g() % 3) & 3)); ++p; }
    else if (u < err * 0.9) out.push_back(base_code(g() & 3u));
    else if (u < err) ++p;
    else { out.push_back(b); ++p; }
  }
  if (rc) out = qgmap::reverse_complement(std::span<const base_code>(out));
  return out;
}

struct Instance {
  qgmap::Reference ref;
  qgmap::PackedReadText text;
  qgm_oracle::RefSet oref;
  qgm_oracle::ReadSet oreads;
};

// n_chrom random chromosomes (some shorter than a read), n_reads reads of
// length in [lmin, lmax] (stride = lmax), drawn from the chromosomes or random.
inline Instance make_instance(std::mt19937_64& g, unsigned n_chrom, std::size_t chrom_len, unsigned n_reads,
                              unsigned lmin, unsigned lmax, double err, unsigned q, bool mask = false,
                              unsigned mask_threshold = 4) {
  Instance in;
  in.ref.chrom_begin.push_back(0);
  for (unsigned c = 0; c < n_chrom; ++c) {
    const std::size_t L = (c % 3 == 2) ? std::size_t(g() % (lmax + 8)) : chrom_len / 2 + g() % (chrom_len / 2 + 1);
    auto s = random_codes(L, g);
    if (c % 4 == 1 && L > 200) {  // a few exact repeats to create multi-hits
      for (int rep = 0; rep < 3; ++rep) {
        const std::size_t a = g() % (L - 100), b = g() % (L - 100);
        std::copy(s.begin() + a, s.begin() + a + 80, s.begin() + b);
      }
    }
    in.ref.names.push_back("chr" + std::to_string(c));
    in.ref.codes.insert(in.ref.codes.end(), s.begin(), s.end());
    in.ref.chrom_begin.push_back(in.ref.codes.size());
  }
  if (mask) in.ref.mask = qgm_oracle::repeat_mask(in.ref.codes, in.ref.chrom_begin, q, mask_threshold);
  std::vector<std::vector<base_code>> reads;
  for (unsigned r = 0; r < n_reads; ++r) {
    const unsigned len = lmin + unsigned(g() % (lmax - lmin + 1));
    const unsigned c = unsigned(g() % n_chrom);
    const std::size_t L = in.ref.length(c);
    if (L > len + 40 && g() % 8 != 0) {
      std::vector<base_code> chrom(in.ref.codes.begin() + std::ptrdiff_t(in.ref.chrom_begin[c]),
                                   in.ref.codes.begin() + std::ptrdiff_t(in.ref.chrom_begin[c + 1]));
      reads.push_back(sample_read(chrom, g() % (L - len - 20), len, err, g() & 1, g));
    } else {
      reads.push_back(random_codes(len, g));
    }
  }
  in.text = qgmap::pack_encoded_reads(reads, lmax, q);
  in.oref.codes = in.ref.codes;
  in.oref.chrom_begin = in.ref.chrom_begin;
  in.oref.mask = in.ref.mask;
  in.oreads.codes = in.text.codes;
  in.oreads.stride = in.text.stride;
  in.oreads.lengths = in.text.read_lengths;
  return in;
}

inline std::vector<qgm_oracle::Cand> to_oracle(const std::vector<qgmap::Hit>& h) {
  std::vector<qgm_oracle::Cand> out(h.size());
  for (std::size_t i = 0; i < h.size(); ++i) out[i] = {h[i].r, h[i].chrom, h[i].d, h[i].strand};
  return out;
}

inline std::vector<qgm_oracle::Hit> to_oracle(const std::vector<qgmap::MappedHit>& h) {
  std::vector<qgm_oracle::Hit> out(h.size());
  for (std::size_t i = 0; i < h.size(); ++i)
    out[i] = {h[i].read_id, h[i].chrom, h[i].ref_start, h[i].edits, h[i].strand};
  return out;
}

inline std::vector<std::uint32_t> sort_intervals(std::vector<std::uint32_t> O, const std::vector<std::uint32_t>& S1) {
  for (std::size_t b = 0; b + 1 < S1.size(); ++b) std::sort(O.begin() + S1[b], O.begin() + S1[b + 1]);
  return O;
}

}  // namespace tu
