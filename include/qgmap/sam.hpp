// sam.hpp -- SAM emission (SPEC.md emit_sam, pipeline_cli module; PAPER.md
// §3.1 "streamed out in SAM format"). Host-side text formatting of the
// device results: hits (dedup + strata), hit ranks -> MAPQ, CIGARs.
//
// Per read: its records ordered by (edits, chromosome, position, strand) --
// score ties broken by (chromosome, position, strand) as SPEC's design
// decisions fix -- the first primary, the rest secondary (FLAG 0x100);
// reverse-strand records FLAG 0x10 with SEQ reverse-complemented and QUAL
// reversed; POS 1-based from the alignment's start; MAPQ = mapping_quality(R,
// |P|); NM = the alignment's edits. A read without records gets one unmapped
// record (FLAG 0x4).
#pragma once

#include <algorithm>
#include <array>
#include <charconv>
#include <numeric>
#include <ostream>
#include <string>
#include <thread>
#include <vector>

#include "qgmap/map.hpp"

namespace qgmap {

inline void write_sam_header(std::ostream& os, const std::vector<std::string>& chrom_names,
                             const std::vector<std::uint64_t>& chrom_begin, const std::string& cmdline = "") {
  os << "@HD\tVN:1.6\tSO:unsorted\n";
  for (std::size_t c = 0; c < chrom_names.size(); ++c)
    os << "@SQ\tSN:" << chrom_names[c] << "\tLN:" << (chrom_begin[c + 1] - chrom_begin[c]) << '\n';
  os << "@PG\tID:qgmap-b200\tPN:qgmap-b200";
  if (!cmdline.empty()) os << "\tCL:" << cmdline;
  os << '\n';
}

namespace detail {
inline void put_uint(std::string& o, std::uint64_t v) {
  char buf[24];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v);
  o.append(buf, r.ptr);
}
inline void put_cigar(std::string& o, const Alignment& a) {
  if (a.ops.empty()) {
    o += '*';
    return;
  }
  for (std::uint32_t x : a.ops) {
    put_uint(o, x >> 4);
    o += "MID"[x & 15];
  }
}
inline void put_revcomp(std::string& o, const std::string& s) {
  static const auto table = [] {
    std::array<char, 256> t{};
    t.fill('N');
    t['A'] = 'T'; t['a'] = 'T'; t['C'] = 'G'; t['c'] = 'G';
    t['G'] = 'C'; t['g'] = 'C'; t['T'] = 'A'; t['t'] = 'A';
    return t;
  }();
  const std::size_t at = o.size(), n = s.size();
  o.resize(at + n);
  char* d = o.data() + at;
  for (std::size_t i = 0; i < n; ++i) d[i] = table[static_cast<unsigned char>(s[n - 1 - i])];
}
inline void put_reversed(std::string& o, const std::string& s) {
  const std::size_t at = o.size();
  o.resize(at + s.size());
  std::reverse_copy(s.begin(), s.end(), o.begin() + std::ptrdiff_t(at));
}

// SAM text of reads [r0, r1) whose hits are [h0, h1)
inline void format_sam(std::string& o, std::uint32_t r0, std::uint32_t r1, std::size_t h0, std::size_t h1,
                       const std::vector<std::string>& names, const std::vector<std::string>& seqs,
                       const std::vector<std::string>& quals, const std::vector<std::string>& chrom_names,
                       const std::vector<MappedHit>& hits, const std::vector<std::uint32_t>& ranks,
                       const std::vector<Alignment>& aligns, std::uint64_t p_size) {
  std::size_t h = h0;
  std::vector<std::size_t> order;
  for (std::uint32_t r = r0; r < r1; ++r) {
    const std::string& seq = seqs[r];
    const bool has_q = r < quals.size() && !quals[r].empty();
    const std::size_t b = h;
    while (h < h1 && hits[h].read_id == r) ++h;
    if (b == h) {  // unmapped
      o += names[r];
      o += "\t4\t*\t0\t0\t*\t*\t0\t0\t";
      o += seq;
      o += '\t';
      if (has_q) o += quals[r];
      else o += '*';
      o += '\n';
      continue;
    }
    order.resize(h - b);
    std::iota(order.begin(), order.end(), b);
    std::sort(order.begin(), order.end(), [&](std::size_t x, std::size_t y) {
      const auto &p = hits[x], &q = hits[y];
      if (p.edits != q.edits) return p.edits < q.edits;
      if (p.chrom != q.chrom) return p.chrom < q.chrom;
      if (aligns[x].ref_start != aligns[y].ref_start) return aligns[x].ref_start < aligns[y].ref_start;
      return p.strand < q.strand;
    });
    for (std::size_t k = 0; k < order.size(); ++k) {
      const std::size_t i = order[k];
      const MappedHit& x = hits[i];
      o += names[r];
      o += '\t';
      put_uint(o, (x.strand ? 0x10u : 0u) | (k ? 0x100u : 0u));
      o += '\t';
      o += chrom_names.at(x.chrom);
      o += '\t';
      put_uint(o, std::uint64_t(aligns[i].ref_start) + 1);
      o += '\t';
      put_uint(o, mapping_quality(ranks[i], p_size));
      o += '\t';
      put_cigar(o, aligns[i]);
      o += "\t*\t0\t0\t";
      if (x.strand) {
        put_revcomp(o, seq);
        o += '\t';
        if (has_q) put_reversed(o, quals[r]);
        else o += '*';
      } else {
        o += seq;
        o += '\t';
        if (has_q) o += quals[r];
        else o += '*';
      }
      o += "\tNM:i:";
      put_uint(o, aligns[i].edits);
      o += '\n';
    }
  }
}
}  // namespace detail

// One buffer of reads. hits sorted by read (map_reads order); ranks and
// aligns parallel to hits; quals may be empty (QUAL '*'). The text is built
// in parallel over read ranges (threads = 0: hardware concurrency) and
// written in read order.
inline void write_sam_records(std::ostream& os, const std::vector<std::string>& names,
                              const std::vector<std::string>& seqs, const std::vector<std::string>& quals,
                              const std::vector<std::string>& chrom_names, const std::vector<MappedHit>& hits,
                              const std::vector<std::uint32_t>& ranks, const std::vector<Alignment>& aligns,
                              std::uint64_t p_size, unsigned threads = 0) {
  if (ranks.size() != hits.size() || aligns.size() != hits.size())
    throw input_error("write_sam_records: ranks/aligns do not match hits");
  for (std::size_t i = 1; i < hits.size(); ++i)
    if (hits[i].read_id < hits[i - 1].read_id) throw input_error("write_sam_records: hits not sorted by read");
  if (!hits.empty() && hits.back().read_id >= names.size()) throw input_error("write_sam_records: hit of an unknown read");
  const std::uint32_t n = std::uint32_t(names.size());
  unsigned T = threads ? threads : std::max(1u, std::thread::hardware_concurrency());
  T = std::max(1u, std::min<unsigned>(T, std::max<std::uint32_t>(1, n / 4096)));
  std::vector<std::string> parts(T);
  auto hit_begin = [&](std::uint32_t r) {  // first hit of read >= r
    return std::size_t(std::lower_bound(hits.begin(), hits.end(), r,
                                        [](const MappedHit& h, std::uint32_t v) { return h.read_id < v; }) -
                       hits.begin());
  };
  auto work = [&](unsigned t) {
    const std::uint32_t r0 = std::uint32_t(std::uint64_t(n) * t / T), r1 = std::uint32_t(std::uint64_t(n) * (t + 1) / T);
    parts[t].reserve(std::size_t(r1 - r0) * 2 * (seqs.empty() ? 64 : seqs[r0 < n ? r0 : 0].size() + 64));
    detail::format_sam(parts[t], r0, r1, hit_begin(r0), hit_begin(r1), names, seqs, quals, chrom_names, hits, ranks,
                       aligns, p_size);
  };
  if (T == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  for (const auto& s : parts) os.write(s.data(), std::streamsize(s.size()));
}

}  // namespace qgmap
