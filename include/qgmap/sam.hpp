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
#include <numeric>
#include <ostream>
#include <string>
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

// One buffer of reads. hits sorted by read (map_reads order); ranks and
// aligns parallel to hits; quals may be empty (QUAL '*').
inline void write_sam_records(std::ostream& os, const std::vector<std::string>& names,
                              const std::vector<std::string>& seqs, const std::vector<std::string>& quals,
                              const std::vector<std::string>& chrom_names, const std::vector<MappedHit>& hits,
                              const std::vector<std::uint32_t>& ranks, const std::vector<Alignment>& aligns,
                              std::uint64_t p_size) {
  if (ranks.size() != hits.size() || aligns.size() != hits.size())
    throw input_error("write_sam_records: ranks/aligns do not match hits");
  std::size_t h = 0;
  std::vector<std::size_t> order;
  for (std::uint32_t r = 0; r < names.size(); ++r) {
    const std::string& seq = seqs[r];
    const std::string qual = r < quals.size() && !quals[r].empty() ? quals[r] : std::string("*");
    const std::size_t b = h;
    while (h < hits.size() && hits[h].read_id == r) ++h;
    if (h < hits.size() && hits[h].read_id < r) throw input_error("write_sam_records: hits not sorted by read");
    if (b == h) {
      os << names[r] << "\t4\t*\t0\t0\t*\t*\t0\t0\t" << seq << '\t' << qual << '\n';
      continue;
    }
    order.resize(h - b);
    std::iota(order.begin(), order.end(), b);
    std::sort(order.begin(), order.end(), [&](std::size_t x, std::size_t y) {
      const auto &a = hits[x], &c = hits[y];
      if (a.edits != c.edits) return a.edits < c.edits;
      if (a.chrom != c.chrom) return a.chrom < c.chrom;
      if (aligns[x].ref_start != aligns[y].ref_start) return aligns[x].ref_start < aligns[y].ref_start;
      return a.strand < c.strand;
    });
    for (std::size_t k = 0; k < order.size(); ++k) {
      const std::size_t i = order[k];
      const MappedHit& x = hits[i];
      const unsigned flag = (x.strand ? 0x10u : 0u) | (k ? 0x100u : 0u);
      os << names[r] << '\t' << flag << '\t' << chrom_names.at(x.chrom) << '\t' << (aligns[i].ref_start + 1) << '\t'
         << mapping_quality(ranks[i], p_size) << '\t' << aligns[i].cigar() << "\t*\t0\t0\t";
      if (x.strand) {
        os << reverse_complement(seq) << '\t';
        if (qual == "*") os << qual;
        else os << std::string(qual.rbegin(), qual.rend());
      } else {
        os << seq << '\t' << qual;
      }
      os << "\tNM:i:" << aligns[i].edits << '\n';
    }
  }
}

}  // namespace qgmap
