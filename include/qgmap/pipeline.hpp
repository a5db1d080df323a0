// pipeline.hpp -- run_map (SPEC.md:531-539 pipeline_cli; Fig. 2):
// FASTQ in, SAM out, one read buffer at a time through the device path.
// The host parses and encodes buffer b+1 on a worker thread while the device
// maps buffer b (the paper's queue between the ingestion and mapping layers,
// capacity 1); the device side of each buffer is map_reads_ranked (index
// build .. strata), hit ranks and CIGARs.
#pragma once

#include <future>
#include <istream>
#include <ostream>
#include <random>

#include "qgmap/fastq.hpp"
#include "qgmap/sam.hpp"

namespace qgmap {

struct RunOptions {
  std::size_t batch_reads = 1 << 20;  // reads per buffer
  std::size_t batch_bases = SIZE_MAX; // bases per buffer
  std::uint64_t seed = 1;             // N replacement (encode_base) is deterministic under it
  std::string cmdline;                // @PG CL
};

struct RunStats {
  std::uint64_t reads = 0, records = 0, unmapped = 0, buffers = 0;
};

inline RunStats run_map(std::istream& fastq, std::ostream& sam, const Reference& ref, const DeviceReference& dref,
                        const MapParams& p, const RunOptions& opt = {}) {
  write_sam_header(sam, ref.names, ref.chrom_begin, opt.cmdline);
  const std::uint64_t p_size = dref.positions(p.q);
  FastqReader reader(fastq);
  rng_engine rng(opt.seed);
  struct Buffer {
    std::vector<FastqRecord> recs;
    PackedWords words;  // the device read layout, straight from the sequences
  };
  auto load = [&]() {  // parse + encode one buffer (worker thread; rng used only here)
    Buffer b;
    b.recs = reader.next_batch(opt.batch_reads, opt.batch_bases);
    std::vector<std::string> seqs;
    seqs.reserve(b.recs.size());
    std::uint32_t stride = 1;
    for (const auto& r : b.recs) {
      seqs.push_back(r.seq);
      stride = std::max<std::uint32_t>(stride, std::uint32_t(r.seq.size()));
    }
    b.words = pack_words(seqs, stride, rng);
    return b;
  };
  RunStats st;
  std::future<Buffer> next = std::async(std::launch::async, load);
  while (true) {
    Buffer cur = next.get();
    if (cur.recs.empty()) break;
    next = std::async(std::launch::async, load);
    std::vector<std::uint32_t> ranks;
    std::vector<Alignment> aligns;
    const auto hits = map_packed_reads(dref, cur.words, p, nullptr, &ranks, &aligns);
    std::vector<std::string> names, seqs, quals;
    names.reserve(cur.recs.size());
    for (auto& r : cur.recs) {
      names.push_back(std::move(r.name));
      seqs.push_back(std::move(r.seq));
      quals.push_back(std::move(r.qual));
    }
    write_sam_records(sam, names, seqs, quals, ref.names, hits, ranks, aligns, p_size);
    ++st.buffers;
    st.reads += names.size();
    st.records += hits.size();
    std::vector<char> seen(names.size(), 0);
    for (const auto& h : hits) seen[h.read_id] = 1;
    for (char x : seen) st.unmapped += !x;
  }
  st.records += st.unmapped;
  return st;
}

}  // namespace qgmap
