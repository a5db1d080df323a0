// run_map (include/qgmap/pipeline.hpp): FASTQ in, SAM out through the device
// path -- SPEC.md run_map / emit_sam examples and invariants (every read
// yields a record; CIGAR consumes the read; NM equals the alignment's edits;
// pipeline/serial equivalence; determinism under a fixed seed).
#include <catch2/catch_amalgamated.hpp>

#include <map>
#include <regex>
#include <sstream>

#include "qgmap/pipeline.hpp"
#include "testutil.hpp"

using namespace qgmap;

namespace {
std::string decode(const std::vector<base_code>& c, std::size_t b, std::size_t n) {
  std::string s;
  for (std::size_t i = b; i < b + n; ++i) s += decode_base(c[i]);
  return s;
}
std::vector<std::vector<std::string>> sam_records(const std::string& sam) {
  std::vector<std::vector<std::string>> out;
  std::istringstream in(sam);
  std::string l;
  while (std::getline(in, l)) {
    if (l.empty() || l[0] == '@') continue;
    std::vector<std::string> f;
    std::istringstream ls(l);
    std::string x;
    while (std::getline(ls, x, '\t')) f.push_back(x);
    out.push_back(f);
  }
  return out;
}
struct Fixture {
  Reference ref;
  std::string chrom;
  Fixture() {
    std::mt19937_64 g(7);
    auto codes = tu::random_codes(5000, g);
    // an exact 120-base duplicate: reads inside it have two equal hits
    std::copy(codes.begin() + 3000, codes.begin() + 3120, codes.begin() + 4200);
    chrom = decode(codes, 0, codes.size());
    rng_engine rng(1);
    ref.add_chromosome("chr1", chrom, rng);
    auto c2 = tu::random_codes(3000, g);
    ref.add_chromosome("chr2", decode(c2, 0, c2.size()), rng);
  }
};
MapParams params(StratumMode mode) {
  MapParams p;
  p.q = 12;
  p.mode = mode;
  return p;
}
}  // namespace

TEST_CASE("run_map: SPEC emit_sam examples through the device") {
  Fixture fx;
  DeviceReference dref(fx.ref);
  const std::string fwd = fx.chrom.substr(10, 60);
  const std::string rev = reverse_complement(fx.chrom.substr(700, 60));
  const std::string dup = fx.chrom.substr(3030, 60);
  std::string rnd;
  std::mt19937_64 g(99);
  for (int i = 0; i < 60; ++i) rnd += "ACGT"[g() & 3];
  std::ostringstream fq;
  fq << "@fwd\n" << fwd << "\n+\n" << std::string(60, 'I') << "\n";
  fq << "@rev\n" << rev << "\n+\n" << std::string(59, 'I') << "#\n";
  fq << "@dup\n" << dup << "\n+\n" << std::string(60, 'I') << "\n";
  fq << "@rnd\n" << rnd << "\n+\n" << std::string(60, 'I') << "\n";
  std::istringstream in(fq.str());
  std::ostringstream out;
  const RunStats st = run_map(in, out, fx.ref, dref, params(StratumMode::all));
  CHECK(st.reads == 4);
  const auto R = sam_records(out.str());
  REQUIRE(R.size() == 5);
  // exact forward unique hit at internal position 10 -> POS 11, FLAG 0, MAPQ 255
  CHECK(R[0][0] == "fwd");
  CHECK(R[0][1] == "0");
  CHECK(R[0][2] == "chr1");
  CHECK(R[0][3] == "11");
  CHECK(R[0][4] == "255");
  CHECK(R[0][5] == "60M");
  CHECK(R[0][11] == "NM:i:0");
  // reverse strand -> FLAG 0x10, SEQ reverse-complemented, QUAL reversed
  CHECK(R[1][1] == "16");
  CHECK(R[1][3] == "701");
  CHECK(R[1][9] == fx.chrom.substr(700, 60));
  CHECK(R[1][10] == "#" + std::string(59, 'I'));
  // two equal-identity hits: one primary + one secondary (0x100)
  CHECK(R[2][0] == "dup");
  CHECK(R[3][0] == "dup");
  CHECK(R[2][1] == "0");
  CHECK(R[3][1] == "256");
  CHECK(R[2][3] == "3031");
  CHECK(R[3][3] == "4231");
  CHECK(R[2][4] == R[3][4]);
  CHECK(R[2][4] != "255");
  // no hit -> unmapped record
  CHECK(R[4][0] == "rnd");
  CHECK(R[4][1] == "4");
}

TEST_CASE("run_map: empty FASTQ gives the header only") {
  Fixture fx;
  DeviceReference dref(fx.ref);
  std::istringstream in("");
  std::ostringstream out;
  const RunStats st = run_map(in, out, fx.ref, dref, params(StratumMode::best_stratum));
  CHECK(st.reads == 0);
  CHECK(out.str() == "@HD\tVN:1.6\tSO:unsorted\n@SQ\tSN:chr1\tLN:5000\n@SQ\tSN:chr2\tLN:3000\n"
                     "@PG\tID:qgmap-b200\tPN:qgmap-b200\n");
}

TEST_CASE("run_map: every read has a record, CIGARs are consistent, buffering does not change the output") {
  Fixture fx;
  DeviceReference dref(fx.ref);
  std::mt19937_64 g(5);
  std::vector<base_code> all;
  for (char ch : fx.chrom) all.push_back(base_code(std::string("ACGT").find(ch)));
  std::ostringstream fq;
  const int n = 300;
  for (int r = 0; r < n; ++r) {
    const std::size_t len = 40 + g() % 80, pos = g() % (all.size() - len - 10);
    auto rd = tu::sample_read(all, pos, len, 0.04, g() & 1, g);
    std::string s;
    for (auto c : rd) s += decode_base(c);
    if (r % 37 == 0) s = std::string(len, 'N');  // all-N reads: seeded random bases
    fq << "@r" << r << "\n" << s << "\n+\n" << std::string(s.size(), 'F') << "\n";
  }
  auto run = [&](std::size_t batch, std::uint64_t seed) {
    std::istringstream in(fq.str());
    std::ostringstream out;
    RunOptions o;
    o.batch_reads = batch;
    o.seed = seed;
    run_map(in, out, fx.ref, dref, params(StratumMode::all), o);
    return out.str();
  };
  const std::string a = run(1 << 20, 3);
  CHECK(a == run(1 << 20, 3));  // deterministic under the seed (N replacement)
  const auto R = sam_records(a);
  std::map<std::string, int> per_read;
  for (const auto& f : R) per_read[f[0]]++;
  CHECK(per_read.size() == std::size_t(n));
  const std::regex op("(\\d+)([MID])");
  std::size_t mapped = 0;
  for (const auto& f : R) {
    if (f[1] == "4") continue;
    ++mapped;
    std::size_t rd = 0, rf = 0;
    for (std::sregex_iterator it(f[5].begin(), f[5].end(), op), e; it != e; ++it) {
      const std::size_t l = std::stoul((*it)[1]);
      const char o = (*it)[2].str()[0];
      if (o != 'D') rd += l;
      if (o != 'I') rf += l;
    }
    CHECK(rd == f[9].size());  // CIGAR consumes the read
    const std::uint64_t pos = std::stoull(f[3]) - 1;
    const std::uint64_t len = fx.ref.length(f[2] == "chr1" ? 0 : 1);
    CHECK(pos + rf <= len);    // and stays inside the chromosome
  }
  CHECK(mapped > std::size_t(n) * 8 / 10);
  // buffers of 7 reads (many device calls, the parser thread always ahead)
  // give the same records as one buffer once the seeded N reads are left out
  auto strip_n = [&](const std::string& sam) {
    std::vector<std::vector<std::string>> v;
    for (auto& f : sam_records(sam))
      if (std::stoi(f[0].substr(1)) % 37 != 0) v.push_back(f);
    return v;
  };
  CHECK(strip_n(run(7, 3)) == strip_n(a));
}

TEST_CASE("map_packed_reads(pack_words) equals map_reads(pack_reads) for the same seed, CIGARs included") {
  Fixture fx;
  DeviceReference dref(fx.ref);
  std::mt19937_64 g(9);
  std::vector<base_code> all;
  for (char ch : fx.chrom) all.push_back(base_code(std::string("ACGT").find(ch)));
  std::vector<std::string> seqs;
  for (int r = 0; r < 500; ++r) {
    const std::size_t len = 30 + g() % 90, pos = g() % (all.size() - len - 10);
    auto rd = tu::sample_read(all, pos, len, 0.04, g() & 1, g);
    std::string s;
    for (auto c : rd) s += decode_base(c);
    if (r % 9 == 0) s[g() % s.size()] = 'N';
    seqs.push_back(s);
  }
  MapParams p = params(StratumMode::all);
  rng_engine a(5), b(5);
  const auto text = pack_reads(seqs, 120, p.q, a);
  const auto pw = pack_words(seqs, 120, b);
  std::vector<std::uint32_t> ra, rb;
  std::vector<Alignment> aa, ab;
  const auto ha = map_reads_ranked(dref, text, p, nullptr, &ra, &aa);
  const auto hb = map_packed_reads(dref, pw, p, nullptr, &rb, &ab);
  REQUIRE(ha.size() > 400);
  CHECK(ha == hb);
  CHECK(ra == rb);
  REQUIRE(aa.size() == ab.size());
  for (std::size_t i = 0; i < aa.size(); ++i) {
    CHECK(aa[i].cigar() == ab[i].cigar());
    CHECK(aa[i].ref_start == ab[i].ref_start);
  }
}
