// FASTQ ingestion (include/qgmap/fastq.hpp) and SAM formatting of given
// records (include/qgmap/sam.hpp) -- host only, no device calls: run by the
// CPU suite (tests/test_host_io.py).
#include <catch2/catch_amalgamated.hpp>

#include <sstream>

#include "qgmap/fastq.hpp"
#include "qgmap/packed_words.hpp"
#include "qgmap/sam.hpp"

using namespace qgmap;

TEST_CASE("FASTQ records, CRLF, blank lines and comments") {
  std::istringstream in("@r1 some comment\nACGTN\n+\nIIIII\n\n@r2\r\nGG\r\n+r2\r\n!!\r\n");
  FastqReader rd(in);
  FastqRecord r;
  REQUIRE(rd.next(r));
  CHECK(r.name == "r1");
  CHECK(r.seq == "ACGTN");
  CHECK(r.qual == "IIIII");
  REQUIRE(rd.next(r));
  CHECK(r.name == "r2");
  CHECK(r.seq == "GG");
  CHECK(r.qual == "!!");
  CHECK_FALSE(rd.next(r));
  CHECK(rd.records() == 2);
}

TEST_CASE("FASTQ malformed input is an input_error") {
  for (const char* bad : {"r1\nACGT\n+\nIIII\n", "@r1\nACGT\n-\nIIII\n", "@r1\nACGT\n+\nIII\n", "@r1\nACGT\n+\n"}) {
    std::istringstream in(bad);
    FastqReader rd(in);
    FastqRecord r;
    CHECK_THROWS_AS(rd.next(r), input_error);
  }
}

TEST_CASE("FASTQ buffers fill by reads or by bases") {
  std::string text;
  for (int i = 0; i < 10; ++i) text += "@r" + std::to_string(i) + "\nACGTACGTAC\n+\nIIIIIIIIII\n";
  {
    std::istringstream in(text);
    FastqReader rd(in);
    CHECK(rd.next_batch(4).size() == 4);
    CHECK(rd.next_batch(4).size() == 4);
    CHECK(rd.next_batch(4).size() == 2);
    CHECK(rd.next_batch(4).empty());
  }
  {
    std::istringstream in(text);
    FastqReader rd(in);
    CHECK(rd.next_batch(100, 25).size() == 3);  // 30 bases >= 25 after the third read
  }
  std::istringstream empty("");
  FastqReader rd(empty);
  CHECK(rd.next_batch(8).empty());
}

TEST_CASE("SAM records: SPEC emit_sam examples on given hits") {
  const std::vector<std::string> chroms{"chrA", "chrB"};
  std::ostringstream os;
  write_sam_header(os, chroms, {0, 100, 250});
  CHECK(os.str() == "@HD\tVN:1.6\tSO:unsorted\n@SQ\tSN:chrA\tLN:100\n@SQ\tSN:chrB\tLN:150\n@PG\tID:qgmap-b200\tPN:qgmap-b200\n");
  // read 0: exact forward unique hit at internal position 10 -> POS 11, FLAG
  // 0, MAPQ 255, CIGAR 4M, NM 0. read 1: reverse strand. read 2: two
  // equal-identity hits -> primary + secondary. read 3: unmapped.
  std::vector<MappedHit> hits{{0, 0, 10, 0, 0}, {1, 1, 5, 1, 1}, {2, 1, 40, 0, 0}, {2, 0, 20, 0, 0}};
  std::vector<std::uint32_t> ranks{1, 1, 2, 2};
  std::vector<Alignment> al(4);
  al[0] = {10, 0, {4u << 4}};
  al[1] = {5, 1, {2u << 4, 1u << 4 | 2, 2u << 4}};
  al[2] = {40, 0, {4u << 4}};
  al[3] = {20, 0, {4u << 4}};
  std::ostringstream rec;
  write_sam_records(rec, {"q0", "q1", "q2", "q3"}, {"ACGT", "AACC", "GGTT", "TTTT"}, {"ABCD", "", "IIII", "IIII"},
                    chroms, hits, ranks, al, 1000000);
  std::istringstream lines(rec.str());
  std::string l;
  std::vector<std::string> L;
  while (std::getline(lines, l)) L.push_back(l);
  REQUIRE(L.size() == 5);
  CHECK(L[0] == "q0\t0\tchrA\t11\t255\t4M\t*\t0\t0\tACGT\tABCD\tNM:i:0");
  CHECK(L[1] == "q1\t16\tchrB\t6\t255\t2M1D2M\t*\t0\t0\tGGTT\t*\tNM:i:1");
  // equal identity: (chrom, position) orders them; the second is secondary
  CHECK(L[2] == "q2\t0\tchrA\t21\t60\t4M\t*\t0\t0\tGGTT\tIIII\tNM:i:0");
  CHECK(L[3] == "q2\t256\tchrB\t41\t60\t4M\t*\t0\t0\tGGTT\tIIII\tNM:i:0");
  CHECK(L[4] == "q3\t4\t*\t0\t0\t*\t*\t0\t0\tTTTT\tIIII");
}

TEST_CASE("pack_words equals pack_reads + PackedReadText::pack (N bases drawn in the same order)") {
  std::mt19937_64 g(3);
  std::vector<std::string> reads;
  for (int r = 0; r < 3000; ++r) {
    std::string s(g() % 130, 'A');
    for (auto& c : s) c = "ACGTNacgtn"[g() % 10];
    if (r % 17 == 0) s.clear();
    reads.push_back(s);
  }
  rng_engine a(11), b(11);
  const auto text = pack_reads(reads, 130, 12, a);
  const auto pw = pack_words(reads, 130, b, 4);
  CHECK(pw.words == text.pack());
  CHECK(pw.lengths == text.read_lengths);
  CHECK(a() == b());  // the same number of draws
  std::vector<std::string> bad{"ACGT", "ACXT"};
  rng_engine c(1);
  CHECK_THROWS_AS(pack_words(bad, 8, c), input_error);
  std::vector<std::string> longr{"ACGTACGTA"};
  CHECK_THROWS_AS(pack_words(longr, 8, c), input_error);
}
