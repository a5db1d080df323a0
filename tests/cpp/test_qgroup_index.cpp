// GPU parity tests of stage 1: the q-group index built by index_build.cu
// against the worked examples of SPEC.md:195-235 and the CPU restatement of
// Alg. 1 (oracle/qgm_oracle.hpp, itself pinned to the reference's
// build_qgroup_index by tests/test_oracle_pins.py).
#include <catch2/catch_amalgamated.hpp>

#include "testutil.hpp"

using namespace qgmap;

namespace {
std::vector<std::uint32_t> occ_sorted(const QGroupIndex<>& ix, std::string_view s) {
  rng_engine rng(1);
  auto sp = ix.occurrences(encode_qgram(encode_sequence(s, rng)));
  std::vector<std::uint32_t> v(sp.begin(), sp.end());
  std::sort(v.begin(), v.end());
  return v;
}
}  // namespace

TEST_CASE("SPEC worked example: ACGTACGT, q=2 sets bits {1,6,11,12} of I[0]") {
  rng_engine rng(1);
  const auto text = pack_reads({"ACGTACGT"}, 8, 2, rng);
  const auto ix = build_qgroup_index<std::uint32_t>(text);
  CHECK(ix.group_count() == 1);
  CHECK(ix.occupancy()[0] == ((1u << 1) | (1u << 6) | (1u << 11) | (1u << 12)));
  CHECK(ix.occupancy()[0] == 0x1842u);
  CHECK(occ_sorted(ix, "AC") == std::vector<std::uint32_t>{0, 4});
  CHECK(occ_sorted(ix, "CG") == std::vector<std::uint32_t>{1, 5});
  CHECK(occ_sorted(ix, "GT") == std::vector<std::uint32_t>{2, 6});
  CHECK(occ_sorted(ix, "TA") == std::vector<std::uint32_t>{3});
  CHECK(!ix.index_pair(15).has_value());  // "TT"
  CHECK(ix.distinct_qgram_count() == 4);
  CHECK(ix.occurrence_count() == 7);
  CHECK(ix.group_starts() == std::vector<std::uint32_t>{0, 4});
}

TEST_CASE("SPEC worked example: AAAA -> code 0 at {0,1,2}") {
  rng_engine rng(1);
  const auto ix = build_qgroup_index<std::uint32_t>(pack_reads({"AAAA"}, 4, 2, rng));
  CHECK(occ_sorted(ix, "AA") == std::vector<std::uint32_t>{0, 1, 2});
  CHECK(ix.distinct_qgram_count() == 1);
}

TEST_CASE("SPEC worked example: boundary q-grams are not indexed") {
  rng_engine rng(1);
  const auto ix = build_qgroup_index<std::uint32_t>(pack_reads({"AC", "GT"}, 2, 2, rng));
  CHECK(occ_sorted(ix, "AC") == std::vector<std::uint32_t>{0});
  CHECK(occ_sorted(ix, "GT") == std::vector<std::uint32_t>{2});
  CHECK(occ_sorted(ix, "CG").empty());
}

TEST_CASE("sampled S keeps every lookup (SPEC.md:234)") {
  rng_engine rng(1);
  const auto full = build_qgroup_index<std::uint32_t>(pack_reads({"ACGTACGT"}, 8, 2, rng));
  const auto half = sample_group_starts(full);
  CHECK(half.sampled());
  CHECK(occ_sorted(half, "CG") == std::vector<std::uint32_t>{1, 5});
  CHECK(half.group_starts().size() == (full.group_starts().size() + 1) / 2);
}

TEST_CASE("empty text: every code absent") {
  rng_engine rng(1);
  const auto ix = build_qgroup_index<std::uint32_t>(pack_reads({}, 4, 3, rng));
  CHECK(ix.occurrence_count() == 0);
  CHECK(ix.distinct_qgram_count() == 0);
  for (qgram_code g = 0; g < 64; ++g) CHECK(!ix.index_pair(g).has_value());
}

template <class W>
void compare_random(unsigned q, bool sampled, int iters, std::uint64_t seed) {
  std::mt19937_64 g(seed);
  for (int it = 0; it < iters; ++it) {
    const unsigned n_reads = unsigned(g() % 300);
    const unsigned stride = q + unsigned(g() % 40);
    std::vector<std::vector<base_code>> reads(n_reads);
    for (auto& r : reads) {
      r = tu::random_codes(g() % (stride + 1), g);
      if (g() % 5 == 0) std::fill(r.begin(), r.end(), base_code(0));  // poly-A: one hot q-gram
    }
    const auto text = pack_encoded_reads(reads, stride, q);
    auto ix = build_qgroup_index<W>(text);
    if (sampled) ix = sample_group_starts(ix);
    qgm_oracle::ReadSet rs{text.codes, text.stride, text.read_lengths};
    const auto ox = qgm_oracle::build_index<W>(rs, q, sampled);
    INFO("q=" << q << " w=" << sizeof(W) * 8 << " sampled=" << sampled << " iter=" << it);
    REQUIRE(ix.occupancy() == ox.occupancy());
    REQUIRE(ix.group_starts() == ox.group_starts());
    REQUIRE(ix.occ_starts() == ox.occ_starts());
    CHECK(tu::sort_intervals(ix.positions(), ix.occ_starts()) == ox.positions());
    ix.normalize();
    CHECK(ix.positions() == ox.positions());
  }
}

TEST_CASE("device index equals the oracle for random texts (u32 groups, q=1..16)") {
  for (unsigned q = 1; q <= 16; ++q) compare_random<std::uint32_t>(q, false, q <= 12 ? 6 : 2, 100 + q);
}

TEST_CASE("device index equals the oracle for random texts (u64 groups, sampled)") {
  for (unsigned q : {2u, 5u, 8u, 11u, 13u}) {
    compare_random<std::uint64_t>(q, false, 4, 200 + q);
    compare_random<std::uint64_t>(q, true, 4, 300 + q);
    compare_random<std::uint32_t>(q, true, 4, 400 + q);
  }
}

TEST_CASE("debug_summary is reproducible after normalisation") {
  std::mt19937_64 g(7);
  std::vector<std::vector<base_code>> reads(2000);
  for (auto& r : reads) r = tu::random_codes(100, g);
  const auto text = pack_encoded_reads(reads, 100, 12);
  auto a = build_qgroup_index<std::uint32_t>(text);
  auto b = build_qgroup_index<std::uint32_t>(text);
  a.normalize();
  b.normalize();
  CHECK(a.debug_summary() == b.debug_summary());
  qgm_oracle::ReadSet rs{text.codes, text.stride, text.read_lengths};
  const auto ox = qgm_oracle::build_index<std::uint32_t>(rs, 12);
  CHECK(a.positions() == ox.positions());
}

TEST_CASE("q out of range is rejected with input_error") {
  rng_engine rng(1);
  auto text = pack_reads({"ACGT"}, 4, 2, rng);
  text.q = 17;
  CHECK_THROWS_AS(build_qgroup_index<std::uint32_t>(text), input_error);
}
