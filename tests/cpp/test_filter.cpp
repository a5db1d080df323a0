// GPU parity tests of stage 2 (filter.cu): Alg. 2 filtration of the reference
// and its reverse complement, against the SPEC example and the
// CPU restatement (oracle::filter), itself pinned to the reference's
// oracle::filter_hits (oracles.hpp:37-51) by tests/test_oracle_pins.py.
#include <catch2/catch_amalgamated.hpp>

#include <set>

#include "testutil.hpp"

using namespace qgmap;

namespace {
Reference one_chrom(std::string_view s) {
  rng_engine rng(1);
  Reference R;
  R.add_chromosome("chr1", s, rng);
  return R;
}
}  // namespace

TEST_CASE("SPEC example: reads ACGT,TACG against ACGT (q=2, forward)") {
  rng_engine rng(1);
  const auto text = pack_reads({"ACGT", "TACG"}, 4, 2, rng);
  const auto ix = build_qgroup_index<std::uint32_t>(text);
  DeviceReference ref(one_chrom("ACGT"));
  const auto hits = filter_reference(ref, ix, FilterMode::full, QGM_STRAND_FWD);
  // oracle::filter_hits gives exactly {(0,0) x3, (-1,1) x2}
  std::multiset<std::pair<std::int64_t, std::uint32_t>> got;
  for (const auto& h : hits) got.insert({h.d, h.r});
  const std::multiset<std::pair<std::int64_t, std::uint32_t>> want{{0, 0}, {0, 0}, {0, 0}, {-1, 1}, {-1, 1}};
  CHECK(got == want);
}

TEST_CASE("empty reference positions give no hits") {
  rng_engine rng(1);
  const auto ix = build_qgroup_index<std::uint32_t>(pack_reads({"ACGTAC"}, 6, 4, rng));
  DeviceReference ref(one_chrom("ACG"));  // shorter than q
  CHECK(filter_reference(ref, ix).empty());
}

TEST_CASE("a read sharing no q-gram with the reference has no hits") {
  rng_engine rng(1);
  const auto ix = build_qgroup_index<std::uint32_t>(pack_reads({"AAAAAAAA", "ACGTACGT"}, 8, 4, rng));
  DeviceReference ref(one_chrom("CCCCCCCCCCCC"));
  for (const auto& h : filter_reference(ref, ix)) CHECK(h.r != 1);
}

template <class W>
void filter_vs_oracle(std::uint64_t seed, unsigned q, bool sampled, bool mask, int iters) {
  std::mt19937_64 g(seed);
  for (int it = 0; it < iters; ++it) {
    auto in = tu::make_instance(g, 1 + unsigned(g() % 5), 3000, 150, 20, 60, 0.05, q, mask, 3);
    auto ix = build_qgroup_index<W>(in.text);
    if (sampled) ix = sample_group_starts(ix);
    DeviceReference ref(in.ref);
    const auto ox = qgm_oracle::build_index<W>(in.oreads, q, false);
    INFO("seed=" << seed << " q=" << q << " iter=" << it);
    for (int strands : {1, 2, 3}) {
      auto want = qgm_oracle::filter(in.oref, in.oreads, ox, q, strands, false, 4);
      std::sort(want.begin(), want.end());
      const auto got = tu::to_oracle(filter_reference(ref, ix, FilterMode::full, strands));
      REQUIRE(got.size() == want.size());
      CHECK(got == want);
      // run-start emission: a sub-multiset with the same candidate SET
      auto rs = tu::to_oracle(filter_reference(ref, ix, FilterMode::run_start, strands, /*unique=*/true));
      want.erase(std::unique(want.begin(), want.end()), want.end());
      CHECK(rs == want);
      auto ors = qgm_oracle::filter(in.oref, in.oreads, ox, q, strands, true, 4);
      std::sort(ors.begin(), ors.end());
      CHECK(tu::to_oracle(filter_reference(ref, ix, FilterMode::run_start, strands)) == ors);
      // the default modes run the bucket-ordered join (join.cu); the forced
      // join and the streaming kernel (filter.cu) emit exactly the same multisets
      auto wfull = qgm_oracle::filter(in.oref, in.oreads, ox, q, strands, false, 4);
      std::sort(wfull.begin(), wfull.end());
      CHECK(tu::to_oracle(filter_reference(ref, ix, FilterMode::full_join, strands)) == wfull);
      CHECK(tu::to_oracle(filter_reference(ref, ix, FilterMode::run_start_join, strands)) == ors);
      CHECK(tu::to_oracle(filter_reference(ref, ix, FilterMode::full_stream, strands)) == wfull);
      CHECK(tu::to_oracle(filter_reference(ref, ix, FilterMode::run_start_stream, strands)) == ors);
    }
  }
}

TEST_CASE("device filtration equals the oracle multiset (multi-chromosome, both strands)") {
  for (unsigned q : {4u, 8u, 11u, 12u}) filter_vs_oracle<std::uint32_t>(10 + q, q, false, false, 3);
  filter_vs_oracle<std::uint32_t>(77, 16, false, false, 1);
}

TEST_CASE("device filtration equals the oracle with sampled S, u64 groups and a repeat mask") {
  filter_vs_oracle<std::uint32_t>(31, 9, true, true, 3);
  filter_vs_oracle<std::uint64_t>(32, 10, false, true, 3);
  filter_vs_oracle<std::uint64_t>(33, 7, true, false, 3);
}
