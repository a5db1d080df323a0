// GPU parity tests of the whole path (qgm_map): index build -> filtration ->
// candidate radix sort/unique -> validation -> dedup + strata, against the CPU
// restatement (qgm_oracle::map_with_index) on seeded inputs, plus the
// postprocess examples of SPEC.md:443-471.
#include <catch2/catch_amalgamated.hpp>

#include "testutil.hpp"

using namespace qgmap;

namespace {
void map_vs_oracle(std::uint64_t seed, unsigned q, unsigned w, bool sampled, unsigned band, unsigned pct,
                   StratumMode mode, bool mask, unsigned n_reads, std::size_t chrom_len, double err, int strands = 3) {
  std::mt19937_64 g(seed);
  auto in = tu::make_instance(g, 1 + unsigned(g() % 4), chrom_len, n_reads, 40, 110, err, q, mask, 6);
  DeviceReference ref(in.ref);
  MapParams p;
  p.q = q;
  p.group_width = w;
  p.sampled = sampled;
  p.band = BandConfig{band, pct / 100.0};
  p.mode = mode;
  p.strands = strands;
  qgm_map_stats st{};
  const auto got = tu::to_oracle(map_reads(ref, in.text, p, &st));
  qgm_oracle::Params op;
  op.q = q; op.band = band; op.pct = pct; op.mode = int(mode); op.strands = strands;
  qgm_oracle::Stats ost;
  const auto ox = qgm_oracle::build_index<std::uint32_t>(in.oreads, q);
  const auto want = qgm_oracle::map_with_index(in.oref, in.oreads, ox, op, 4, &ost);
  INFO("seed=" << seed << " q=" << q << " w=" << w << " band=" << band << " pct=" << pct << " mode=" << int(mode)
                << " hits=" << want.size() << "/" << got.size());
  CHECK(st.unique_candidates == ost.unique);
  // both modes: candidates are abandoned only against the identity threshold
  CHECK(st.validated == ost.validated_kept);
  REQUIRE(got.size() == want.size());
  CHECK(got == want);
}
}  // namespace

TEST_CASE("map equals the oracle: best-stratum, q=12 (C1 shape, scaled down)") {
  map_vs_oracle(1, 12, 32, false, 32, 80, StratumMode::best_stratum, false, 600, 40000, 0.03);
  map_vs_oracle(2, 12, 32, false, 32, 80, StratumMode::best_stratum, false, 600, 40000, 0.08);
}

TEST_CASE("map equals the oracle: all mode, q=16 and q=10") {
  map_vs_oracle(3, 16, 32, false, 32, 80, StratumMode::all, false, 500, 30000, 0.03);
  map_vs_oracle(4, 10, 32, false, 32, 60, StratumMode::all, false, 400, 20000, 0.05);
}

TEST_CASE("map equals the oracle: u64 groups, sampled S, repeat mask, single strands") {
  map_vs_oracle(5, 11, 64, true, 32, 80, StratumMode::all, true, 400, 20000, 0.04);
  map_vs_oracle(6, 9, 32, true, 32, 80, StratumMode::best_stratum, true, 300, 15000, 0.04, 1);
  map_vs_oracle(7, 9, 64, false, 32, 80, StratumMode::all, false, 300, 15000, 0.04, 2);
}

TEST_CASE("map equals the oracle: bands 1..64 and identity thresholds") {
  map_vs_oracle(8, 12, 32, false, 16, 90, StratumMode::all, false, 300, 20000, 0.05);
  map_vs_oracle(9, 12, 32, false, 48, 70, StratumMode::best_stratum, false, 300, 20000, 0.08);
  map_vs_oracle(10, 12, 32, false, 64, 0, StratumMode::all, false, 150, 8000, 0.10);
  map_vs_oracle(11, 12, 32, false, 1, 95, StratumMode::all, false, 300, 20000, 0.02);
}

TEST_CASE("two identical chromosome copies: best-stratum keeps both equal hits (SPEC.md:470)") {
  std::mt19937_64 g(3);
  const auto chrom = tu::random_codes(2000, g);
  Reference R;
  R.names = {"a", "b"};
  R.codes = chrom;
  R.codes.insert(R.codes.end(), chrom.begin(), chrom.end());
  R.chrom_begin = {0, 2000, 4000};
  DeviceReference ref(R);
  std::vector<std::vector<base_code>> reads{std::vector<base_code>(chrom.begin() + 500, chrom.begin() + 600)};
  reads[0][50] = base_code((reads[0][50] + 1) & 3);  // one substitution
  const auto text = pack_encoded_reads(reads, 100, 16);
  MapParams p;
  const auto best = map_reads(ref, text, p);
  REQUIRE(best.size() == 2);
  CHECK(best[0].chrom == 0);
  CHECK(best[1].chrom == 1);
  CHECK(best[0].ref_start == 500);
  CHECK(best[0].edits == 1);
  CHECK(best[1].edits == 1);
  p.mode = StratumMode::all;
  const auto all = map_reads(ref, text, p);
  CHECK(all.size() >= best.size());  // best-stratum is a subset of all
}

TEST_CASE("cluster duplicates of one alignment collapse to a single record (SPEC.md:445)") {
  std::mt19937_64 g(4);
  const auto chrom = tu::random_codes(5000, g);
  Reference R;
  R.names = {"c"};
  R.codes = chrom;
  R.chrom_begin = {0, 5000};
  DeviceReference ref(R);
  std::vector<std::vector<base_code>> reads{std::vector<base_code>(chrom.begin() + 1000, chrom.begin() + 1100)};
  reads[0].erase(reads[0].begin() + 40);  // a deletion splits the q-gram runs over two diagonals
  reads[0].push_back(chrom[1100]);
  const auto text = pack_encoded_reads(reads, 100, 12);
  MapParams p;
  p.q = 12;
  p.mode = StratumMode::all;
  qgm_map_stats st{};
  const auto hits = map_reads(ref, text, p, &st);
  CHECK(st.unique_candidates >= 2);
  std::size_t at_origin = 0;
  for (const auto& h : hits) at_origin += (h.ref_start == 1000 && h.strand == 0);
  CHECK(at_origin == 1);
}

TEST_CASE("empty read buffer maps to no hits") {
  std::mt19937_64 g(1);
  Reference R;
  R.names = {"c"};
  R.codes = tu::random_codes(1000, g);
  R.chrom_begin = {0, 1000};
  DeviceReference ref(R);
  const auto text = pack_encoded_reads({}, 100, 16);
  CHECK(map_reads(ref, text).empty());
}

TEST_CASE("bad parameters raise input_error") {
  std::mt19937_64 g(1);
  Reference R;
  R.names = {"c"};
  R.codes = tu::random_codes(1000, g);
  R.chrom_begin = {0, 1000};
  DeviceReference ref(R);
  const auto text = pack_encoded_reads({tu::random_codes(50, g)}, 50, 8);
  MapParams p;
  p.band.band_width = 65;
  CHECK_THROWS_AS(map_reads(ref, text, p), input_error);
  p.band.band_width = 32;
  p.band.identity_threshold = 1.5;
  CHECK_THROWS_AS(map_reads(ref, text, p), input_error);
  p.band.identity_threshold = 0.8;
  p.q = 0;
  CHECK_THROWS_AS(map_reads(ref, text, p), input_error);
}

TEST_CASE("device repeat mask: SPEC examples (SPEC.md:283-284)") {
  rng_engine rng(1);
  {  // "AAAAAAAA", q=2, threshold=3: code 0 occurs 7 > 3 times -> P empty
    Reference R;
    R.add_chromosome("a", "AAAAAAAA", rng);
    DeviceReference ref(R);
    ref.mask_repeats(2, 3);
    const auto m = ref.mask();
    REQUIRE(m.size() == 8);
    for (int x = 0; x < 7; ++x) CHECK(m[x] == 1);
    CHECK(m[7] == 0);  // no full window at the last base
  }
  {  // "ACGTACGT", q=2, threshold=100: nothing masked
    Reference R;
    R.add_chromosome("a", "ACGTACGT", rng);
    DeviceReference ref(R);
    ref.mask_repeats(2, 100);
    const auto m = ref.mask();
    CHECK(std::count(m.begin(), m.end(), 1) == 0);
  }
}

TEST_CASE("device repeat mask equals the oracle's, per chromosome, and maps identically") {
  for (std::uint64_t seed : {21u, 22u, 23u}) {
    std::mt19937_64 g(seed);
    for (unsigned q : {8u, 12u, 16u}) {
      auto in = tu::make_instance(g, 1 + unsigned(g() % 4), 30000, 200, 40, 110, 0.02, q, false);
      const unsigned thr = 1 + unsigned(g() % 3);
      // chromosome copies inside the instance make some q-grams frequent
      const auto want = qgm_oracle::repeat_mask(in.ref.codes, in.ref.chrom_begin, q, thr);
      DeviceReference ref(in.ref);
      ref.mask_repeats(q, thr);
      INFO("seed=" << seed << " q=" << q << " thr=" << thr);
      REQUIRE(ref.mask() == want);
      MapParams p;
      p.q = q;
      p.mode = StratumMode::all;
      const auto got = tu::to_oracle(map_reads(ref, in.text, p));
      in.oref.mask = want;
      qgm_oracle::Params op;
      op.q = q; op.mode = 1;
      const auto ox = qgm_oracle::build_index<std::uint32_t>(in.oreads, q);
      const auto oh = qgm_oracle::map_with_index(in.oref, in.oreads, ox, op, 4, nullptr);
      CHECK(got == oh);
    }
  }
}

TEST_CASE("mapping_quality: SPEC examples (SPEC.md:455-457)") {
  CHECK(mapping_quality(1, 12345) == 255);
  CHECK(mapping_quality(2, 1000000) == 60);
  CHECK(mapping_quality(11, 1000000) == 50);
  CHECK(mapping_quality(1000001, 1000000) == 0);  // floored at 0
  for (unsigned r = 2; r < 200; ++r) CHECK(mapping_quality(r + 1, 1000000) <= mapping_quality(r, 1000000));
}

TEST_CASE("hit_rank on the device: counts of identity >= own, per read (SPEC.md:446-451)") {
  for (std::uint64_t seed : {41u, 42u}) {
    std::mt19937_64 g(seed);
    auto in = tu::make_instance(g, 3, 20000, 300, 40, 110, 0.02, 12, false);
    DeviceReference ref(in.ref);
    for (StratumMode mode : {StratumMode::all, StratumMode::best_stratum}) {
      MapParams p;
      p.q = 12;
      p.mode = mode;
      std::vector<std::uint32_t> R;
      const auto hits = map_reads_ranked(ref, in.text, p, nullptr, &R);
      REQUIRE(R.size() == hits.size());
      for (std::size_t i = 0; i < hits.size(); ++i) {
        std::uint32_t want = 0;
        for (const auto& h : hits)
          if (h.read_id == hits[i].read_id && h.edits <= hits[i].edits) ++want;
        CHECK(R[i] == want);
        if (mode == StratumMode::best_stratum) {  // the size of the read's best stratum
          std::uint32_t same = 0;
          for (const auto& h : hits) same += h.read_id == hits[i].read_id;
          CHECK(R[i] == same);
        }
      }
    }
  }
}
