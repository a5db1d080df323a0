// GPU parity tests of stage 4 (validate.cu): banded bit-parallel validation
// against SPEC.md:384-395's examples and the CPU restatement
// (qgm_oracle::validate_candidate), whose k is pinned to the reference's
// oracle::banded_semiglobal_distance and whose start is pinned to a banded
// anchored-start DP by tests/test_oracle_pins.py.
#include <catch2/catch_amalgamated.hpp>

#include "testutil.hpp"

using namespace qgmap;

namespace {
std::vector<base_code> enc(std::string_view s) {
  rng_engine rng(1);
  return encode_sequence(s, rng);
}
}  // namespace

TEST_CASE("SPEC myers_banded examples") {
  const auto a = myers_banded(enc("ACGT"), enc("ACGT"));
  CHECK(a.k == 0);
  CHECK(a.start_offset == 0);
  CHECK(myers_banded(enc("ACGT"), enc("AGGT")).k == 1);
  const auto c = myers_banded(enc("ACGT"), enc("CCACGTCC"));  // B = 5
  CHECK(c.k == 0);
  CHECK(c.start_offset == 2);
}

TEST_CASE("identity threshold: n=100, k=25 dropped, k=5 kept (SPEC.md:393-395)") {
  std::mt19937_64 g(5);
  auto read = tu::random_codes(100, g);
  for (int k : {5, 25}) {
    auto chrom = tu::random_codes(400, g);
    std::copy(read.begin(), read.end(), chrom.begin() + 150);
    for (int e = 0; e < k; ++e) chrom[150 + std::size_t(e) * 4] = base_code((read[std::size_t(e) * 4] + 1) & 3);
    Reference R;
    R.names = {"c"};
    R.codes = chrom;
    R.chrom_begin = {0, chrom.size()};
    DeviceReference ref(R);
    std::vector<std::vector<base_code>> one{read};
    const auto text = pack_encoded_reads(one, 100, 16);
    const auto ix = build_qgroup_index<std::uint32_t>(text);
    const std::vector<Hit> hits{{150, 0, 0, 0}};
    const auto v = validate_hits(hits, ix, text, ref, BandConfig{32, 0.80});
    if (k == 25) {
      CHECK(v.empty());
    } else {
      REQUIRE(v.size() == 1);
      CHECK(v[0].k == 5);
      CHECK(v[0].ref_start == 150);
      CHECK(v[0].identity * 100 + v[0].k == 100);  // identity * n + k == n
    }
  }
}

TEST_CASE("device validation equals the oracle on random candidates (all bands, boundary windows)") {
  std::mt19937_64 g(99);
  for (int it = 0; it < 6; ++it) {
    auto in = tu::make_instance(g, 1 + unsigned(g() % 4), 2500, 200, 10 + unsigned(g() % 20), 120, 0.08, 8);
    const auto ix = build_qgroup_index<std::uint32_t>(in.text);
    DeviceReference ref(in.ref);
    const auto ox = qgm_oracle::build_index<std::uint32_t>(in.oreads, 8);
    auto cands = qgm_oracle::filter(in.oref, in.oreads, ox, 8, 3, true, 4);
    std::sort(cands.begin(), cands.end());
    cands.erase(std::unique(cands.begin(), cands.end()), cands.end());
    // extra diagonals hugging chromosome ends (sentinel windows)
    for (std::uint32_t c = 0; c < in.oref.chroms(); ++c) {
      const std::int64_t Lc = std::int64_t(in.oref.len(c));
      for (int e = 0; e < 20; ++e) {
        const std::uint32_t r = std::uint32_t(g() % in.oreads.count());
        const std::int64_t d = (e & 1) ? -std::int64_t(g() % 90) : Lc - 1 - std::int64_t(g() % 90);
        if (d < Lc && d > -60000) cands.push_back({r, c, d, std::uint8_t(g() & 1)});
      }
    }
    std::vector<Hit> hits(cands.size());
    std::vector<qgm_candidate> raw(cands.size());
    for (std::size_t i = 0; i < cands.size(); ++i)
      raw[i] = {cands[i].diag, cands[i].read, cands[i].chrom, cands[i].strand, 0};
    auto ctx = device::Context::default_context();
    for (unsigned B : {1u, 7u, 16u, 31u, 32u, 33u, 48u, 64u}) {
      const unsigned pct = std::vector<unsigned>{0, 60, 80, 100}[g() % 4];
      std::vector<qgm_validated> got(raw.size());
      ctx->check(qgm_validate(ctx->get(), ix.device_reads().get(), ref.get(), raw.data(), raw.size(), B, pct,
                              got.data()));
      int bad = 0;
      for (std::size_t i = 0; i < cands.size(); ++i) {
        const auto w = qgm_oracle::validate_candidate(in.oref, in.oreads, cands[i], B, pct);
        const bool same = w.in_range == bool(got[i].in_range) &&
                          (!w.in_range || (w.k == got[i].edits && w.start == got[i].start &&
                                           w.ref_start == got[i].ref_start && w.kept == bool(got[i].kept)));
        if (!same && bad++ < 3)
          std::fprintf(stderr, "B=%u cand %zu: oracle k=%d s=%u rs=%u kept=%d in=%d | gpu k=%d s=%u rs=%u kept=%d in=%d\n",
                       B, i, w.k, w.start, w.ref_start, w.kept, w.in_range, got[i].edits, got[i].start,
                       got[i].ref_start, got[i].kept, got[i].in_range);
      }
      INFO("B=" << B << " pct=" << pct << " iter=" << it << " n=" << cands.size());
      CHECK(bad == 0);
    }
  }
}
