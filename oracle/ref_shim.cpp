// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY. Compiled (by oracle/Makefile) against
// the reference's own headers under /root/reference/proj/{include,tests}; the
// reference sources are #included at build time, never copied into this repo.
// Output: oracle/_ref/libqgm_ref.so (git-ignored, travels to the GPU box).
//
// Exposes the reference's real code for pinning the oracle and as the CPU
// baseline of bench.py (--impl reference):
//   build_qgroup_index<W>      qgroup_index.hpp:124-180 (+ sample_group_starts :185-196)
//   oracle::filter_hits        oracles.hpp:37-51
//   banded/semiglobal/anchored oracles.hpp:57-135
//   pack_reads / encode_qgram  seq.hpp:80-84, 142-148
//   par::exclusive_scan        parallel.hpp:64-121
//   index_size_words           qgroup_index.hpp:198-213
// ref_map() = the reference's build_qgroup_index (stage 1, the only stage the
// reference ships) followed by the oracle restatement of stages 2-5
// (qgm_oracle.hpp), because the reference has no code for them.
#include <algorithm>
#include <chrono>
#include <sstream>

#include "oracles.hpp"            // /root/reference/proj/tests
#include "qgmap/qgroup_index.hpp"  // /root/reference/proj/include

#include "orc_capi.hpp"

namespace {

qgmap::PackedReadText make_text(const uint8_t* codes, uint32_t stride, const uint32_t* lengths,
                                uint32_t n_reads, unsigned q) {
  std::vector<std::vector<qgmap::base_code>> reads(n_reads);
  for (uint32_t r = 0; r < n_reads; ++r)
    reads[r].assign(codes + size_t(r) * stride, codes + size_t(r) * stride + lengths[r]);
  return qgmap::pack_encoded_reads(reads, stride, q);
}

template <class Fn>
int guarded_ref(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const qgmap::input_error& e) {
    orc::g_err = e.what();
    return 1;
  } catch (const qgm_oracle::input_error& e) {
    orc::g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    orc::g_err = e.what();
    return 2;
  }
}

template <class W>
void build_copy(const qgmap::PackedReadText& text, int sampled, unsigned threads, orc_buf** I, orc_buf** S,
                orc_buf** S1, orc_buf** O, std::string* summary) {
  auto ix = qgmap::build_qgroup_index<W>(text, threads);
  if (sampled) ix = qgmap::sample_group_starts(ix);
  *I = orc::make_buf(ix.occupancy());
  *S = orc::make_buf(ix.group_starts());
  *S1 = orc::make_buf(ix.occ_starts());
  *O = orc::make_buf(ix.positions());
  if (summary) *summary = ix.debug_summary();
}

}  // namespace

extern "C" {

uint64_t ref_buf_size(const orc_buf* b) { return b ? b->bytes.size() : 0; }
const void* ref_buf_data(const orc_buf* b) { return b ? b->bytes.data() : nullptr; }
void ref_buf_free(orc_buf* b) { delete b; }
const char* ref_last_error(void) { return orc::g_err.c_str(); }

int ref_build_index(const uint8_t* codes, uint32_t stride, const uint32_t* lengths, uint32_t n_reads,
                    unsigned q, unsigned w, int sampled, unsigned threads, orc_buf** I, orc_buf** S,
                    orc_buf** S1, orc_buf** O) {
  return guarded_ref([&] {
    auto text = make_text(codes, stride, lengths, n_reads, q);
    if (w == 32) build_copy<uint32_t>(text, sampled, threads, I, S, S1, O, nullptr);
    else if (w == 64) build_copy<uint64_t>(text, sampled, threads, I, S, S1, O, nullptr);
    else throw qgmap::input_error("group width must be 32 or 64");
  });
}

// Wall time of the reference index build alone (seconds), for BASELINE notes.
int ref_build_index_timed(const uint8_t* codes, uint32_t stride, const uint32_t* lengths, uint32_t n_reads,
                          unsigned q, unsigned threads, double* seconds, uint64_t* distinct) {
  return guarded_ref([&] {
    auto text = make_text(codes, stride, lengths, n_reads, q);
    auto t0 = std::chrono::steady_clock::now();
    auto ix = qgmap::build_qgroup_index<uint32_t>(text, threads);
    auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    *distinct = ix.distinct_qgram_count();
  });
}

// oracle::filter_hits over explicit (position, code) lists: 16-byte
// {int64 diagonal, uint32 read_id, uint32 pad} records sorted by (d, r).
int ref_filter_hits(const uint32_t* ref_positions, const uint32_t* ref_codes, uint64_t n_pos,
                    const uint8_t* codes, uint32_t stride, const uint32_t* lengths, uint32_t n_reads,
                    unsigned q, orc_buf** out) {
  return guarded_ref([&] {
    auto text = make_text(codes, stride, lengths, n_reads, q);
    auto hits = oracle::filter_hits({ref_positions, size_t(n_pos)}, {ref_codes, size_t(n_pos)}, text);
    struct Rec { int64_t d; uint32_t r, pad; };
    std::vector<Rec> v(hits.size());
    for (size_t i = 0; i < hits.size(); ++i) v[i] = {hits[i].diagonal, hits[i].read_id, 0};
    *out = orc::make_buf(v);
  });
}

int ref_banded_distance(const uint8_t* read, uint32_t n, const uint8_t* win, uint32_t L, unsigned B) {
  return oracle::banded_semiglobal_distance({read, n}, {win, L}, B);
}

int ref_semiglobal_distance(const uint8_t* read, uint32_t n, const uint8_t* win, uint32_t L) {
  return oracle::semiglobal_distance({read, n}, {win, L});
}

int ref_anchored_start_distance(const uint8_t* read, uint32_t n, const uint8_t* win, uint32_t L,
                                uint32_t start) {
  return oracle::anchored_start_distance({read, n}, {win, L}, start);
}

int ref_encode_qgram(const uint8_t* w, unsigned q, uint32_t* out) {
  return guarded_ref([&] { *out = qgmap::encode_qgram({w, q}); });
}

// pack_reads over '\0'-separated strings with a seeded rng (seq.hpp:142-148).
int ref_pack_reads(const char* joined, uint32_t n_reads, uint32_t stride, unsigned q, uint64_t seed,
                   orc_buf** codes, orc_buf** valid) {
  return guarded_ref([&] {
    std::vector<std::string> reads;
    const char* p = joined;
    for (uint32_t r = 0; r < n_reads; ++r) {
      reads.emplace_back(p);
      p += reads.back().size() + 1;
    }
    qgmap::rng_engine rng(seed);
    auto text = qgmap::pack_reads(reads, stride, q, rng);
    *codes = orc::make_buf(text.codes);
    *valid = orc::make_buf(text.valid_qgram_positions);
  });
}

int ref_exclusive_scan(const uint32_t* in, uint64_t n, unsigned threads, uint32_t* out, uint32_t* total) {
  return guarded_ref([&] {
    std::vector<uint32_t> v(in, in + n);
    auto res = qgmap::par::exclusive_scan(v, threads);
    std::copy(res.sums.begin(), res.sums.end(), out);
    *total = res.total;
  });
}

int ref_index_size_words(unsigned q, uint64_t text_len, unsigned width, uint64_t* qgroup, uint64_t* classic,
                         double* ratio) {
  auto s = qgmap::index_size_words(q, text_len, width);
  *qgroup = s.qgroup_words;
  *classic = s.classic_words;
  *ratio = s.ratio;
  return 0;
}

// CPU baseline of the whole path: reference index build + restated stages 2-5.
int ref_map(const uint8_t* ref_codes, const uint64_t* chrom_begin, uint32_t n_chrom, const uint8_t* mask,
            const uint8_t* read_codes, uint32_t stride, const uint32_t* lengths, uint32_t n_reads, unsigned q,
            unsigned w, int sampled, unsigned band, unsigned pct, int mode, int strands, unsigned threads,
            orc_buf** hits, uint64_t* stats) {
  return guarded_ref([&] {
    auto ref = orc::make_ref(ref_codes, chrom_begin, n_chrom, mask);
    auto rs = orc::make_reads(read_codes, stride, lengths, n_reads);
    auto t0 = std::chrono::steady_clock::now();  // stage 1 = pack_encoded_reads + build_qgroup_index
    auto text = make_text(read_codes, stride, lengths, n_reads, q);
    qgm_oracle::Params P;
    P.q = q; P.band = band; P.pct = pct; P.mode = mode; P.strands = strands;
    qgm_oracle::Stats st;
    std::vector<qgm_oracle::Hit> h;
    const unsigned th = qgm_oracle::eff_threads(threads);
    if (w == 64) {
      auto ix = qgmap::build_qgroup_index<uint64_t>(text, th);
      if (sampled) ix = qgmap::sample_group_starts(ix);
      st.sec_index = qgm_oracle::seconds_since(t0);
      h = qgm_oracle::map_with_index(ref, rs, ix, P, th, &st);
    } else {
      auto ix = qgmap::build_qgroup_index<uint32_t>(text, th);
      if (sampled) ix = qgmap::sample_group_starts(ix);
      st.sec_index = qgm_oracle::seconds_since(t0);
      h = qgm_oracle::map_with_index(ref, rs, ix, P, th, &st);
    }
    *hits = orc::make_buf(orc::to_recs(h));
    if (stats) {
      stats[0] = st.raw; stats[1] = st.unique; stats[2] = st.validated_kept; stats[3] = st.hits;
      const double sec[5] = {st.sec_index, st.sec_filter, st.sec_sort, st.sec_validate, st.sec_strata};
      for (int i = 0; i < 5; ++i) stats[4 + i] = uint64_t(sec[i] * 1e9);  // stage nanoseconds
    }
  });
}

}  // extern "C"
