// orc_oracle.cpp -- TEST INFRASTRUCTURE ONLY. extern "C" surface of the CPU
// restatement (qgm_oracle.hpp), built into oracle/build/libqgm_oracle.so.
#include "orc_capi.hpp"

using namespace qgm_oracle;

extern "C" {

uint64_t orc_buf_size(const orc_buf* b) { return b ? b->bytes.size() : 0; }
const void* orc_buf_data(const orc_buf* b) { return b ? b->bytes.data() : nullptr; }
void orc_buf_free(orc_buf* b) { delete b; }
const char* orc_last_error(void) { return orc::g_err.c_str(); }

int orc_encode_qgram(const uint8_t* w, unsigned q, uint32_t* out) {
  return orc::guarded([&] { *out = encode_qgram(w, q); });
}

int orc_rc_qgram(uint32_t g, unsigned q, uint32_t* out) {
  return orc::guarded([&] { *out = rc_qgram(g, q); });
}

// Alg. 1 restatement; O sorted within every interval.
int orc_build_index(const uint8_t* codes, uint32_t stride, const uint32_t* lengths, uint32_t n_reads,
                    unsigned q, unsigned w, int sampled, orc_buf** I, orc_buf** S, orc_buf** S1,
                    orc_buf** O) {
  return orc::guarded([&] {
    auto rs = orc::make_reads(codes, stride, lengths, n_reads);
    if (w == 32) {
      auto ix = build_index<uint32_t>(rs, q, sampled != 0);
      *I = orc::make_buf(ix.I); *S = orc::make_buf(ix.S); *S1 = orc::make_buf(ix.S1); *O = orc::make_buf(ix.O);
    } else if (w == 64) {
      auto ix = build_index<uint64_t>(rs, q, sampled != 0);
      *I = orc::make_buf(ix.I); *S = orc::make_buf(ix.S); *S1 = orc::make_buf(ix.S1); *O = orc::make_buf(ix.O);
    } else {
      throw input_error("group width must be 32 or 64");
    }
  });
}

// Filtration (Alg. 2) over all chromosomes with the restated index. Output is
// the candidate multiset sorted by (read, strand, chrom, diag).
int orc_filter(const uint8_t* ref_codes, const uint64_t* chrom_begin, uint32_t n_chrom, const uint8_t* mask,
               const uint8_t* read_codes, uint32_t stride, const uint32_t* lengths, uint32_t n_reads,
               unsigned q, int strands, int run_start, unsigned threads, orc_buf** out) {
  return orc::guarded([&] {
    auto ref = orc::make_ref(ref_codes, chrom_begin, n_chrom, mask);
    auto rs = orc::make_reads(read_codes, stride, lengths, n_reads);
    auto ix = build_index<uint32_t>(rs, q, false);
    auto c = filter(ref, rs, ix, q, strands, run_start != 0, threads);
    std::sort(c.begin(), c.end());
    *out = orc::make_buf(orc::to_recs(c));
  });
}

// One (read', window) pair: banded DP (use_dp=1) or the bit-parallel pass.
int orc_validate(const uint8_t* read, uint32_t n, const uint8_t* win, uint32_t L, unsigned B, int use_dp,
                 int32_t* k, uint32_t* start) {
  return orc::guarded([&] {
    const VRes r = use_dp ? validate_dp(read, n, win, L, B) : validate_myers(read, n, win, L, B);
    *k = r.k;
    *start = r.start;
  });
}

// Validation of explicit candidates (24-byte CandRec) -> 20-byte ValRec each.
int orc_validate_cands(const uint8_t* ref_codes, const uint64_t* chrom_begin, uint32_t n_chrom,
                       const uint8_t* read_codes, uint32_t stride, const uint32_t* lengths, uint32_t n_reads,
                       const void* cands, uint64_t n_cands, unsigned B, unsigned pct, int use_dp,
                       unsigned threads, void* out) {
  return orc::guarded([&] {
    if (B == 0 || B > kMaxBand) throw input_error("band must be in [1, 64]");
    auto ref = orc::make_ref(ref_codes, chrom_begin, n_chrom, nullptr);
    auto rs = orc::make_reads(read_codes, stride, lengths, n_reads);
    auto* cr = static_cast<const orc::CandRec*>(cands);
    auto* vr = static_cast<orc::ValRec*>(out);
    parallel_chunks(n_cands, threads, [&](size_t b, size_t e) {
      for (size_t i = b; i < e; ++i) {
        Cand c{cr[i].read, cr[i].chrom, cr[i].diag, uint8_t(cr[i].strand)};
        Validated v = validate_candidate(ref, rs, c, B, pct, use_dp != 0);
        vr[i] = {v.k, v.start, v.ref_start, uint8_t(v.kept), uint8_t(v.in_range), 0, 0, 0};
      }
    });
  });
}

// traceback_cigar (DESIGN.md section 2 item 9) of explicit 16-byte hit records. ops: n *
// max_ops u32 (BAM-style); info per hit: {ref_start u32, n_ops u16, edits u16}
// (n_ops > max_ops: truncated).
int orc_cigar(const uint8_t* ref_codes, const uint64_t* chrom_begin, uint32_t n_chrom, const uint8_t* read_codes,
              uint32_t stride, const uint32_t* lengths, uint32_t n_reads, const void* hits, uint64_t n_hits,
              unsigned B, uint32_t max_ops, unsigned threads, uint32_t* ops, void* info) {
  return orc::guarded([&] {
    auto ref = orc::make_ref(ref_codes, chrom_begin, n_chrom, nullptr);
    auto rs = orc::make_reads(read_codes, stride, lengths, n_reads);
    auto* hr = static_cast<const orc::HitRec*>(hits);
    struct Info { uint32_t ref_start; uint16_t n_ops, edits; };
    auto* inf = static_cast<Info*>(info);
    parallel_chunks(n_hits, threads, [&](size_t b, size_t e) {
      for (size_t i = b; i < e; ++i) {
        const orc::HitRec& h = hr[i];
        if (h.read >= rs.count() || h.chrom + 1 >= ref.chrom_begin.size()) throw input_error("hit out of range");
        const uint32_t n = rs.lengths[h.read];
        std::vector<uint8_t> rd(rs.read(h.read), rs.read(h.read) + n);
        if (h.strand) rd = reverse_complement(rd.data(), n);
        const uint8_t* chrom = ref.codes.data() + ref.chrom_begin[h.chrom];
        const Cigar c = traceback_cigar(rd.data(), n, chrom, int64_t(ref.len(h.chrom)), h.ref_start, B);
        inf[i] = {c.ref_start, uint16_t(c.ops.size()), uint16_t(c.edits)};
        for (size_t t = 0; t < c.ops.size() && t < max_ops; ++t) ops[i * max_ops + t] = c.ops[t];
      }
    });
  });
}

// Whole path with the restated index: stats = {raw, unique, kept, hits}.
int orc_map(const uint8_t* ref_codes, const uint64_t* chrom_begin, uint32_t n_chrom, const uint8_t* mask,
            const uint8_t* read_codes, uint32_t stride, const uint32_t* lengths, uint32_t n_reads,
            unsigned q, unsigned w, int sampled, unsigned band, unsigned pct, int mode, int strands,
            unsigned threads, orc_buf** hits, uint64_t* stats) {
  return orc::guarded([&] {
    auto ref = orc::make_ref(ref_codes, chrom_begin, n_chrom, mask);
    auto rs = orc::make_reads(read_codes, stride, lengths, n_reads);
    Params P;
    P.q = q; P.band = band; P.pct = pct; P.mode = mode; P.strands = strands;
    Stats st;
    std::vector<Hit> h;
    auto t0 = std::chrono::steady_clock::now();
    if (w == 64) {
      auto ix = build_index<uint64_t>(rs, q, sampled != 0);
      st.sec_index = seconds_since(t0);
      h = map_with_index(ref, rs, ix, P, threads, &st);
    } else {
      auto ix = build_index<uint32_t>(rs, q, sampled != 0);
      st.sec_index = seconds_since(t0);
      h = map_with_index(ref, rs, ix, P, threads, &st);
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
