// orc_capi.hpp -- TEST INFRASTRUCTURE ONLY. Shared extern "C" glue of the CPU
// oracle (oracle/libqgm_oracle.so) and of the reference shim
// (oracle/_ref/libqgm_ref.so). Loaded only by tests/, smoke() and bench.py's
// cpu_baseline / --impl reference legs.
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "qgm_oracle.hpp"

struct orc_buf {
  std::vector<uint8_t> bytes;
};

namespace orc {

inline thread_local std::string g_err;

template <class T>
orc_buf* make_buf(const std::vector<T>& v) {
  auto* b = new orc_buf;
  b->bytes.resize(v.size() * sizeof(T));
  if (!v.empty()) std::memcpy(b->bytes.data(), v.data(), b->bytes.size());
  return b;
}

inline qgm_oracle::ReadSet make_reads(const uint8_t* codes, uint32_t stride, const uint32_t* lengths,
                                      uint32_t n_reads) {
  qgm_oracle::ReadSet rs;
  rs.stride = stride;
  rs.lengths.assign(lengths, lengths + n_reads);
  rs.codes.assign(codes, codes + size_t(stride) * n_reads);
  for (uint32_t r = 0; r < n_reads; ++r)
    if (rs.lengths[r] > stride) throw qgm_oracle::input_error("read longer than stride");
  if (uint64_t(stride) * n_reads > 0xFFFFFFFFull)
    throw qgm_oracle::input_error("read text exceeds 2^32 positions");
  return rs;
}

inline qgm_oracle::RefSet make_ref(const uint8_t* codes, const uint64_t* chrom_begin, uint32_t n_chrom,
                                   const uint8_t* mask) {
  qgm_oracle::RefSet ref;
  ref.chrom_begin.assign(chrom_begin, chrom_begin + n_chrom + 1);
  const uint64_t total = chrom_begin[n_chrom];
  ref.codes.assign(codes, codes + total);
  if (mask) ref.mask.assign(mask, mask + total);
  return ref;
}

// 24-byte candidate record shared with the python side.
struct CandRec {
  int64_t diag;
  uint32_t read;
  uint32_t chrom;
  uint32_t strand;
  uint32_t pad;
};

// 16-byte hit record (== qgm_hit in include/qgm_c.h).
struct HitRec {
  uint32_t read, chrom, ref_start;
  uint16_t k;
  uint8_t strand, pad;
};

// 20-byte per-candidate validation record.
struct ValRec {
  int32_t k;
  uint32_t start;
  uint32_t ref_start;
  uint8_t kept, in_range, pad0, pad1;
  uint32_t pad2;
};

inline std::vector<CandRec> to_recs(const std::vector<qgm_oracle::Cand>& c) {
  std::vector<CandRec> out(c.size());
  for (size_t i = 0; i < c.size(); ++i) out[i] = {c[i].diag, c[i].read, c[i].chrom, c[i].strand, 0};
  return out;
}

inline std::vector<HitRec> to_recs(const std::vector<qgm_oracle::Hit>& h) {
  std::vector<HitRec> out(h.size());
  for (size_t i = 0; i < h.size(); ++i) out[i] = {h[i].read, h[i].chrom, h[i].ref_start, h[i].k, h[i].strand, 0};
  return out;
}

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const qgm_oracle::input_error& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

}  // namespace orc
