// qgm_oracle.hpp -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
//
// CPU restatement of the PEANUT (arXiv 1403.1706) read-mapping hot path:
//   q-group index build -> filtration (+RC) -> candidate dedup -> banded Myers
//   validation -> best-stratum / all-hits reduction.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
// this code. The CUDA product path (paper_1403_1706_b200/csrc) never links it.
//
// Anchors in the reference (/root/reference, read-only; cited as path:line):
//   codec            proj/include/qgmap/seq.hpp:18-84, 98-140
//   index (Alg. 1)   proj/include/qgmap/qgroup_index.hpp:50-63 (lookup),
//                    :80-96 (rank / sampled base), :124-180 (build), :185-196
//                    (sampling)
//   filtration       PAPER.md:284-321 (Alg. 2); proj/tests/oracles.hpp:29-51
//   validation       proj/tests/oracles.hpp:86-111 (banded DP, band j-i in [0,B)),
//                    :116-135 (anchored start)
//   postprocess      SPEC.md:437-472 (dedup min-k, best-stratum / all)
//
// Stages 2-5 have no reference code; the details SPEC.md leaves open are frozen
// by SURVEY.md Appendix B and restated in DESIGN.md section 2 ("parity
// contract"). Every function below follows that contract literally and is
// kept simple; it is pinned against the reference's own build_qgroup_index and
// brute-force oracles (oracle/_ref, tests/golden) by tests/test_oracle_pins.py.
#pragma once

#include <algorithm>
#include <type_traits>
#include <chrono>
#include <atomic>
#include <bit>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

namespace qgm_oracle {

inline constexpr uint8_t kSentinel = 4;     // window base outside the chromosome
inline constexpr unsigned kMaxQ = 16;       // seq.hpp:27
inline constexpr unsigned kMaxBand = 64;    // one 64-bit band word

struct input_error : std::runtime_error {
  explicit input_error(const std::string& w) : std::runtime_error(w) {}
};

// ---------------------------------------------------------------- threads
inline unsigned eff_threads(unsigned t) {
  if (t == 0) {
    unsigned hw = std::thread::hardware_concurrency();
    return hw ? hw : 1;
  }
  return t;
}

// body(begin, end) over contiguous chunks, like par::parallel_for
// (parallel.hpp:31-49) but exception-safe (the reference terminates).
template <class Fn>
void parallel_chunks(size_t count, unsigned threads, Fn&& body) {
  threads = eff_threads(threads);
  if (count == 0) return;
  if (threads <= 1 || count < 1024) { body(size_t(0), count); return; }
  const size_t chunk = (count + threads - 1) / threads;
  std::vector<std::thread> ws;
  std::vector<std::exception_ptr> errs(threads);
  for (unsigned t = 0; t < threads; ++t) {
    size_t b = std::min(count, size_t(t) * chunk), e = std::min(count, b + chunk);
    if (b >= e) break;
    ws.emplace_back([&, t, b, e] {
      try { body(b, e); } catch (...) { errs[t] = std::current_exception(); }
    });
  }
  for (auto& w : ws) w.join();
  for (auto& e : errs) if (e) std::rethrow_exception(e);
}

// ---------------------------------------------------------------- inputs
// PackedReadText equivalent (seq.hpp:98-115): 1 byte per base, fixed stride.
struct ReadSet {
  std::vector<uint8_t> codes;
  uint32_t stride = 0;
  std::vector<uint32_t> lengths;
  uint32_t count() const { return uint32_t(lengths.size()); }
  const uint8_t* read(uint32_t r) const { return codes.data() + size_t(r) * stride; }
};

// Concatenated chromosomes (ReferenceIndex), 1 byte per base.
struct RefSet {
  std::vector<uint8_t> codes;
  std::vector<uint64_t> chrom_begin;  // n_chrom + 1 offsets into codes
  std::vector<uint8_t> mask;          // empty, or 1 byte/base: 1 = position not in P
  uint32_t chroms() const { return chrom_begin.empty() ? 0 : uint32_t(chrom_begin.size() - 1); }
  uint64_t len(uint32_t c) const { return chrom_begin[c + 1] - chrom_begin[c]; }
  bool masked(uint64_t global) const { return !mask.empty() && mask[global]; }
};

// encode_qgram (seq.hpp:80-84): first base in the most significant digit.
inline uint32_t encode_qgram(const uint8_t* w, unsigned q) {
  uint32_t g = 0;
  for (unsigned t = 0; t < q; ++t) g = (g << 2) | uint32_t(w[t] & 3u);
  return g;
}

// Code of the reverse complement of the window whose code is g.
inline uint32_t rc_qgram(uint32_t g, unsigned q) {
  uint32_t r = 0;
  for (unsigned t = 0; t < q; ++t) { r = (r << 2) | (3u - (g & 3u)); g >>= 2; }
  return r;
}

inline std::vector<uint8_t> reverse_complement(const uint8_t* s, size_t n) {
  std::vector<uint8_t> rc(n);
  for (size_t i = 0; i < n; ++i) rc[i] = uint8_t(3u - s[n - 1 - i]);
  return rc;
}

// ---------------------------------------------------------------- stage 1
// q-group index restatement (Alg. 1; qgroup_index.hpp:124-180). Positions are
// written in ascending text order, so each O interval is sorted -- the
// normalisation test_parallel.cpp:121-122 applies before comparing.
// Repeat mask of build_reference_index: 1 for every
// position whose forward q-gram occurs more than `threshold` times among the
// windows of its own chromosome (counted over all windows).
inline std::vector<uint8_t> repeat_mask(const std::vector<uint8_t>& codes, const std::vector<uint64_t>& chrom_begin,
                                        unsigned q, uint64_t threshold) {
  std::vector<uint8_t> mask(codes.size(), 0);
  for (size_t c = 0; c + 1 < chrom_begin.size(); ++c) {
    const uint64_t b = chrom_begin[c], L = chrom_begin[c + 1] - b;
    if (L < q) continue;
    std::vector<uint32_t> g(L - q + 1);
    for (uint64_t p = 0; p + q <= L; ++p) g[p] = encode_qgram(codes.data() + b + p, q);
    std::vector<uint32_t> s = g;
    std::sort(s.begin(), s.end());
    for (uint64_t p = 0; p + q <= L; ++p) {
      const auto r = std::equal_range(s.begin(), s.end(), g[p]);
      if (uint64_t(r.second - r.first) > threshold) mask[b + p] = 1;
    }
  }
  return mask;
}

template <class W>
struct Index {
  static constexpr unsigned group_width = std::numeric_limits<W>::digits;
  unsigned q_ = 0;
  bool sampled_ = false;
  std::vector<W> I;
  std::vector<uint32_t> S, S1, O;

  unsigned q() const { return q_; }
  bool sampled() const { return sampled_; }
  const std::vector<W>& occupancy() const { return I; }
  const std::vector<uint32_t>& group_starts() const { return S; }
  const std::vector<uint32_t>& occ_starts() const { return S1; }
  const std::vector<uint32_t>& positions() const { return O; }

  static uint32_t rank_below(W word, unsigned j) {  // qgroup_index.hpp:80-83
    const W m = j == 0 ? W(0) : W(~W(0) >> (group_width - j));
    return uint32_t(std::popcount(W(word & m)));
  }
  uint32_t group_base(size_t i) const {  // qgroup_index.hpp:91-96
    if (!sampled_) return S[i];
    const uint32_t even = S[i / 2];
    return (i & 1) ? even + uint32_t(std::popcount(I[i - 1])) : even;
  }
  std::optional<std::pair<uint32_t, uint32_t>> index_pair(uint32_t g) const {  // :50-57
    const size_t i = g / group_width;
    const unsigned j = g % group_width;
    const W word = I[i];
    if (word == 0 || !((word >> j) & W(1))) return std::nullopt;
    const uint32_t b = group_base(i) + rank_below(word, j);
    return std::make_pair(S1[b], S1[b + 1]);
  }
};

template <class W>
Index<W> build_index(const ReadSet& text, unsigned q, bool sampled = false) {
  if (q == 0 || q > kMaxQ) throw input_error("q must be in [1, 16]");
  constexpr unsigned w = Index<W>::group_width;
  Index<W> ix;
  ix.q_ = q;
  const uint64_t space = uint64_t(1) << (2 * q);
  const size_t ngroups = size_t((space + w - 1) / w);
  ix.I.assign(ngroups, W(0));
  // valid positions: window fully inside one read (seq.hpp:135-137)
  std::vector<uint32_t> valid_pos, valid_code;
  for (uint32_t r = 0; r < text.count(); ++r) {
    const uint32_t n = text.lengths[r];
    for (uint32_t o = 0; o + q <= n; ++o) {
      valid_pos.push_back(uint32_t(uint64_t(r) * text.stride + o));
      valid_code.push_back(encode_qgram(text.read(r) + o, q));
    }
  }
  for (uint32_t g : valid_code) ix.I[g / w] |= W(1) << (g % w);
  std::vector<uint32_t> Sfull(ngroups + 1);
  uint64_t run = 0;
  for (size_t i = 0; i < ngroups; ++i) { Sfull[i] = uint32_t(run); run += std::popcount(ix.I[i]); }
  Sfull[ngroups] = uint32_t(run);
  const uint32_t distinct = uint32_t(run);
  std::vector<uint32_t> cnt(distinct + 1, 0);
  auto slot = [&](uint32_t g) {
    return Sfull[g / w] + Index<W>::rank_below(ix.I[g / w], g % w);
  };
  for (uint32_t g : valid_code) cnt[slot(g)]++;
  ix.S1.assign(distinct + 1, 0);
  run = 0;
  for (uint32_t b = 0; b < distinct; ++b) { ix.S1[b] = uint32_t(run); run += cnt[b]; }
  ix.S1[distinct] = uint32_t(run);
  ix.O.assign(valid_pos.size(), 0);
  std::vector<uint32_t> cur(ix.S1.begin(), ix.S1.end() - 1);
  for (size_t t = 0; t < valid_pos.size(); ++t) ix.O[cur[slot(valid_code[t])]++] = valid_pos[t];
  if (sampled) {  // sample_group_starts (qgroup_index.hpp:185-196)
    for (size_t i = 0; i < Sfull.size(); i += 2) ix.S.push_back(Sfull[i]);
    ix.sampled_ = true;
  } else {
    ix.S = std::move(Sfull);
  }
  return ix;
}

// ---------------------------------------------------------------- stage 2
// One candidate = (read, strand, chromosome, diagonal). Diagonals are
// chromosome-relative; strand 1 means RC(read) aligns forward at `diag`
// (Appendix B.2: d = p + o + q - n_r).
struct Cand {
  uint32_t read;
  uint32_t chrom;
  int64_t diag;
  uint8_t strand;
  friend bool operator<(const Cand& a, const Cand& b) {
    if (a.read != b.read) return a.read < b.read;
    if (a.strand != b.strand) return a.strand < b.strand;
    if (a.chrom != b.chrom) return a.chrom < b.chrom;
    return a.diag < b.diag;
  }
  friend bool operator==(const Cand& a, const Cand& b) {
    return a.read == b.read && a.strand == b.strand && a.chrom == b.chrom && a.diag == b.diag;
  }
};

// Alg. 2 over every reference position p of every chromosome
// whose q-gram window lies inside the chromosome and is not masked
// (SPEC.md:272, 302). Forward: d = p - (p' mod m), r = p' / m (oracles.hpp:46).
// `strands`: bit 0 forward, bit 1 reverse complement.
// `run_start`: emit only the leftmost q-gram of each run of consecutive q-gram
// matches on one diagonal. The multiset shrinks but the SET of candidates is
// unchanged (every run has exactly one leftmost member); the CUDA path relies on
// this and the tests check the set equality against the full multiset.
template <class IndexT>
std::vector<Cand> filter(const RefSet& ref, const ReadSet& reads, const IndexT& idx, unsigned q,
                         int strands = 3, bool run_start = false, unsigned threads = 1) {
  const auto& O = idx.positions();
  const uint32_t m = reads.stride;
  // the index's arrays, read directly so the random probes can be prefetched
  using W = std::decay_t<decltype(idx.occupancy()[0])>;
  constexpr unsigned gw = sizeof(W) * 8;
  const W* I = idx.occupancy().data();
  const uint32_t* S = idx.group_starts().data();
  const uint32_t* S1 = idx.occ_starts().data();
  const bool smp = idx.sampled();
  auto group_base = [&](size_t i) -> uint32_t {  // qgroup_index.hpp:91-96
    if (!smp) return S[i];
    const uint32_t even = S[i / 2];
    return (i & 1) ? even + uint32_t(std::popcount(I[i - 1])) : even;
  };
  struct Job { uint32_t c; uint64_t b, e; };
  std::vector<Job> jobs;
  const uint64_t step = 1 << 16;
  for (uint32_t c = 0; c < ref.chroms(); ++c) {
    const uint64_t Lc = ref.len(c);
    if (Lc < q) continue;
    for (uint64_t b = 0; b <= Lc - q; b += step) jobs.push_back({c, b, std::min(Lc - q + 1, b + step)});
  }
  std::vector<std::vector<Cand>> parts(jobs.size());
  parallel_chunks(jobs.size(), threads, [&](size_t jb, size_t je) {
    // Positions in blocks of kBlk: (1) rolling codes, prefetch the occupancy
    // word and group start of every lookup; (2) occupancy test + rank,
    // prefetch the S' pair; (3) expand the intervals. Same candidates as a
    // position-by-position index_pair loop (Alg. 2), with
    // ~2 x kBlk independent memory probes in flight instead of one.
    constexpr unsigned kBlk = 64;
    uint32_t code[2][kBlk];
    int64_t slot[2][kBlk];
    const uint32_t cmask = q == 16 ? 0xFFFFFFFFu : (1u << (2 * q)) - 1u;
    for (size_t j = jb; j < je; ++j) {
      const Job& J = jobs[j];
      const uint64_t cb = ref.chrom_begin[J.c];
      const uint8_t* R = ref.codes.data() + cb;
      auto& out = parts[j];
      uint32_t gf = 0;
      for (uint64_t p0 = J.b; p0 < J.e; p0 += kBlk) {
        const unsigned nb = unsigned(std::min<uint64_t>(kBlk, J.e - p0));
        for (unsigned t = 0; t < nb; ++t) {
          const uint64_t p = p0 + t;
          gf = p == J.b ? encode_qgram(R + p, q) : (((gf << 2) | R[p + q - 1]) & cmask);
          code[0][t] = gf;
          code[1][t] = rc_qgram(gf, q);
          for (int s = 0; s < 2; ++s) {
            __builtin_prefetch(I + code[s][t] / gw);
            __builtin_prefetch(S + (smp ? code[s][t] / gw / 2 : code[s][t] / gw));
          }
        }
        for (unsigned t = 0; t < nb; ++t)
          for (int s = 0; s < 2; ++s) {
            slot[s][t] = -1;
            if (!((strands >> s) & 1) || ref.masked(cb + p0 + t)) continue;
            const uint32_t g = code[s][t];
            const size_t i = g / gw;
            const unsigned jj = g % gw;
            const W word = I[i];
            if (!((word >> jj) & W(1))) continue;
            const uint32_t b = group_base(i) + IndexT::rank_below(word, jj);
            slot[s][t] = b;
            __builtin_prefetch(S1 + b);
          }
        for (unsigned t = 0; t < nb; ++t) {
          const uint64_t p = p0 + t;
          const bool prev_ok = p >= 1 && !ref.masked(cb + p - 1);
          if (slot[0][t] >= 0) {
            const uint32_t k0 = S1[slot[0][t]], k1 = S1[slot[0][t] + 1];
            for (uint32_t k = k0; k < k1; ++k) {
              const uint32_t r = O[k] / m, o = O[k] % m;
              if (run_start && prev_ok && o >= 1 && R[p - 1] == reads.read(r)[o - 1]) continue;
              out.push_back({r, J.c, int64_t(p) - int64_t(o), 0});
            }
          }
          if (slot[1][t] >= 0) {
            const uint32_t k0 = S1[slot[1][t]], k1 = S1[slot[1][t] + 1];
            for (uint32_t k = k0; k < k1; ++k) {
              const uint32_t r = O[k] / m, o = O[k] % m, n = reads.lengths[r];
              if (run_start && prev_ok && o + q + 1 <= n &&
                  uint8_t(3u - R[p - 1]) == reads.read(r)[o + q])
                continue;
              out.push_back({r, J.c, int64_t(p) + int64_t(o) + int64_t(q) - int64_t(n), 1});
            }
          }
        }
      }
    }
  });
  size_t total = 0;
  for (auto& v : parts) total += v.size();
  std::vector<Cand> all;
  all.reserve(total);
  for (auto& v : parts) all.insert(all.end(), v.begin(), v.end());
  return all;
}

// Sort by read id into `threads` buckets, sort each bucket in parallel.
template <class T, class Key>
void parallel_sort_by_read(std::vector<T>& v, uint32_t n_reads, unsigned threads, Key read_of) {
  threads = eff_threads(threads);
  if (threads <= 1 || v.size() < 100000 || n_reads == 0) { std::sort(v.begin(), v.end()); return; }
  const unsigned nb = threads * 4;
  auto bucket = [&](const T& x) { return unsigned(uint64_t(read_of(x)) * nb / n_reads); };
  // per-thread bucket counts over contiguous slices, then a parallel scatter
  const size_t per = (v.size() + threads - 1) / threads;
  std::vector<std::vector<size_t>> tc(threads, std::vector<size_t>(nb, 0));
  parallel_chunks(threads, threads, [&](size_t t0, size_t t1) {
    for (size_t t = t0; t < t1; ++t)
      for (size_t i = t * per; i < std::min(v.size(), (t + 1) * per); ++i) tc[t][bucket(v[i])]++;
  });
  std::vector<size_t> cnt(nb + 1, 0);
  for (unsigned b = 0; b < nb; ++b) {
    size_t run = cnt[b];
    for (unsigned t = 0; t < threads; ++t) {
      const size_t c = tc[t][b];
      tc[t][b] = run;
      run += c;
    }
    cnt[b + 1] = run;
  }
  std::vector<T> tmp(v.size());
  parallel_chunks(threads, threads, [&](size_t t0, size_t t1) {
    for (size_t t = t0; t < t1; ++t)
      for (size_t i = t * per; i < std::min(v.size(), (t + 1) * per); ++i) tmp[tc[t][bucket(v[i])]++] = v[i];
  });
  parallel_chunks(nb, threads, [&](size_t b0, size_t b1) {
    for (size_t b = b0; b < b1; ++b) std::sort(tmp.begin() + cnt[b], tmp.begin() + cnt[b + 1]);
  });
  v.swap(tmp);
}

// ---------------------------------------------------------------- stage 4
struct VRes {
  int k;           // banded semi-global edit distance
  uint32_t start;  // smallest window column at which an optimal alignment starts
};

// Banded semi-global DP over band j - i in [0, B) exactly as
// oracle::banded_semiglobal_distance (oracles.hpp:86-111); returns the whole
// bottom row (in-band cells only; others = kInf).
inline constexpr int kInf = std::numeric_limits<int>::max() / 4;
inline std::vector<int> banded_bottom_row(const uint8_t* rd, uint32_t n, const uint8_t* win,
                                          uint32_t L, unsigned B) {
  std::vector<int> prev(L + 1, kInf), cur(L + 1, kInf);
  for (uint32_t j = 0; j <= L; ++j) if (j < B) prev[j] = 0;
  for (uint32_t i = 1; i <= n; ++i) {
    std::fill(cur.begin(), cur.end(), kInf);
    const uint32_t jlo = i, jhi = std::min<uint64_t>(L, uint64_t(i) + B - 1);
    for (uint32_t j = jlo; j <= jhi; ++j) {
      int best = kInf;
      if (prev[j - 1] < kInf) best = std::min(best, prev[j - 1] + (rd[i - 1] == win[j - 1] ? 0 : 1));
      if (prev[j] < kInf) best = std::min(best, prev[j] + 1);
      if (cur[j - 1] < kInf) best = std::min(best, cur[j - 1] + 1);
      cur[j] = best;
    }
    std::swap(prev, cur);
  }
  return prev;
}

// DP restatement of validation. k from the forward banded DP; start from the
// same DP over the reversed read and window (Appendix B.5): the reversed
// bottom row at column j' is the cost of the best alignment starting at
// forward column L - j', so start = L - max{j' : bottom'[j'] == k}.
inline VRes validate_dp(const uint8_t* rd, uint32_t n, const uint8_t* win, uint32_t L, unsigned B) {
  const auto fwd = banded_bottom_row(rd, n, win, L, B);
  int k = kInf;
  for (int v : fwd) k = std::min(k, v);
  std::vector<uint8_t> rr(n), rw(L);  // reversed read and window
  for (uint32_t x = 0; x < n; ++x) rr[x] = rd[n - 1 - x];
  for (uint32_t x = 0; x < L; ++x) rw[x] = win[L - 1 - x];
  const auto bwd = banded_bottom_row(rr.data(), n, rw.data(), L, B);
  int64_t jmax = -1;
  for (uint32_t j = 0; j <= L; ++j) if (bwd[j] == k) jmax = j;
  return {k, jmax < 0 ? 0u : uint32_t(L - jmax)};
}

// Bit-parallel restatement (Myers 1999 / Hyyro 2003 banded),
// in diagonal coordinates over the reversed read and window: cell (i, t) is
// E'[i][i+t], t in [0,B). Per read row: Eq (match bits along the band), the
// carry chain Z of zero diagonal steps, then the new vertical deltas along t.
// One pass yields k = min_t D[n][t] and start = B-1-max{t : D[n][t] == k}.
// Requires L == n + B - 1 and B <= 64.
inline VRes validate_myers(const uint8_t* rd, uint32_t n, const uint8_t* win, uint32_t L, unsigned B) {
  if (B == 0 || B > kMaxBand || L != n + B - 1) throw input_error("band/window mismatch");
  const uint64_t mask = B == 64 ? ~uint64_t(0) : ((uint64_t(1) << B) - 1);
  // peq[c] bit y: reversed window rw[y] = win[L-1-y] equals base c (the
  // sentinel matches nothing); row i's Eq is the 64-bit slice at y = i-1
  const size_t nw = (L + 63) / 64 + 2;
  thread_local std::vector<uint64_t> peq;
  peq.assign(4 * nw, 0);
  for (uint32_t y = 0; y < L; ++y) {
    const uint8_t wc = win[L - 1 - y];
    if (wc < 4) peq[wc * nw + y / 64] |= uint64_t(1) << (y % 64);
  }
  uint64_t Pv = 0, Mv = 0;
  int64_t score0 = 0;  // D[i][0]
  for (uint32_t i = 1; i <= n; ++i) {
    const uint8_t c = rd[n - i];  // reversed read at row i: rr[i-1] = rd[n-1-(i-1)]
    const uint64_t* pw = peq.data() + size_t(c & 3) * nw;
    const uint32_t y = i - 1, wi = y / 64, sh = y % 64;
    const uint64_t Eq = c < 4 ? ((pw[wi] >> sh) | (sh ? pw[wi + 1] << (64 - sh) : 0)) & mask : 0;
    const uint64_t X = Eq | (Mv >> 1);
    const uint64_t Pp = Pv >> 1;
    const uint64_t Z = ((((X & Pp) + Pp) ^ Pp) | X) & mask;
    const uint64_t D1 = ~Z & mask;
    const uint64_t Bs = (D1 << 1) & mask;
    const uint64_t up = Bs & ~D1, dn = D1 & ~Bs, zr = ~(Pv | Mv);
    const uint64_t nP = ((Pv & ~up) | (zr & dn)) & mask & ~uint64_t(1);
    const uint64_t nM = ((Mv & ~dn) | (zr & up)) & mask & ~uint64_t(1);
    Pv = nP;
    Mv = nM;
    score0 += int64_t(D1 & 1);
  }
  int64_t v = score0, best = score0;
  unsigned tbest = 0;
  for (unsigned t = 1; t < B; ++t) {
    v += int64_t((Pv >> t) & 1) - int64_t((Mv >> t) & 1);
    if (v <= best) { best = v; tbest = t; }
  }
  return {int(best), B - 1 - tbest};
}

// ---------------------------------------------------------------- stages 4-5
struct Params {
  unsigned q = 16;
  unsigned band = 32;     // B
  unsigned pct = 80;      // identity threshold in percent
  int mode = 0;           // 0 best-stratum, 1 all
  int strands = 3;
};

struct Hit {
  uint32_t read, chrom, ref_start;
  uint16_t k;
  uint8_t strand;
  friend bool operator<(const Hit& a, const Hit& b) {
    if (a.read != b.read) return a.read < b.read;
    if (a.chrom != b.chrom) return a.chrom < b.chrom;
    if (a.ref_start != b.ref_start) return a.ref_start < b.ref_start;
    if (a.strand != b.strand) return a.strand < b.strand;
    return a.k < b.k;
  }
  friend bool operator==(const Hit& a, const Hit& b) {
    return a.read == b.read && a.chrom == b.chrom && a.ref_start == b.ref_start &&
           a.strand == b.strand && a.k == b.k;
  }
};

struct Validated {
  int k;
  uint32_t start;      // window column
  uint32_t ref_start;  // chromosome-relative, clamped (Appendix B.5)
  bool kept;           // 100*(n-k) >= pct*n (Appendix B.6)
  bool in_range;       // window overlaps the chromosome (Appendix B.4)
};

// Window W = ref[d-H, d-H+n+B-1) with H = floor((B-1)/2); bases outside the
// chromosome are the sentinel (Appendix B.4).
inline Validated validate_candidate(const RefSet& ref, const ReadSet& reads, const Cand& c,
                                    unsigned B, unsigned pct, bool use_dp = false) {
  const uint32_t n = reads.lengths[c.read];
  const int64_t H = (int64_t(B) - 1) / 2;
  const int64_t Lc = int64_t(ref.len(c.chrom));
  const uint32_t L = n + B - 1;
  const int64_t w0 = c.diag - H;
  Validated v{0, 0, 0, false, false};
  if (w0 + int64_t(L) <= 0 || w0 >= Lc) return v;
  v.in_range = true;
  thread_local std::vector<uint8_t> win, rd;  // reused: no allocation per candidate
  win.resize(L);
  const uint8_t* R = ref.codes.data() + ref.chrom_begin[c.chrom];
  for (uint32_t j = 0; j < L; ++j) {
    const int64_t x = w0 + j;
    win[j] = (x >= 0 && x < Lc) ? R[x] : kSentinel;
  }
  rd.resize(n);
  const uint8_t* src = reads.read(c.read);
  for (uint32_t j = 0; j < n; ++j) rd[j] = c.strand ? uint8_t(3u - src[n - 1 - j]) : src[j];
  const VRes r = use_dp ? validate_dp(rd.data(), n, win.data(), L, B)
                        : validate_myers(rd.data(), n, win.data(), L, B);
  v.k = r.k;
  v.start = r.start;
  v.ref_start = uint32_t(std::clamp<int64_t>(w0 + r.start, 0, Lc - 1));
  v.kept = uint64_t(100) * (uint64_t(n) - uint64_t(std::min<int64_t>(r.k, n))) >= uint64_t(pct) * n &&
           r.k <= int(n);
  return v;
}

// Hit-level dedup on (read, chrom, ref_start, strand) keeping the minimum k
// (SPEC.md:437-445), then best-stratum (k == min k of the read) or
// all. Input must be sorted by read. Output sorted by (read, chrom, ref_start, strand).
inline std::vector<Hit> stratify(std::vector<Hit> hits, int mode) {
  std::sort(hits.begin(), hits.end());
  std::vector<Hit> dd;
  for (size_t i = 0; i < hits.size(); ++i) {
    if (!dd.empty() && dd.back().read == hits[i].read && dd.back().chrom == hits[i].chrom &&
        dd.back().ref_start == hits[i].ref_start && dd.back().strand == hits[i].strand)
      continue;  // sorted: first of the group has the minimum k
    dd.push_back(hits[i]);
  }
  if (mode == 1) return dd;
  std::vector<Hit> out;
  size_t i = 0;
  while (i < dd.size()) {
    size_t j = i;
    uint16_t kmin = dd[i].k;
    while (j < dd.size() && dd[j].read == dd[i].read) { kmin = std::min(kmin, dd[j].k); ++j; }
    for (size_t t = i; t < j; ++t) if (dd[t].k == kmin) out.push_back(dd[t]);
    i = j;
  }
  return out;
}

// ---------------------------------------------------------------- traceback
// traceback_cigar, frozen as DESIGN.md section 2 item 9: the
// oriented read (n bases) against the chromosome from ref_start, global at the
// start (D[0][j] = j, D[i][0] = i), free at the end, cells restricted to the
// band |j - i| <= W with W = B - 1 (the validation band widened to both sides:
// it holds every alignment the validation band allowed from this start).
// Column j >= 1 is chromosome base ref_start + j - 1 (kSentinel past the end).
// End = the largest j with minimal D[n][j] among the columns inside the
// chromosome (or j = max(0, n - W) if none is in the band). Traceback prefers M (diagonal),
// then I (read base against no reference base), then D; leading D operations
// are dropped and move ref_start right ("possibly improved ref_start").
// ops are BAM-style: length << 4 | op with M = 0, I = 1, D = 2.
struct Cigar {
  uint32_t ref_start = 0;
  int edits = 0;  // I + D + mismatched M columns of the reported alignment
  std::vector<uint32_t> ops;
  std::string str() const {
    std::string o;
    for (uint32_t x : ops) o += std::to_string(x >> 4) + "MID"[x & 15];
    return o;
  }
};

inline Cigar traceback_cigar(const uint8_t* rd, uint32_t n, const uint8_t* chrom, int64_t Lc, uint32_t ref_start,
                             unsigned B) {
  if (B == 0 || B > kMaxBand) throw input_error("band must be in [1, 64]");
  const int64_t W = int64_t(B) - 1, J = int64_t(n) + W;
  auto base = [&](int64_t j) -> uint8_t {  // column j >= 1
    const int64_t x = int64_t(ref_start) + j - 1;
    return x >= 0 && x < Lc ? chrom[x] : kSentinel;
  };
  std::vector<std::vector<int>> D(n + 1, std::vector<int>(size_t(J + 1), kInf));
  auto in_band = [&](int64_t i, int64_t j) { return j >= 0 && j <= J && j - i <= W && i - j <= W; };
  for (int64_t j = 0; j <= std::min<int64_t>(J, W); ++j) D[0][j] = int(j);
  for (int64_t i = 1; i <= int64_t(n); ++i)
    for (int64_t j = std::max<int64_t>(0, i - W); j <= std::min(J, i + W); ++j) {
      int b = kInf;
      if (j == 0) b = int(i);
      else {
        if (D[i - 1][j - 1] < kInf) b = std::min(b, D[i - 1][j - 1] + (rd[i - 1] == base(j) ? 0 : 1));
        if (in_band(i - 1, j) && D[i - 1][j] < kInf) b = std::min(b, D[i - 1][j] + 1);
        if (D[i][j - 1] < kInf) b = std::min(b, D[i][j - 1] + 1);
      }
      D[i][j] = b;
    }
  // end column: in the chromosome when the band reaches it (no alignment
  // running into the sentinels past its end), the largest j on ties (a
  // trailing mismatch or deletion rather than an insertion)
  const int64_t jlo = std::max<int64_t>(0, int64_t(n) - W);
  const int64_t jhi = std::min(J, std::max(Lc - int64_t(ref_start), jlo));
  int64_t je = -1;
  for (int64_t j = jlo; j <= jhi; ++j)
    if (je < 0 || D[n][j] <= D[n][je]) je = j;
  Cigar c;
  c.ref_start = ref_start;
  c.edits = D[n][je];
  std::vector<uint32_t> rev;  // ops from the end
  auto push = [&](uint32_t op) {
    if (!rev.empty() && (rev.back() & 15) == op) rev.back() += 16;
    else rev.push_back(16 | op);
  };
  int64_t i = n, j = je;
  while (i > 0 || j > 0) {
    if (i == 0) { push(2); --j; continue; }
    if (j == 0) { push(1); --i; continue; }
    const int cur = D[i][j];
    if (D[i - 1][j - 1] < kInf && D[i - 1][j - 1] + (rd[i - 1] == base(j) ? 0 : 1) == cur) { push(0); --i; --j; }
    else if (in_band(i - 1, j) && D[i - 1][j] < kInf && D[i - 1][j] + 1 == cur) { push(1); --i; }
    else { push(2); --j; }
  }
  if (!rev.empty() && (rev.back() & 15) == 2) {  // leading deletions
    c.ref_start += rev.back() >> 4;
    c.edits -= int(rev.back() >> 4);
    rev.pop_back();
  }
  c.ops.assign(rev.rbegin(), rev.rend());
  return c;
}

struct Stats {
  uint64_t raw = 0, unique = 0, validated_kept = 0, hits = 0;
  // wall seconds per stage: index build (filled by the caller), filtration,
  // sort + unique, validation, strata
  double sec_index = 0, sec_filter = 0, sec_sort = 0, sec_validate = 0, sec_strata = 0;
};
inline double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// run_map core for one read buffer: filter every chromosome,
// dedup candidates, validate, stratify.
template <class IndexT>
std::vector<Hit> map_with_index(const RefSet& ref, const ReadSet& reads, const IndexT& idx,
                                const Params& P, unsigned threads = 1, Stats* st = nullptr) {
  if (P.band == 0 || P.band > kMaxBand) throw input_error("band must be in [1, 64]");
  if (P.pct > 100) throw input_error("percent identity must be in [0, 100]");
  auto t0 = std::chrono::steady_clock::now();
  std::vector<Cand> c = filter(ref, reads, idx, P.q, P.strands, /*run_start=*/false, threads);
  if (st) st->raw = c.size();
  if (st) st->sec_filter = seconds_since(t0);
  t0 = std::chrono::steady_clock::now();
  parallel_sort_by_read(c, reads.count(), threads, [](const Cand& x) { return x.read; });
  c.erase(std::unique(c.begin(), c.end()), c.end());
  if (st) st->unique = c.size();
  if (st) st->sec_sort = seconds_since(t0);
  t0 = std::chrono::steady_clock::now();
  std::vector<Hit> hits_all(c.size());
  std::vector<uint8_t> keep(c.size(), 0);
  parallel_chunks(c.size(), threads, [&](size_t b, size_t e) {
    for (size_t i = b; i < e; ++i) {
      const Validated v = validate_candidate(ref, reads, c[i], P.band, P.pct);
      if (v.in_range && v.kept) {
        keep[i] = 1;
        hits_all[i] = {c[i].read, c[i].chrom, v.ref_start, uint16_t(v.k), c[i].strand};
      }
    }
  });
  std::vector<Hit> kept;
  for (size_t i = 0; i < c.size(); ++i) if (keep[i]) kept.push_back(hits_all[i]);
  if (st) st->validated_kept = kept.size();
  if (st) st->sec_validate = seconds_since(t0);
  t0 = std::chrono::steady_clock::now();
  // stratify per contiguous read range, in parallel (input sorted by read)
  threads = eff_threads(threads);
  std::vector<size_t> cuts{0};
  const size_t per = std::max<size_t>(1, kept.size() / (threads * 4));
  for (size_t x = per; x < kept.size(); x += per) {
    while (x < kept.size() && kept[x].read == kept[x - 1].read) ++x;
    if (x < kept.size() && x > cuts.back()) cuts.push_back(x);
  }
  cuts.push_back(kept.size());
  std::vector<std::vector<Hit>> outs(cuts.size() - 1);
  parallel_chunks(outs.size(), threads, [&](size_t b, size_t e) {
    for (size_t t = b; t < e; ++t)
      outs[t] = stratify(std::vector<Hit>(kept.begin() + cuts[t], kept.begin() + cuts[t + 1]), P.mode);
  });
  std::vector<Hit> out;
  for (auto& o : outs) out.insert(out.end(), o.begin(), o.end());
  if (st) st->hits = out.size();
  if (st) st->sec_strata = seconds_since(t0);
  return out;
}

}  // namespace qgm_oracle
