// synth.cpp -- deterministic synthetic inputs for tests and bench.py
// (SURVEY.md section 8(d)): random references, a repetitive reference for the
// candidate-explosion config, and simulated reads with substitutions /
// insertions / deletions in ratio 0.8 / 0.1 / 0.1, reverse-complemented with
// probability 1/2. Host-only, no CUDA; built into libqgm_synth.so.
//
// Randomness: splitmix64-seeded xoshiro256** streams, one per read / per
// chromosome chunk, so results do not depend on the thread count.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

namespace {

struct Rng {
  uint64_t s[4];
  static uint64_t splitmix(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  explicit Rng(uint64_t seed) {
    for (auto& v : s) v = splitmix(seed);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
    s[2] ^= t; s[3] = rotl(s[3], 45);
    return r;
  }
  double uniform() { return double(next() >> 11) * (1.0 / 9007199254740992.0); }
  uint64_t below(uint64_t n) { return n ? next() % n : 0; }
};

template <class Fn>
void parallel(size_t n, Fn&& fn) {
  unsigned T = std::max(1u, std::thread::hardware_concurrency());
  T = std::min<unsigned>(T, 64);
  if (n < 4096) T = 1;
  std::vector<std::thread> ws;
  const size_t chunk = (n + T - 1) / T;
  for (unsigned t = 0; t < T; ++t) {
    const size_t b = std::min(n, t * chunk), e = std::min(n, b + chunk);
    if (b >= e) break;
    ws.emplace_back([&fn, b, e] { fn(b, e); });
  }
  for (auto& w : ws) w.join();
}

void random_fill(uint64_t seed, uint64_t total, uint8_t* out) {
  const uint64_t block = 1 << 20;
  const uint64_t nb = (total + block - 1) / block;
  parallel(nb, [&](size_t b0, size_t b1) {
    for (size_t b = b0; b < b1; ++b) {
      Rng rng(seed * 0x100000001B3ull + b);
      const uint64_t s = b * block, e = std::min(total, s + block);
      for (uint64_t i = s; i < e; i += 32) {
        uint64_t x = rng.next();
        for (uint64_t j = i; j < std::min(e, i + 32); ++j, x >>= 2) out[j] = uint8_t(x & 3);
      }
    }
  });
}

}  // namespace

extern "C" {

// total random bases (A/C/G/T uniform), 1 byte each.
int qgs_random_reference(uint64_t seed, uint64_t total, uint8_t* out) {
  random_fill(seed, total, out);
  return 0;
}

// Repetitive reference (config C5): a random backbone overwritten with tandem
// arrays (unit 2..500 bp, 10..10^4 copies, log-uniform; about 10% of the
// sequence) and segmental duplications (1..10 kb, 2..100 copies, 0..2%
// substitutions; about 10% of the sequence).
int qgs_repetitive_reference(uint64_t seed, uint64_t total, uint8_t* out) {
  random_fill(seed, total, out);
  Rng rng(seed ^ 0xC5C5C5C5ull);
  auto logu = [&](double lo, double hi) { return std::exp(std::log(lo) + rng.uniform() * (std::log(hi) - std::log(lo))); };
  uint64_t tandem = 0;
  while (tandem < total / 10 && total > 20000) {
    const uint64_t unit = uint64_t(logu(2, 500));
    uint64_t copies = uint64_t(logu(10, 1e4));
    uint64_t len = std::min<uint64_t>(unit * copies, total / 50);
    const uint64_t pos = rng.below(total - len);
    std::vector<uint8_t> u(unit);
    for (auto& b : u) b = uint8_t(rng.next() & 3);
    for (uint64_t i = 0; i < len; ++i) out[pos + i] = u[i % unit];
    tandem += len;
  }
  uint64_t dup = 0;
  while (dup < total / 10 && total > 200000) {
    const uint64_t len = 1000 + rng.below(9001);
    const uint64_t copies = 2 + uint64_t(logu(1, 99));
    const uint64_t src = rng.below(total - len);
    std::vector<uint8_t> seg(out + src, out + src + len);
    const double div = rng.uniform() * 0.02;
    for (uint64_t c = 1; c < copies; ++c) {
      const uint64_t dst = rng.below(total - len);
      for (uint64_t i = 0; i < len; ++i) {
        uint8_t b = seg[i];
        if (rng.uniform() < div) b = uint8_t((b + 1 + rng.below(3)) & 3);
        out[dst + i] = b;
      }
      dup += len;
    }
  }
  return 0;
}

// Simulated reads of exactly `len` bases (len <= stride) sampled uniformly
// from the chromosomes (weighted by length). Per base: with probability err an
// edit, 80% substitution / 10% insertion / 10% deletion. Half of the reads
// are reverse-complemented. Truth = (chrom, forward start, strand).
int qgs_simulate_reads(uint64_t seed, const uint8_t* ref, const uint64_t* cb, uint32_t n_chrom, uint32_t n_reads,
                       uint32_t len, double err, uint32_t stride, uint8_t* codes, uint32_t* lengths,
                       uint32_t* truth_chrom, uint64_t* truth_pos, uint8_t* truth_strand) {
  if (len > stride || n_chrom == 0) return 1;
  const uint64_t total = cb[n_chrom];
  const uint64_t slack = uint64_t(len) + len / 2 + 64;
  parallel(n_reads, [&](size_t b, size_t e) {
    std::vector<uint8_t> frag;
    for (size_t r = b; r < e; ++r) {
      Rng rng(seed * 0x9E3779B97F4A7C15ull + r * 0xD1B54A32D192ED03ull + 1);
      uint32_t c = 0;
      uint64_t Lc = 0;
      for (int tries = 0; tries < 64; ++tries) {
        const uint64_t x = rng.below(total);
        c = uint32_t(std::upper_bound(cb, cb + n_chrom + 1, x) - cb - 1);
        Lc = cb[c + 1] - cb[c];
        if (Lc > slack) break;
      }
      uint8_t* out = codes + size_t(r) * stride;
      std::fill(out, out + stride, 0);
      if (Lc <= slack) {  // degenerate tiny reference: random read
        for (uint32_t i = 0; i < len; ++i) out[i] = uint8_t(rng.next() & 3);
        lengths[r] = len;
        if (truth_chrom) truth_chrom[r] = c;
        if (truth_pos) truth_pos[r] = 0;
        if (truth_strand) truth_strand[r] = 0;
        continue;
      }
      const uint64_t start = rng.below(Lc - slack);
      const uint8_t* R = ref + cb[c] + start;
      frag.clear();
      uint64_t p = 0;
      while (frag.size() < len) {
        const double u = rng.uniform();
        if (u < err * 0.8) {
          frag.push_back(uint8_t((R[p] + 1 + rng.below(3)) & 3));
          ++p;
        } else if (u < err * 0.9) {
          frag.push_back(uint8_t(rng.next() & 3));
        } else if (u < err) {
          ++p;
        } else {
          frag.push_back(R[p]);
          ++p;
        }
      }
      const bool rc = rng.next() & 1;
      for (uint32_t i = 0; i < len; ++i) out[i] = rc ? uint8_t(3 - frag[len - 1 - i]) : frag[i];
      lengths[r] = len;
      if (truth_chrom) truth_chrom[r] = c;
      if (truth_pos) truth_pos[r] = start;
      if (truth_strand) truth_strand[r] = rc;
    }
  });
  return 0;
}

// 1-byte codes -> 2-bit MSB-first words (the qgm_c.h layout), multithreaded.
int qgs_pack(const uint8_t* codes, uint64_t n, uint64_t* words) {
  const uint64_t nw = (n + 31) / 32;
  parallel(nw, [&](size_t b, size_t e) {
    for (size_t k = b; k < e; ++k) {
      uint64_t w = 0;
      const uint64_t s = k * 32, t = std::min<uint64_t>(n, s + 32);
      for (uint64_t j = s; j < t; ++j) w |= uint64_t(codes[j] & 3) << (62 - 2 * (j - s));
      words[k] = w;
    }
  });
  return 0;
}

// n_reads reads of `stride` codes -> n_reads * ceil(stride/32) words.
int qgs_pack_reads(const uint8_t* codes, uint32_t stride, uint32_t n_reads, uint64_t* words) {
  const uint32_t W = (stride + 31) / 32;
  parallel(n_reads, [&](size_t b, size_t e) {
    for (size_t r = b; r < e; ++r) {
      const uint8_t* c = codes + r * stride;
      for (uint32_t k = 0; k < W; ++k) {
        uint64_t w = 0;
        const uint32_t s = k * 32, t = std::min<uint32_t>(stride, s + 32);
        for (uint32_t j = s; j < t; ++j) w |= uint64_t(c[j] & 3) << (62 - 2 * (j - s));
        words[r * W + k] = w;
      }
    }
  });
  return 0;
}

}  // extern "C"
