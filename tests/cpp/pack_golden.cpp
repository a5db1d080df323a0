// Prints pack_reads(reads, stride, q, rng(seed)) codes and valid positions using
// this repo's include/qgmap/seq.hpp (compared to the reference's golden output
// by tests/test_oracle_pins.py).
#include <cstdio>
#include <cstdlib>
#include "qgmap/seq.hpp"
int main(int argc, char** argv) {
  const unsigned stride = unsigned(std::atoi(argv[1])), q = unsigned(std::atoi(argv[2]));
  qgmap::rng_engine rng(std::strtoull(argv[3], nullptr, 10));
  std::vector<std::string> reads(argv + 4, argv + argc);
  const auto t = qgmap::pack_reads(reads, stride, q, rng);
  for (auto c : t.codes) std::printf("%u ", unsigned(c));
  std::printf("\n");
  for (auto p : t.valid_qgram_positions) std::printf("%u ", p);
  std::printf("\n");
}
