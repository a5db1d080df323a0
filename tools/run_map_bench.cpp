// FASTQ -> SAM throughput of run_map (include/qgmap/pipeline.hpp) on one GPU:
// a synthetic 100 Mbp reference and N simulated 100 bp reads (3% edits) as
// in-memory FASTQ, SAM written to /dev/null. Prints reads/s per stage mix.
// Build: make tools/run_map_bench (see Makefile), run on the GPU box.
#include <chrono>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>

#include "qgmap/pipeline.hpp"

using namespace qgmap;

int main(int argc, char** argv) {
  const std::size_t L = argc > 1 ? std::stoull(argv[1]) : 100000000ull;
  const std::size_t N = argc > 2 ? std::stoull(argv[2]) : 2000000ull;
  std::mt19937_64 g(7);
  std::string chrom(L, 'A');
  for (auto& c : chrom) c = "ACGT"[g() & 3];
  rng_engine rng(1);
  Reference ref;
  ref.add_chromosome("chr1", chrom, rng);
  DeviceReference dref(ref);
  std::ostringstream fq;
  std::uniform_real_distribution<double> U(0, 1);
  for (std::size_t r = 0; r < N; ++r) {
    std::size_t p = g() % (L - 200);
    std::string s;
    while (s.size() < 100) {
      const double u = U(g);
      const char b = chrom[p];
      if (u < 0.024) { s += "ACGT"[(std::string("ACGT").find(b) + 1 + g() % 3) & 3]; ++p; }
      else if (u < 0.027) s += "ACGT"[g() & 3];
      else if (u < 0.03) ++p;
      else { s += b; ++p; }
    }
    if (g() & 1) s = reverse_complement(s);
    fq << "@r" << r << '\n' << s << "\n+\n" << std::string(100, 'I') << '\n';
  }
  const std::string text = fq.str();
  MapParams p;
  p.q = 16;
  p.mode = StratumMode::all;
  RunOptions o;
  o.batch_reads = 1 << 20;
  for (int rep = 0; rep < 2; ++rep) {
    std::istringstream in(text);
    std::ofstream out("/dev/null");
    const auto t0 = std::chrono::steady_clock::now();
    const RunStats st = run_map(in, out, ref, dref, p, o);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::cout << "run_map: " << st.reads << " reads, " << st.records << " SAM records, " << st.buffers
              << " buffers, " << s << " s, " << st.reads / s / 1e6 << " M reads/s (FASTQ in memory, SAM to /dev/null)"
              << std::endl;
  }
}
