// TEST/MEASUREMENT INFRASTRUCTURE ONLY: a command-line driver around the
// reference's own benchmark harness (nttkit::bench::run_bench / emit,
// /root/reference/proj/include/nttkit/bench.hpp:234-400), compiled from the
// unmodified reference headers into oracle/_ref/refbench by oracle/Makefile.
// tools/bench_records.py runs it to obtain the reference's records (naive,
// optimized_64, optimized_52, float) and appends the GPU rows in the same
// CSV format.
//
//   refbench [--sizes 1024,4096,16384] [--q-bits 50] [--kernels fwd_ntt,...]
//            [--reps 10] [--format csv|json|table]
#include <cstdlib>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "nttkit/bench.hpp"

namespace {
std::vector<std::string> split(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string t;
  while (std::getline(ss, t, ',')) out.push_back(t);
  return out;
}
}  // namespace

int main(int argc, char** argv) {
  nttkit::bench::Config cfg;
  nttkit::bench::Format fmt = nttkit::bench::Format::csv;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    if (k == "--sizes") {
      cfg.sizes.clear();
      for (auto& t : split(v)) cfg.sizes.push_back(std::stoull(t));
    } else if (k == "--q-bits") {
      cfg.q_bits.clear();
      for (auto& t : split(v)) cfg.q_bits.push_back(static_cast<unsigned>(std::stoul(t)));
    } else if (k == "--kernels") {
      cfg.kernels.clear();
      for (auto& t : split(v)) {
        auto kk = nttkit::bench::kernel_from_string(t);
        if (!kk) {
          std::cerr << "unknown kernel " << t << "\n";
          return 2;
        }
        cfg.kernels.push_back(*kk);
      }
    } else if (k == "--reps") {
      cfg.reps = static_cast<unsigned>(std::stoul(v));
    } else if (k == "--format") {
      fmt = v == "json" ? nttkit::bench::Format::json
                        : (v == "table" ? nttkit::bench::Format::table : nttkit::bench::Format::csv);
    } else {
      std::cerr << "unknown option " << k << "\n";
      return 2;
    }
  }
  try {
    const auto records = nttkit::bench::run_bench(cfg);
    nttkit::bench::emit(records, fmt, std::cout);
  } catch (const std::exception& e) {
    std::cerr << "refbench: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
