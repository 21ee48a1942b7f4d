// Prints the ppsim/serialize.hpp emitters (nlohmann::ordered_json, .dump()) for one AMDP
// schedule, one JSON document per line: timeline, mismatch, window, memory.  The CPU test
// (tests/test_reference_cpp_suites.py) compares them with the reference's own emitters run
// on the same schedule (oracle/_ref/ppsim_ref json mode).
#include <cstdio>
#include <cstdlib>

#include "ppsim/analysis.hpp"
#include "ppsim/builder.hpp"
#include "ppsim/engine.hpp"
#include "ppsim/serialize.hpp"

int main(int argc, char** argv) {
  const int depth = argc > 1 ? std::atoi(argv[1]) : 4;
  const int thr = argc > 2 ? std::atoi(argv[2]) : 8;
  const int M = argc > 3 ? std::atoi(argv[3]) : 32;
  const int bwd = argc > 4 ? std::atoi(argv[4]) : 2;
  const bool zero = argc > 5 ? std::atoi(argv[5]) != 0 : true;
  ppsim::PolicyConfig cfg;
  cfg.policy = ppsim::Policy::AMDP;
  cfg.injection_limit = 2;
  cfg.num_pipelines = depth / 2;
  cfg.accumulation_threshold = thr;
  cfg.num_minibatches = M;
  cfg.zero_enabled = zero;
  const auto cl = ppsim::ClusterSpec::uniform(depth, depth, ppsim::Rat(1), ppsim::Rat(bwd));
  const auto tl = ppsim::simulate(ppsim::build(cfg, cl), cl);
  std::printf("%s\n", ppsim::timeline_json(tl).dump().c_str());
  std::printf("%s\n", ppsim::mismatch_json(ppsim::mismatch_report(tl)).dump().c_str());
  std::printf("%s\n", ppsim::window_json(ppsim::window_mismatch(tl, depth)).dump().c_str());
  std::printf("%s\n", ppsim::memory_json(ppsim::memory_report(tl, cfg, ppsim::MemoryModel{})).dump().c_str());
  return 0;
}
