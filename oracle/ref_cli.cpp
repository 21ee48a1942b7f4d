// Test-infrastructure driver around the UNMODIFIED reference headers
// (/root/reference/proj/include/ppsim, compiled where they lie; nothing is copied).
// It is the oracle for the schedule path: tests/ and bench.py's reference arm call it
// as a checker/baseline, never as part of the product.
//
//   ppsim_ref <policy> <depth> <devices> <fwd> <bwd> <update> <comm> <inj> <pipes> <thr> <M>
//             <zero> <mode> [warmup]
//   costs are "n" or "n/d" (uniform across stages; "a,b,c,..." gives per-stage costs)
//   mode: csv | summary | json | bench <reps>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <string>
#include <vector>

#include "ppsim/analysis.hpp"
#include "ppsim/builder.hpp"
#include "ppsim/engine.hpp"
#include "ppsim/serialize.hpp"
#include "ppsim/validate.hpp"

using namespace ppsim;

static std::vector<Rat> costs(const std::string& s, int depth) {
  std::vector<Rat> out;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ',')) out.push_back(Rat::parse(tok));
  if (out.size() == 1) out.assign(static_cast<std::size_t>(depth), out[0]);
  return out;
}

int main(int argc, char** argv) {
  if (argc < 14) {
    std::fprintf(stderr, "usage: see header\n");
    return 2;
  }
  try {
    auto pol = policy_from_name(argv[1]);
    if (!pol) throw std::invalid_argument("unknown policy");
    ClusterSpec cl;
    cl.depth = std::atoi(argv[2]);
    cl.devices = std::atoi(argv[3]);
    cl.fwd_cost = costs(argv[4], cl.depth);
    cl.bwd_cost = costs(argv[5], cl.depth);
    cl.update_cost = Rat::parse(argv[6]);
    cl.comm_cost = Rat::parse(argv[7]);
    PolicyConfig cfg;
    cfg.policy = *pol;
    cfg.injection_limit = std::atoi(argv[8]);
    cfg.num_pipelines = std::atoi(argv[9]);
    cfg.accumulation_threshold = std::atoi(argv[10]);
    cfg.num_minibatches = std::atoi(argv[11]);
    cfg.zero_enabled = std::atoi(argv[12]) != 0;
    const std::string mode = argv[13];
    const int warm = argc > 14 ? std::atoi(argv[14]) : 1;
    if (mode == "csv") {
      auto tl = simulate(build(cfg, cl), cl);
      std::fputs(timeline_csv(tl).c_str(), stdout);
    } else if (mode == "summary") {
      auto tl = simulate(build(cfg, cl), cl);
      ordered_json j;
      j["makespan"] = rat_json(tl.makespan);
      try {
        j["bubble_ratio"] = bubble_ratio(tl, warm).str();
      } catch (const std::exception& e) {
        j["bubble_ratio"] = nullptr;
      }
      j["bubble_w0"] = bubble_ratio(tl, 0).str();
      auto mm = mismatch_report(tl);
      j["mismatch"] = mismatch_json(mm);
      j["windows"] = window_json(window_mismatch(tl, cl.depth));
      j["memory"] = memory_json(memory_report(tl, cfg, MemoryModel{}));
      j["causality_issues"] = validate_causality(tl, cl).size();
      j["overlap_issues"] = validate_non_overlap(tl).size();
      std::puts(j.dump().c_str());
    } else if (mode == "json") {
      // the reference's serialize.hpp emitters, one dump() per line
      auto tl = simulate(build(cfg, cl), cl);
      std::puts(timeline_json(tl).dump().c_str());
      std::puts(mismatch_json(mismatch_report(tl)).dump().c_str());
      std::puts(window_json(window_mismatch(tl, cl.depth)).dump().c_str());
      std::puts(memory_json(memory_report(tl, cfg, MemoryModel{})).dump().c_str());
    } else if (mode == "bench") {
      // build + simulate + mismatch_report, single-threaded, as the reference runs
      const int reps = argc > 14 ? std::atoi(argv[14]) : 10;
      auto t0 = std::chrono::steady_clock::now();
      std::size_t sink = 0;
      for (int r = 0; r < reps; ++r) {
        auto tl = simulate(build(cfg, cl), cl);
        sink += mismatch_report(tl).entries.size();
      }
      double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      std::printf("{\"reps\": %d, \"seconds\": %.6f, \"sink\": %zu}\n", reps, s, sink);
    } else {
      throw std::invalid_argument("unknown mode");
    }
  } catch (const std::exception& e) {
    std::printf("ERROR %s\n", e.what());
    return 1;
  }
  return 0;
}
