// One rank of a multi-rank ppsim::execute (the C++ drop-in path of the multi-GPU data plane):
//   execute_multirank <rank> <world> <exchange dir>
// Ranks exchange their communication descriptors through ExecuteOptions::allgather, here a
// shared directory (each rank writes r<k>.bin, then reads everyone's) — any transport works
// (MPI_Allgather, a key-value store, ...).  Runs the tiny GPT config of execute_tiny.cpp and
// prints this rank's losses (0 where another rank ran the minibatch's last stage), version
// trace and stats as JSON; tests/test_cpp_execute_gpu.py runs two ranks on one GPU and checks
// them against the single-rank program.
#include <chrono>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "ppsim/builder.hpp"
#include "ppsim/engine.hpp"
#include "ppsim/execute.hpp"
#include "ppsim/serialize.hpp"

static std::vector<std::string> file_allgather(const std::string& dir, int rank, int world, const std::string& mine) {
  {
    const std::string tmp = dir + "/r" + std::to_string(rank) + ".tmp";
    std::ofstream(tmp, std::ios::binary).write(mine.data(), static_cast<std::streamsize>(mine.size()));
    std::rename(tmp.c_str(), (dir + "/r" + std::to_string(rank) + ".bin").c_str());  // atomic publish
  }
  std::vector<std::string> all(static_cast<size_t>(world));
  for (int r = 0; r < world; ++r) {
    const std::string path = dir + "/r" + std::to_string(r) + ".bin";
    for (int tries = 0;; ++tries) {
      std::ifstream in(path, std::ios::binary);
      if (in) {
        all[static_cast<size_t>(r)].assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
        break;
      }
      if (tries > 60000) throw std::runtime_error("allgather: timed out waiting for " + path);
      std::this_thread::sleep_for(std::chrono::milliseconds(5));
    }
  }
  return all;
}

int main(int argc, char** argv) {
  if (argc < 4) return 2;
  const int rank = std::atoi(argv[1]), world = std::atoi(argv[2]);
  const std::string dir = argv[3];
  ppsim::PolicyConfig cfg;
  cfg.policy = ppsim::Policy::AMDP;
  cfg.injection_limit = 2;
  cfg.num_pipelines = 2;
  cfg.accumulation_threshold = 8;
  cfg.num_minibatches = 32;
  cfg.zero_enabled = true;
  const auto declared = ppsim::ClusterSpec::uniform(4, 4, ppsim::Rat(1), ppsim::Rat(1));
  static const int parts[4] = {1, 1, 1, 1};
  ppsim::ExecuteOptions opt;
  opt.model = amdp_model_config{4, 128, 4, 512, 1024, 64, 4, 1, 0.02f, 1e-5f, 1234, parts, 0, 0, 0};
  opt.optimizer = amdp_opt_args{AMDP_OPT_ADAMW, 1e-3f, 0.9f, 0.95f, 1e-8f, 0.f, 1e-8f, 1e6f, 1.f, 1};
  opt.world_size = world;
  opt.rank = rank;
  opt.allgather = [&](const std::string& mine) { return file_allgather(dir, rank, world, mine); };
  const int T = 4 * 64;
  std::vector<int32_t> inputs(static_cast<size_t>(cfg.num_minibatches) * T), labels(inputs.size());
  if (amdp_synthetic_tokens(&opt.model, opt.data_seed, 0, cfg.num_minibatches, inputs.data(), labels.data()) != 0)
    return 2;
  const auto run = ppsim::execute(cfg, declared, opt, inputs.data(), labels.data());
  ppsim::ordered_json j;
  j["rank"] = rank;
  j["losses"] = run.losses;
  j["version_trace"] = run.version_trace;
  j["p2p_bytes_sent"] = run.stats.p2p_bytes_sent;
  j["overlap_issues"] = ppsim::validate_non_overlap(run.timeline).size();
  std::puts(j.dump().c_str());
  return 0;
}
