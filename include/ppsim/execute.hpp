// ppsim::execute — the GPU counterpart of ppsim::simulate (engine.hpp:28).
//
//   auto g  = ppsim::build(cfg, declared);          // unchanged reference API
//   auto tl = ppsim::simulate(g, declared);         // declared-cost order (the trace)
//   auto run = ppsim::execute(cfg, declared, opts, inputs, labels);  // same order on B200s
//   ppsim::bubble_ratio(run.timeline, 1);           // analyses apply unchanged
//
// execute() builds the same TaskGraph from (cfg, declared), replays its simulate() dispatch
// order on this process's GPU (logical devices folded world_size ways), and returns the
// measured Timeline (integer nanoseconds as Rat) plus the per-minibatch losses.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "amdp_engine.h"
#include "ppsim/ppsim.hpp"

namespace ppsim {

struct ExecuteOptions {
  amdp_model_config model{};
  amdp_opt_args optimizer{AMDP_OPT_ADAMW, 3e-4f, 0.9f, 0.95f, 1e-8f, 0.f, 1e-8f, 1e6f, 1.f, 1};
  int world_size = 1;
  int rank = 0;
  int comm_backend = AMDP_COMM_IPC;   // world_size > 1: peer-memory data plane or NCCL
  const uint8_t* nccl_id = nullptr;  // AMDP_COMM_NCCL: amdp_nccl_unique_id() from rank 0
  // AMDP_COMM_IPC with world_size > 1: gathers this rank's descriptor from every rank and
  // returns all of them in rank order (MPI_Allgather, torch.distributed, a shared file ...)
  std::function<std::vector<std::string>(const std::string&)> allgather;
  uint64_t data_seed = 1234;
};

struct ExecuteResult {
  Timeline timeline;          // measured, this rank's logical devices
  std::vector<float> losses;  // per minibatch (valid on the rank hosting the last stage)
  amdp_run_stats stats{};
  // per-logical-device F/B order with the parameter version each task read on the GPU
  // (device,kind,stage,minibatch,pipeline,window,preloaded,version; = version_trace_csv)
  std::string version_trace;
};

// Throws std::invalid_argument for configurations the executor does not run (non-AMDP
// policy, ZeRO disabled, depth not divisible by world_size) and std::runtime_error for
// CUDA/NCCL failures.  inputs/labels: host [num_minibatches][tokens_per_minibatch].
PPSIM_API ExecuteResult execute(const PolicyConfig& cfg, const ClusterSpec& declared,
                                const ExecuteOptions& opt, const int32_t* inputs,
                                const int32_t* labels);

}  // namespace ppsim
