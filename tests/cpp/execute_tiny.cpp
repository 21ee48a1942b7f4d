// A C++ consumer of the drop-in API: the reference's build/simulate calls plus
// ppsim::execute (the GPU counterpart of simulate) on the tiny GPT config (D=4, 2 pipelines,
// 8 minibatches per window, 4 windows), linked against libamdp.so.  Prints one JSON object:
// declared trace (timeline_csv of simulate), measured trace (timeline_csv of execute),
// GPU version trace and per-minibatch losses; tests/test_cpp_execute_gpu.py checks it
// against the reference fixture and the CPU oracle.
#include <cstdio>
#include <string>
#include <vector>

#include "ppsim/builder.hpp"
#include "ppsim/engine.hpp"
#include "ppsim/execute.hpp"
#include "ppsim/serialize.hpp"

int main() {
  ppsim::PolicyConfig cfg;
  cfg.policy = ppsim::Policy::AMDP;
  cfg.injection_limit = 2;
  cfg.num_pipelines = 2;
  cfg.accumulation_threshold = 8;
  cfg.num_minibatches = 32;
  cfg.zero_enabled = true;
  const auto declared = ppsim::ClusterSpec::uniform(4, 4, ppsim::Rat(1), ppsim::Rat(1));
  const auto reference_order = ppsim::simulate(ppsim::build(cfg, declared), declared);

  static const int parts[4] = {1, 1, 1, 1};
  ppsim::ExecuteOptions opt;
  opt.model = amdp_model_config{4, 128, 4, 512, 1024, 64, 4, 1, 0.02f, 1e-5f, 1234, parts, 0, 0, 0};
  opt.optimizer = amdp_opt_args{AMDP_OPT_ADAMW, 1e-3f, 0.9f, 0.95f, 1e-8f, 0.f, 1e-8f, 1e6f, 1.f, 1};
  const int T = 4 * 64;
  std::vector<int32_t> inputs(static_cast<size_t>(cfg.num_minibatches) * T), labels(inputs.size());
  if (amdp_synthetic_tokens(&opt.model, opt.data_seed, 0, cfg.num_minibatches, inputs.data(), labels.data()) != 0)
    return 2;
  const auto run = ppsim::execute(cfg, declared, opt, inputs.data(), labels.data());

  ppsim::ordered_json j;
  j["declared_csv"] = ppsim::timeline_csv(reference_order);
  j["measured_csv"] = ppsim::timeline_csv(run.timeline);
  j["version_trace"] = run.version_trace;
  j["losses"] = run.losses;
  j["bubble_w1"] = ppsim::bubble_ratio(run.timeline, 1).to_double();
  j["max_mismatch"] = ppsim::mismatch_report(run.timeline).max_overall();
  j["causality_issues"] = ppsim::validate_causality(run.timeline, declared).size();
  j["overlap_issues"] = ppsim::validate_non_overlap(run.timeline).size();
  std::puts(j.dump().c_str());
  return 0;
}
