// C-ABI of the stage executor (include/amdp_engine.h) and the C++ drop-in ppsim::execute
// (include/ppsim/execute.hpp), both over amdp::Engine (executor.hpp).
#include "executor.hpp"

// ====================================================================== C-ABI
namespace {
void put_err(char* err, size_t len, const std::string& m) {
  if (!err || !len) return;
  const size_t n = std::min(len - 1, m.size());
  std::memcpy(err, m.data(), n);
  err[n] = 0;
}
size_t put_text(const std::string& s, char* buf, size_t len) {
  if (buf && len) {
    const size_t n = std::min(len - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return s.size();
}
}  // namespace

using amdp::Engine;

extern "C" {


amdp_engine* amdp_engine_create(const amdp_model_config* model, const amdp_run_config* run,
                                const uint8_t* nccl_id, char* err, size_t errlen) {
  try {
    return reinterpret_cast<amdp_engine*>(new Engine(*model, *run, nccl_id));
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return nullptr;
  }
}

void amdp_engine_destroy(amdp_engine* e) { delete reinterpret_cast<Engine*>(e); }

size_t amdp_engine_comm_export(amdp_engine* e, uint8_t* buf, size_t len) {
  try {
    const std::string b = reinterpret_cast<Engine*>(e)->comm_export();
    if (buf) std::memcpy(buf, b.data(), std::min(len, b.size()));
    return b.size();
  } catch (...) {
    return 0;
  }
}

int amdp_engine_comm_connect(amdp_engine* e, const uint8_t* const* blobs, const size_t* lens, int count, char* err,
                             size_t errlen) {
  try {
    std::vector<std::string> all;
    for (int r = 0; r < count; ++r)
      all.emplace_back(reinterpret_cast<const char*>(blobs[r]), lens[r]);
    reinterpret_cast<Engine*>(e)->comm_connect(all);
    return 0;
  } catch (const std::exception& ex) {
    put_err(err, errlen, ex.what());
    return AMDP_ERR_CUDA;
  }
}

void* amdp_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) return nullptr;
  return p;
}
void amdp_host_free(void* p) { cudaFreeHost(p); }

int amdp_synthetic_tokens(const amdp_model_config* m, uint64_t seed, int first, int count, int32_t* inputs,
                          int32_t* labels) {
  const int S = m->seq, B = m->seqs_per_minibatch, V = m->vocab;
  if (S <= 0 || B <= 0 || V <= 0 || count < 0) return AMDP_ERR_INVALID;
  const size_t T = static_cast<size_t>(S) * B;
  const uint64_t UV = static_cast<uint64_t>(V);
  for (int j = 0; j < count; ++j) {
    const uint64_t mb = static_cast<uint64_t>(first + j);
    for (int b = 0; b < B; ++b) {
      const uint64_t r = amdp::splitmix64(seed * 0x100000001B3ull + mb * 1024ull + static_cast<uint64_t>(b));
      const uint64_t start = r % UV;
      const uint64_t stride = 1 + (r >> 32) % 7;
      const size_t base = static_cast<size_t>(j) * T + static_cast<size_t>(b) * S;
      for (int p = 0; p <= S; ++p) {
        const uint64_t nz = amdp::splitmix64(r + static_cast<uint64_t>(p) + 1);
        const int32_t tok = static_cast<int32_t>((nz & 7) == 0 ? (nz >> 8) % UV
                                                               : (start + static_cast<uint64_t>(p) * stride) % UV);
        if (m->causal) {  // GPT: next-token prediction
          if (p < S) inputs[base + static_cast<size_t>(p)] = tok;
          if (p > 0) labels[base + static_cast<size_t>(p) - 1] = tok;
        } else if (p < S) {  // BERT MLM: 15% of positions, 80/10/10 mask/random/keep
          const uint64_t hm = amdp::splitmix64((r ^ 0xA5A5A5A5A5A5A5A5ull) + static_cast<uint64_t>(p));
          int32_t in = tok, lab = -1;
          if (hm % 100 < 15) {
            lab = tok;
            const uint64_t act = (hm >> 8) % 10;
            if (act < 8) in = static_cast<int32_t>(UV - 1);  // [MASK] = last vocabulary id
            else if (act == 8) in = static_cast<int32_t>((hm >> 16) % UV);
          }
          if (m->pad_token > 0) {  // padded to a length in [S/2, S]; no real token is the pad id
            const int len = S / 2 + static_cast<int>((r >> 40) % static_cast<uint64_t>(S - S / 2 + 1));
            if (in == m->pad_token) in = static_cast<int32_t>((m->pad_token + 1) % V);
            if (p >= len) {
              in = m->pad_token;
              lab = -1;
            }
          }
          inputs[base + static_cast<size_t>(p)] = in;
          labels[base + static_cast<size_t>(p)] = lab;
        }
      }
    }
  }
  return 0;
}

int amdp_engine_run(amdp_engine* e, const int32_t* inputs, const int32_t* labels, float* losses_out, char* err,
                    size_t errlen) {
  try {
    reinterpret_cast<Engine*>(e)->run(inputs, labels, losses_out);
    return 0;
  } catch (const std::exception& ex) {
    put_err(err, errlen, ex.what());
    return AMDP_ERR_CUDA;
  }
}

int amdp_engine_run_windows(amdp_engine* e, int num_windows, const int32_t* inputs, const int32_t* labels,
                            float* losses_out, int resident, char* err, size_t errlen) {
  try {
    reinterpret_cast<Engine*>(e)->run(inputs, labels, losses_out, num_windows, resident != 0);
    return 0;
  } catch (const std::exception& ex) {
    put_err(err, errlen, ex.what());
    return AMDP_ERR_CUDA;
  }
}

int amdp_engine_stage_tokens(amdp_engine* e, const int32_t* inputs, const int32_t* labels) {
  try {
    reinterpret_cast<Engine*>(e)->stage_tokens(inputs, labels);
    return 0;
  } catch (...) {
    return AMDP_ERR_CUDA;
  }
}

int amdp_engine_set_kernel_timing(amdp_engine* e, int enable) {
  reinterpret_cast<Engine*>(e)->set_kernel_timing(enable != 0);
  return 0;
}

int amdp_engine_set_streams(amdp_engine* e, int n) {
  try {
    return reinterpret_cast<Engine*>(e)->set_streams(n);
  } catch (...) {
    return AMDP_ERR_CUDA;
  }
}

int amdp_engine_set_graphs(amdp_engine* e, int enable) {
  reinterpret_cast<Engine*>(e)->graphs_enabled_ = enable != 0;
  return 0;
}

int amdp_engine_kernel_stats(const amdp_engine* e, amdp_kernel_class_stats* out, int cap) {
  const auto& kt = reinterpret_cast<const Engine*>(e)->ktimer_;
  const int n = std::min(cap, static_cast<int>(amdp::K_NUM));
  for (int c = 0; c < n; ++c) {
    std::memset(out[c].name, 0, sizeof(out[c].name));
    std::strncpy(out[c].name, amdp::kclass_name(c), sizeof(out[c].name) - 1);
    out[c].launches = kt.launches[static_cast<size_t>(c)];
    out[c].total_ms = kt.ms[static_cast<size_t>(c)];
    out[c].flops = kt.flops[static_cast<size_t>(c)];
    out[c].bytes = kt.bytes[static_cast<size_t>(c)];
  }
  return n;
}

int amdp_engine_stats(const amdp_engine* e, amdp_run_stats* out) {
  *out = reinterpret_cast<const Engine*>(e)->stats;
  return 0;
}

int amdp_engine_num_events(const amdp_engine* e) {
  return static_cast<int>(reinterpret_cast<const Engine*>(e)->events.size());
}

int amdp_engine_num_lane_events(const amdp_engine* e) {
  return static_cast<int>(reinterpret_cast<const Engine*>(e)->lane_events.size());
}

int amdp_engine_lane_events(const amdp_engine* e, amdp_event* out, int cap) {
  const auto& ev = reinterpret_cast<const Engine*>(e)->lane_events;
  const int n = std::min(cap, static_cast<int>(ev.size()));
  for (int i = 0; i < n; ++i) {
    const auto& x = ev[static_cast<size_t>(i)];
    out[i] = amdp_event{static_cast<int>(x.kind), x.stage, x.minibatch, x.pipeline, x.device, x.window,
                        x.preloaded ? 1 : 0, amdp_rat{x.start.num(), x.start.den()},
                        amdp_rat{x.duration.num(), x.duration.den()}};
  }
  return n;
}

int amdp_engine_events(const amdp_engine* e, amdp_event* out, int cap) {
  const auto& ev = reinterpret_cast<const Engine*>(e)->events;
  const int n = std::min(cap, static_cast<int>(ev.size()));
  for (int i = 0; i < n; ++i) {
    const auto& x = ev[static_cast<size_t>(i)];
    out[i] = amdp_event{static_cast<int>(x.kind), x.stage, x.minibatch, x.pipeline, x.device, x.window,
                        x.preloaded ? 1 : 0, amdp_rat{x.start.num(), x.start.den()},
                        amdp_rat{x.duration.num(), x.duration.den()}};
  }
  return n;
}

size_t amdp_engine_version_trace(const amdp_engine* e, char* buf, size_t len) {
  return put_text(reinterpret_cast<const Engine*>(e)->version_csv(), buf, len);
}

amdp_schedule* amdp_engine_schedule(const amdp_engine* e) {
  return reinterpret_cast<amdp_schedule*>(new amdp::SchedHandle(reinterpret_cast<const Engine*>(e)->sched));
}

int64_t amdp_engine_stage_numel(const amdp_engine* e, int stage) {
  try {
    return reinterpret_cast<const Engine*>(e)->stage_numel(stage);
  } catch (...) {
    return -1;
  }
}

int amdp_engine_get_stage_params(const amdp_engine* e, int stage, float* out, int64_t n) {
  try {
    const_cast<Engine*>(reinterpret_cast<const Engine*>(e))->copy_params(stage, out, n, true);
    return 0;
  } catch (...) {
    return AMDP_ERR_INVALID;
  }
}

int amdp_engine_set_stage_params(amdp_engine* e, int stage, const float* in, int64_t n) {
  try {
    reinterpret_cast<Engine*>(e)->copy_params(stage, const_cast<float*>(in), n, false);
    return 0;
  } catch (...) {
    return AMDP_ERR_INVALID;
  }
}

size_t amdp_engine_plan_json(const amdp_engine* e, char* buf, size_t len) {
  return put_text(reinterpret_cast<const Engine*>(e)->plan_json(), buf, len);
}

}  // extern "C"

// ====================================================================== C++ API
#include "ppsim/execute.hpp"

namespace ppsim {

ExecuteResult execute(const PolicyConfig& cfg, const ClusterSpec& declared, const ExecuteOptions& opt,
                      const int32_t* inputs, const int32_t* labels) {
  if (declared.fwd_cost.empty() || declared.bwd_cost.empty())
    throw std::invalid_argument("execute: declared cluster needs per-stage costs");
  for (std::size_t i = 1; i < declared.fwd_cost.size(); ++i)
    if (declared.fwd_cost[i] != declared.fwd_cost[0] || declared.bwd_cost[i] != declared.bwd_cost[0])
      throw std::invalid_argument("execute: the executor replays uniform declared costs");
  if (declared.comm_cost != Rat(0) || declared.update_cost != Rat(0))
    throw std::invalid_argument("execute: declared comm/update costs must be 0 (they change the order)");
  amdp_run_config rc{};
  rc.policy = amdp_policy_config{static_cast<int>(cfg.policy), cfg.injection_limit, cfg.num_pipelines,
                                 cfg.accumulation_threshold, cfg.num_minibatches, cfg.zero_enabled ? 1 : 0,
                                 cfg.injection_override ? 1 : 0};
  rc.declared_fwd = amdp_rat{declared.fwd_cost[0].num(), declared.fwd_cost[0].den()};
  rc.declared_bwd = amdp_rat{declared.bwd_cost[0].num(), declared.bwd_cost[0].den()};
  rc.optimizer = opt.optimizer;
  rc.world_size = opt.world_size;
  rc.rank = opt.rank;
  rc.record_events = 1;
  rc.data_seed = opt.data_seed;
  rc.depth = declared.depth;
  rc.comm_backend = opt.comm_backend;
  amdp::Engine eng(opt.model, rc, opt.nccl_id);
  if (opt.world_size > 1 && opt.comm_backend == AMDP_COMM_IPC) {
    if (!opt.allgather) throw std::invalid_argument("execute: world_size > 1 needs ExecuteOptions::allgather");
    eng.comm_connect(opt.allgather(eng.comm_export()));
  }
  ExecuteResult out;
  out.losses.assign(static_cast<std::size_t>(cfg.num_minibatches), 0.f);
  eng.run(inputs, labels, out.losses.data());
  out.stats = eng.stats;
  out.version_trace = eng.version_csv();
  out.timeline.policy = cfg.policy;
  out.timeline.depth = declared.depth;
  out.timeline.devices = declared.devices;
  out.timeline.threshold = cfg.accumulation_threshold;
  out.timeline.per_device.assign(static_cast<std::size_t>(declared.devices), {});
  for (const auto& e : eng.events) {
    out.timeline.makespan = max(out.timeline.makespan, e.finish());
    out.timeline.per_device[static_cast<std::size_t>(e.device)].push_back(e);
  }
  return out;
}

}  // namespace ppsim
