// C-ABI of the schedule library (include/amdp_sched.h).  Exceptions never cross it:
// they become error codes plus the exception text.
#include <cstring>
#include <stdexcept>

#include "amdp_sched.h"
#include "ppsim/ppsim.hpp"
#include "sched_handle.hpp"

using namespace ppsim;

namespace {

void put_err(char* err, std::size_t len, const std::string& msg) {
  if (!err || len == 0) return;
  const std::size_t n = std::min(len - 1, msg.size());
  std::memcpy(err, msg.data(), n);
  err[n] = '\0';
}

template <class F>
int guarded(char* err, std::size_t len, F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    put_err(err, len, e.what());
    return AMDP_SCHED_EINVAL;
  } catch (const std::out_of_range& e) {
    put_err(err, len, e.what());
    return AMDP_SCHED_EINVAL;
  } catch (const std::overflow_error& e) {
    put_err(err, len, e.what());
    return AMDP_SCHED_EARITH;
  } catch (const std::domain_error& e) {
    put_err(err, len, e.what());
    return AMDP_SCHED_EARITH;
  } catch (const std::exception& e) {
    put_err(err, len, e.what());
    return AMDP_SCHED_ERUNTIME;
  }
}

std::size_t put_text(const std::string& s, char* buf, std::size_t len) {
  if (buf && len > 0) {
    const std::size_t n = std::min(len - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return s.size();
}

amdp_rat to_c(const Rat& r) { return amdp_rat{r.num(), r.den()}; }

std::string jrat(const Rat& r) {
  return r.den() == 1 ? std::to_string(r.num()) : "\"" + r.str() + "\"";
}

}  // namespace

namespace amdp {

Rat from_c(const amdp_rat& r) { return Rat(r.num, r.den == 0 ? 1 : r.den); }

ClusterSpec cluster_from_c(const amdp_cluster_spec* c) {
  ClusterSpec cl;
  if (!c) return cl;
  cl.depth = c->depth;
  cl.devices = c->devices;
  for (int i = 0; i < c->n_fwd; ++i) cl.fwd_cost.push_back(from_c(c->fwd_cost[i]));
  for (int i = 0; i < c->n_bwd; ++i) cl.bwd_cost.push_back(from_c(c->bwd_cost[i]));
  cl.update_cost = from_c(c->update_cost);
  cl.comm_cost = from_c(c->comm_cost);
  int off = 0;
  for (int g = 0; g < c->num_nodes; ++g) {
    std::vector<int> grp(c->node_devices + off, c->node_devices + off + c->node_sizes[g]);
    off += c->node_sizes[g];
    cl.nodes.push_back(std::move(grp));
  }
  if (c->has_inter_node_cost) cl.inter_node_cost = from_c(c->inter_node_cost);
  return cl;
}

PolicyConfig policy_from_c(const amdp_policy_config* p) {
  PolicyConfig cfg;
  cfg.policy = static_cast<Policy>(p->policy);
  cfg.injection_limit = p->injection_limit;
  cfg.num_pipelines = p->num_pipelines;
  cfg.accumulation_threshold = p->accumulation_threshold;
  cfg.num_minibatches = p->num_minibatches;
  cfg.zero_enabled = p->zero_enabled != 0;
  cfg.injection_override = p->injection_override != 0;
  return cfg;
}

std::string report_json(const Timeline& tl, const ClusterSpec& cl, const PolicyConfig& cfg,
                        int warmup) {
  std::string s = "{\"policy\":\"" + std::string(policy_name(tl.policy)) + "\",\"depth\":" +
                  std::to_string(tl.depth) + ",\"devices\":" + std::to_string(tl.devices) +
                  ",\"threshold\":" + std::to_string(tl.threshold) + ",\"makespan\":" + jrat(tl.makespan);
  try {
    s += ",\"bubble_ratio\":\"" + bubble_ratio(tl, warmup).str() + "\"";
  } catch (const std::exception& e) {
    s += ",\"bubble_ratio\":null,\"bubble_error\":\"" + std::string(e.what()) + "\"";
  }
  s += ",\"bubble_warmup_windows\":" + std::to_string(warmup);
  const auto mm = mismatch_report(tl);
  s += ",\"mismatch\":{\"entries\":[";
  bool first = true;
  for (const auto& [k, v] : mm.entries) {
    s += (first ? "[" : ",[") + std::to_string(k.first) + "," + std::to_string(k.second) + "," + std::to_string(v) + "]";
    first = false;
  }
  s += "],\"max_per_stage\":[";
  first = true;
  for (const auto& [k, v] : mm.max_per_stage) {
    s += (first ? "[" : ",[") + std::to_string(k) + "," + std::to_string(v) + "]";
    first = false;
  }
  s += "],\"max_overall\":" + std::to_string(mm.max_overall()) + ",\"missing\":[";
  first = true;
  for (const auto& k : mm.missing) {
    s += (first ? "[" : ",[") + std::to_string(k.first) + "," + std::to_string(k.second) + "]";
    first = false;
  }
  s += "]},\"windows\":[";
  first = true;
  for (const auto& w : window_mismatch(tl, tl.depth).windows) {
    s += first ? "{" : ",{";
    first = false;
    s += "\"window\":" + std::to_string(w.window) + ",\"window_size\":" + std::to_string(w.window_size) +
         ",\"update_count\":" + std::to_string(w.update_count) + ",\"mismatched\":[";
    for (std::size_t i = 0; i < w.mismatched.size(); ++i)
      s += (i ? "," : "") + std::to_string(w.mismatched[i]);
    s += "]}";
  }
  s += "],\"memory\":{\"per_device\":[";
  const auto mem = memory_report(tl, cfg, MemoryModel{});
  for (std::size_t d = 0; d < mem.per_device.size(); ++d) {
    const auto& m = mem.per_device[d];
    s += std::string(d ? ",{" : "{") + "\"weight\":" + jrat(m.weight) + ",\"activation_peak\":" +
         jrat(m.activation_peak) + ",\"gradient\":" + jrat(m.gradient) + ",\"optimizer_state\":" +
         jrat(m.optimizer_state) + "}";
  }
  s += "],\"closed_form\":{\"bubble\":" + (mem.table1.bubble ? jrat(*mem.table1.bubble) : std::string("null")) +
       ",\"weight_min\":" + jrat(mem.table1.weight_min) + ",\"weight_max\":" + jrat(mem.table1.weight_max) +
       ",\"activation_peak\":" + jrat(mem.table1.activation_peak) + "}}";
  auto list = [&](const std::vector<std::string>& v) {
    std::string o = "[";
    for (std::size_t i = 0; i < v.size(); ++i) {
      o += i ? ",\"" : "\"";
      for (char c : v[i]) o += (c == '"' || c == '\\') ? std::string("\\") + c : std::string(1, c);
      o += "\"";
    }
    return o + "]";
  };
  s += ",\"causality_issues\":" + list(validate_causality(tl, cl));
  s += ",\"overlap_issues\":" + list(validate_non_overlap(tl)) + "}";
  return s;
}

}  // namespace amdp

using amdp::SchedHandle;

extern "C" {

int amdp_validate(const amdp_policy_config* cfg, const amdp_cluster_spec* cl, char* buf, size_t len) {
  const auto c = amdp::cluster_from_c(cl);
  auto v = validate_cluster(c);
  auto vp = validate_policy(amdp::policy_from_c(cfg), c);
  v.insert(v.end(), vp.begin(), vp.end());
  std::string all;
  for (std::size_t i = 0; i < v.size(); ++i) all += (i ? "\n" : "") + v[i];
  put_text(all, buf, len);
  return static_cast<int>(v.size());
}

static int join_msgs(const std::vector<std::string>& v, char* buf, size_t len) {
  std::string all;
  for (std::size_t i = 0; i < v.size(); ++i) all += (i ? "\n" : "") + v[i];
  put_text(all, buf, len);
  return static_cast<int>(v.size());
}
int amdp_validate_cluster(const amdp_cluster_spec* cl, char* buf, size_t len) {
  return join_msgs(validate_cluster(amdp::cluster_from_c(cl)), buf, len);
}
int amdp_validate_policy(const amdp_policy_config* cfg, const amdp_cluster_spec* cl, char* buf, size_t len) {
  return join_msgs(validate_policy(amdp::policy_from_c(cfg), amdp::cluster_from_c(cl)), buf, len);
}

int amdp_map_stage_to_device(int pipeline, int stage, int depth, int* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] { *out = map_stage_to_device(pipeline, stage, depth); });
}
int amdp_default_num_pipelines(int depth, int* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] { *out = default_num_pipelines(depth); });
}
int amdp_preload_count(amdp_rat bwd, amdp_rat fwd, int* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] { *out = preload_count(amdp::from_c(bwd), amdp::from_c(fwd)); });
}

amdp_schedule* amdp_schedule_build(const amdp_policy_config* cfg, const amdp_cluster_spec* cl,
                                   char* err, size_t errlen) {
  auto* h = new SchedHandle;
  const int rc = guarded(err, errlen, [&] {
    h->cl = amdp::cluster_from_c(cl);
    h->cfg = amdp::policy_from_c(cfg);
    h->g = build(h->cfg, h->cl);
    h->has_graph = true;
  });
  if (rc != 0) {
    delete h;
    return nullptr;
  }
  return reinterpret_cast<amdp_schedule*>(h);
}

amdp_schedule* amdp_graph_new(int policy, int depth, int devices, int threshold, const amdp_cluster_spec* cl) {
  auto* h = new SchedHandle;
  h->g.policy = static_cast<Policy>(policy);
  h->g.depth = depth;
  h->g.devices = devices;
  h->g.threshold = threshold;
  h->cl = amdp::cluster_from_c(cl);
  h->cfg.policy = static_cast<Policy>(policy);
  h->has_graph = true;
  return reinterpret_cast<amdp_schedule*>(h);
}

int amdp_graph_add_task(amdp_schedule* s, const amdp_task_info* t) {
  auto* h = reinterpret_cast<SchedHandle*>(s);
  h->g.tasks.push_back(Task{static_cast<Kind>(t->kind), t->stage, t->minibatch, t->pipeline, t->device,
                            amdp::from_c(t->duration), t->window, t->preloaded != 0});
  return static_cast<int>(h->g.tasks.size()) - 1;
}
int amdp_graph_add_dep(amdp_schedule* s, int pred, int succ) {
  reinterpret_cast<SchedHandle*>(s)->g.deps.emplace_back(pred, succ);
  return 0;
}
int amdp_graph_add_lane(amdp_schedule* s, const int* ids, int n) {
  reinterpret_cast<SchedHandle*>(s)->g.lanes.emplace_back(ids, ids + n);
  return 0;
}

amdp_schedule* amdp_timeline_new(int policy, int depth, int devices, int threshold,
                                 const amdp_event* ev, int n, const amdp_cluster_spec* cl) {
  auto* h = new SchedHandle;
  h->tl.policy = static_cast<Policy>(policy);
  h->tl.depth = depth;
  h->tl.devices = devices;
  h->tl.threshold = threshold;
  h->tl.per_device.assign(static_cast<std::size_t>(devices), {});
  h->cl = amdp::cluster_from_c(cl);
  h->cfg.policy = static_cast<Policy>(policy);
  for (int i = 0; i < n; ++i) {
    TaskEvent e;
    e.kind = static_cast<Kind>(ev[i].kind);
    e.stage = ev[i].stage;
    e.minibatch = ev[i].minibatch;
    e.pipeline = ev[i].pipeline;
    e.device = ev[i].device;
    e.window = ev[i].window;
    e.preloaded = ev[i].preloaded != 0;
    e.start = amdp::from_c(ev[i].start);
    e.duration = amdp::from_c(ev[i].duration);
    if (e.device >= 0 && e.device < devices) {
      h->tl.makespan = max(h->tl.makespan, e.finish());
      h->tl.per_device[static_cast<std::size_t>(e.device)].push_back(e);
    }
  }
  h->has_timeline = true;
  return reinterpret_cast<amdp_schedule*>(h);
}

amdp_schedule* amdp_schedule_clone(const amdp_schedule* s) {
  return reinterpret_cast<amdp_schedule*>(new SchedHandle(*reinterpret_cast<const SchedHandle*>(s)));
}

void amdp_schedule_free(amdp_schedule* s) { delete reinterpret_cast<SchedHandle*>(s); }

int amdp_schedule_simulate(amdp_schedule* s, char* err, size_t errlen) {
  auto* h = reinterpret_cast<SchedHandle*>(s);
  if (!h->has_graph) return AMDP_SCHED_ESTATE;
  return guarded(err, errlen, [&] {
    h->tl = simulate_with_order(h->g, h->cl, &h->order);
    h->has_timeline = true;
  });
}

int amdp_schedule_num_tasks(const amdp_schedule* s) {
  return static_cast<int>(reinterpret_cast<const SchedHandle*>(s)->g.tasks.size());
}
int amdp_schedule_tasks(const amdp_schedule* s, amdp_task_info* out, int cap) {
  const auto& g = reinterpret_cast<const SchedHandle*>(s)->g;
  const int n = std::min(cap, static_cast<int>(g.tasks.size()));
  for (int i = 0; i < n; ++i) {
    const Task& t = g.tasks[static_cast<std::size_t>(i)];
    out[i] = amdp_task_info{static_cast<int>(t.kind), t.stage, t.minibatch, t.pipeline, t.device,
                            t.window, t.preloaded ? 1 : 0, to_c(t.duration)};
  }
  return n;
}
int amdp_schedule_num_deps(const amdp_schedule* s) {
  return static_cast<int>(reinterpret_cast<const SchedHandle*>(s)->g.deps.size());
}
int amdp_schedule_deps(const amdp_schedule* s, int* out, int cap) {
  const auto& d = reinterpret_cast<const SchedHandle*>(s)->g.deps;
  const int n = std::min(cap, static_cast<int>(d.size()));
  for (int i = 0; i < n; ++i) {
    out[2 * i] = d[static_cast<std::size_t>(i)].first;
    out[2 * i + 1] = d[static_cast<std::size_t>(i)].second;
  }
  return n;
}
int amdp_schedule_order(const amdp_schedule* s, int* out, int cap) {
  const auto& o = reinterpret_cast<const SchedHandle*>(s)->order;
  const int n = std::min(cap, static_cast<int>(o.size()));
  std::copy(o.begin(), o.begin() + n, out);
  return n;
}
int amdp_schedule_num_events(const amdp_schedule* s) {
  int n = 0;
  for (const auto& d : reinterpret_cast<const SchedHandle*>(s)->tl.per_device) n += static_cast<int>(d.size());
  return n;
}
int amdp_schedule_events(const amdp_schedule* s, amdp_event* out, int cap) {
  int n = 0;
  for (const auto& dev : reinterpret_cast<const SchedHandle*>(s)->tl.per_device)
    for (const auto& e : dev) {
      if (n >= cap) return n;
      out[n++] = amdp_event{static_cast<int>(e.kind), e.stage, e.minibatch, e.pipeline, e.device,
                            e.window, e.preloaded ? 1 : 0, to_c(e.start), to_c(e.duration)};
    }
  return n;
}
int amdp_schedule_makespan(const amdp_schedule* s, amdp_rat* out) {
  const auto* h = reinterpret_cast<const SchedHandle*>(s);
  if (!h->has_timeline) return AMDP_SCHED_ESTATE;
  *out = to_c(h->tl.makespan);
  return 0;
}
int amdp_schedule_bubble(const amdp_schedule* s, int warmup, amdp_rat* out, char* err, size_t errlen) {
  const auto* h = reinterpret_cast<const SchedHandle*>(s);
  if (!h->has_timeline) return AMDP_SCHED_ESTATE;
  return guarded(err, errlen, [&] { *out = to_c(bubble_ratio(h->tl, warmup)); });
}

size_t amdp_schedule_text(const amdp_schedule* s, int which, char* buf, size_t len) {
  const auto* h = reinterpret_cast<const SchedHandle*>(s);
  switch (which) {
    case AMDP_TEXT_TIMELINE_CSV: return put_text(timeline_csv(h->tl), buf, len);
    case AMDP_TEXT_VERSION_CSV: return put_text(version_trace_csv(h->tl), buf, len);
    case AMDP_TEXT_TIMELINE_JSON: return put_text(timeline_json_text(h->tl), buf, len);
  }
  return put_text("", buf, len);
}

size_t amdp_schedule_report_json(const amdp_schedule* s, const amdp_policy_config* cfg, int warmup,
                                 char* buf, size_t len) {
  const auto* h = reinterpret_cast<const SchedHandle*>(s);
  const PolicyConfig pc = cfg ? amdp::policy_from_c(cfg) : h->cfg;
  return put_text(amdp::report_json(h->tl, h->cl, pc, warmup), buf, len);
}

}  // extern "C"
