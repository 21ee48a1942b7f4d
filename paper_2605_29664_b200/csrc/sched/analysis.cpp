// Trace audits and reports over a Timeline (simulated or measured on the GPU):
// causality/overlap audits (validate.hpp:118-177), parameter-version oracle
// (analysis.hpp:28-88, 126-155), memory/comm accounting (analysis.hpp:226-346),
// and the trace emitters (serialize.hpp:41-94).
#include <algorithm>
#include <map>
#include <numeric>
#include <random>
#include <set>
#include <sstream>
#include <stdexcept>

#include "ppsim/ppsim.hpp"

namespace ppsim {

namespace {
std::string ev_name(const char* k, int s, int j) {
  return std::string(k) + "(" + std::to_string(s) + "," + std::to_string(j) + ")";
}

// Parameter changes of one stage: Broadcast finishes rewrite every replica (sharded
// state); Update finishes rewrite their own pipeline's replica.
struct Change {
  Rat when;
  int pipeline;
  bool all_replicas;
};
std::vector<std::vector<Change>> changes_by_stage(const Timeline& t) {
  std::vector<std::vector<Change>> ch;
  for (const auto& dev : t.per_device)
    for (const auto& e : dev) {
      if (e.kind != Kind::Update && e.kind != Kind::Broadcast) continue;
      if (static_cast<int>(ch.size()) <= e.stage) ch.resize(static_cast<std::size_t>(e.stage) + 1);
      ch[static_cast<std::size_t>(e.stage)].push_back(
          {e.finish(), e.kind == Kind::Update ? e.pipeline : 0, e.kind == Kind::Broadcast});
    }
  return ch;
}
}  // namespace

std::vector<std::string> validate_causality(const Timeline& t, const ClusterSpec& c) {
  std::vector<std::string> out;
  std::map<std::pair<int, int>, const TaskEvent*> F, B;
  for (const auto& dev : t.per_device)
    for (const auto& e : dev) {
      if (e.kind != Kind::Forward && e.kind != Kind::Backward) continue;
      auto& m = e.kind == Kind::Forward ? F : B;
      if (!m.emplace(std::make_pair(e.stage, e.minibatch), &e).second)
        out.push_back(std::string(e.kind == Kind::Forward ? "duplicate forward" : "duplicate backward") +
                      "(" + std::to_string(e.stage) + "," + std::to_string(e.minibatch) + ")");
    }
  auto need_before = [&](const TaskEvent* a, const TaskEvent* b, const char* ka, const char* kb) {
    const Rat bound = a->finish() + c.gap(a->device, b->device);
    if (b->start < bound)
      out.push_back(ev_name(kb, b->stage, b->minibatch) + " starts at " + b->start.str() +
                    " before " + ev_name(ka, a->stage, a->minibatch) + " ends at " +
                    a->finish().str() + (a->device != b->device ? " plus transfer gap" : ""));
  };
  for (const auto& [k, f] : F) {
    if (auto it = B.find(k); it != B.end()) need_before(f, it->second, "forward", "backward");
    if (auto it = F.find({k.first + 1, k.second}); it != F.end())
      need_before(f, it->second, "forward", "forward");
  }
  for (const auto& [k, b] : B)
    if (k.first > 0)
      if (auto it = B.find({k.first - 1, k.second}); it != B.end())
        need_before(b, it->second, "backward", "backward");
  return out;
}

std::vector<std::string> validate_non_overlap(const Timeline& t) {
  std::vector<std::string> out;
  for (std::size_t d = 0; d < t.per_device.size(); ++d) {
    const auto& ev = t.per_device[d];
    for (std::size_t i = 1; i < ev.size(); ++i)
      if (ev[i].start < ev[i - 1].finish())
        out.push_back("device " + std::to_string(d) + ": " + kind_name(ev[i].kind) + "(" +
                      std::to_string(ev[i].stage) + "," + std::to_string(ev[i].minibatch) +
                      ") overlaps previous event");
  }
  return out;
}

MismatchReport mismatch_report(const Timeline& t) {
  struct Pair {
    bool f = false, b = false;
    Rat f_finish, b_start;
    int pipeline = 0;
  };
  std::map<std::pair<int, int>, Pair> pairs;
  for (const auto& dev : t.per_device)
    for (const auto& e : dev) {
      if (e.kind == Kind::Forward) {
        auto& p = pairs[{e.stage, e.minibatch}];
        p.f = true;
        p.f_finish = e.finish();
        p.pipeline = e.pipeline;
      } else if (e.kind == Kind::Backward) {
        auto& p = pairs[{e.stage, e.minibatch}];
        p.b = true;
        p.b_start = e.start;
      }
    }
  const auto ch = changes_by_stage(t);
  MismatchReport rep;
  for (const auto& [key, p] : pairs) {
    if (!p.f || !p.b) {
      rep.missing.push_back(key);
      continue;
    }
    int n = 0;
    if (key.first < static_cast<int>(ch.size()))
      for (const Change& c : ch[static_cast<std::size_t>(key.first)])
        if ((c.all_replicas || c.pipeline == p.pipeline) && p.f_finish <= c.when && c.when <= p.b_start)
          ++n;
    rep.entries[key] = n;
    auto [it, fresh] = rep.max_per_stage.try_emplace(key.first, n);
    if (!fresh) it->second = std::max(it->second, n);
  }
  return rep;
}

WindowReport window_mismatch(const Timeline& t, int /*depth*/) {
  const auto rep = mismatch_report(t);
  std::map<int, int> win_of;
  std::map<int, WindowEntry> entries;
  for (const auto& dev : t.per_device)
    for (const auto& e : dev) {
      if (e.kind == Kind::Forward && e.stage == 0) {
        win_of[e.minibatch] = e.window;
        auto& w = entries[e.window];
        w.window = e.window;
        ++w.window_size;
      }
      if (e.kind == Kind::Update || e.kind == Kind::Broadcast) {
        auto& w = entries[e.window];
        w.window = e.window;
        ++w.update_count;
      }
    }
  std::map<int, std::set<int>> hit;
  for (const auto& [key, n] : rep.entries)
    if (n > 0) hit[win_of[key.second]].insert(key.second);
  WindowReport out;
  for (auto& [w, entry] : entries) {
    if (auto it = hit.find(w); it != hit.end()) entry.mismatched.assign(it->second.begin(), it->second.end());
    out.windows.push_back(std::move(entry));
  }
  return out;
}

MemoryReport memory_report(const Timeline& t, const PolicyConfig& policy, const MemoryModel& mem) {
  const int D = t.devices;
  MemoryReport out;
  out.per_device.resize(static_cast<std::size_t>(std::max(D, 0)));
  std::vector<std::set<std::pair<int, int>>> replicas(out.per_device.size());
  struct Live {
    bool f = false, b = false;
    Rat s, e;
    int device = 0;
  };
  std::map<std::pair<int, int>, Live> lives;
  for (int d = 0; d < D; ++d)
    for (const auto& e : t.per_device[static_cast<std::size_t>(d)]) {
      if (e.kind != Kind::Forward && e.kind != Kind::Backward) continue;
      replicas[static_cast<std::size_t>(d)].insert({e.stage, e.pipeline});
      auto& lv = lives[{e.stage, e.minibatch}];
      lv.device = d;
      if (e.kind == Kind::Forward) {
        lv.f = true;
        lv.s = e.start;
      } else {
        lv.b = true;
        lv.e = e.finish();
      }
    }
  std::vector<std::vector<std::pair<Rat, int>>> sweep(out.per_device.size());
  for (const auto& [k, lv] : lives)
    if (lv.f && lv.b) {
      sweep[static_cast<std::size_t>(lv.device)].push_back({lv.s, +1});
      sweep[static_cast<std::size_t>(lv.device)].push_back({lv.e, -1});
    }
  const bool sharded = policy.policy == Policy::AMDP && policy.zero_enabled;
  for (int d = 0; d < D; ++d) {
    auto& ev = sweep[static_cast<std::size_t>(d)];
    std::sort(ev.begin(), ev.end(), [](const auto& a, const auto& b) {
      if (a.first != b.first) return a.first < b.first;
      return a.second > b.second;  // allocations before frees at equal times
    });
    int cur = 0, peak = 0;
    for (const auto& [when, delta] : ev) peak = std::max(peak, cur += delta);
    const auto& reps = replicas[static_cast<std::size_t>(d)];
    Rat weight_units(0);
    if (policy.policy == Policy::PipeDreamAsync) {
      for (const auto& [stage, pipe] : reps) weight_units += Rat(std::min(policy.injection_limit, t.depth - stage));
    } else {
      weight_units = Rat(static_cast<std::int64_t>(reps.size()));
    }
    const Rat n_reps(static_cast<std::int64_t>(reps.size()));
    DeviceMemory& dm = out.per_device[static_cast<std::size_t>(d)];
    dm.weight = weight_units * mem.weight_per_stage;
    dm.activation_peak = Rat(peak) * mem.activation_per_stage_per_minibatch;
    dm.gradient = n_reps * mem.weight_per_stage * mem.gradient_multiplier;
    dm.optimizer_state = n_reps * mem.weight_per_stage * mem.optimizer_state_multiplier;
    if (sharded) dm.optimizer_state = dm.optimizer_state * Rat(2, t.depth);
  }
  const int d = t.depth, n = policy.accumulation_threshold;
  Table1View& v = out.table1;
  const Rat W = mem.weight_per_stage, A = mem.activation_per_stage_per_minibatch;
  switch (policy.policy) {
    case Policy::DAPPLE:
    case Policy::GPipe:
      v.bubble = Rat(d - 1, n + d - 1);
      v.weight_min = v.weight_max = W;
      v.activation_peak = Rat(n) * A;
      break;
    case Policy::Interleaved1F1B:
      v.bubble = Rat(d - 1, 2 * n + d - 1);
      v.weight_min = v.weight_max = W;
      v.activation_peak = Rat(d) * A;
      break;
    case Policy::Chimera:
      v.bubble = Rat(d - 2, 2 * n + d - 2);
      v.weight_min = v.weight_max = Rat(2) * W;
      v.activation_peak = Rat(d) * A;
      break;
    case Policy::PipeDreamAsync:
      v.bubble.reset();
      v.weight_min = W;
      v.weight_max = Rat(d) * W;
      v.activation_peak = Rat(d) * A;
      break;
    case Policy::AMDP:
      v.bubble.reset();
      v.weight_min = v.weight_max = W;
      v.activation_peak = Rat(d) * A;
      break;
  }
  return out;
}

CommVolume reduce_broadcast_cost(int replicas, const Rat& bytes) {
  if (replicas < 1) throw std::invalid_argument("replicas must be at least 1");
  if (replicas == 1) return {Rat(0), Rat(0), Rat(0)};
  const Rat phase = bytes * Rat(replicas - 1, replicas);
  return {phase, phase, phase * Rat(2)};
}

// ------------------------------------------------------------------ emitters
// Property check of analysis.hpp:96-121: a PipeDreamAsync pipeline (update after every
// backward) with at most n minibatches in flight shows min(n, depth - i) - 1 parameter changes
// between F(i, j) and B(i, j) for every steady minibatch j (ramp-up / drain: the first and last
// `depth` minibatches, excluded).
Verdict verify_steady_mismatch(int depth, int injection_limit) {
  if (injection_limit < 1 || injection_limit > depth) return {false, "injection limit must lie in [1, depth]"};
  const ClusterSpec cl = ClusterSpec::uniform(depth, depth, Rat(1), Rat(1));
  PolicyConfig cfg;
  cfg.policy = Policy::PipeDreamAsync;
  cfg.injection_limit = injection_limit;
  cfg.num_minibatches = 4 * depth;
  const MismatchReport rep = mismatch_report(simulate(build(cfg, cl), cl));
  for (int i = 0; i < depth; ++i) {
    const int expect = std::min(injection_limit, depth - i) - 1;
    for (int j = depth; j < 3 * depth; ++j) {
      const auto it = rep.entries.find({i, j});
      const std::string where = "stage " + std::to_string(i) + " minibatch " + std::to_string(j);
      if (it == rep.entries.end()) return {false, "no measurement for " + where};
      if (it->second != expect)
        return {false, where + ": measured " + std::to_string(it->second) + ", predicted " + std::to_string(expect)};
    }
  }
  return {true, "steady mismatch matches min(n, depth - stage) - 1 at every stage"};
}

// Property check of analysis.hpp:161-221: AMDP's one-step staleness bound comes from the
// dependency edges alone, so it must hold for any declared costs, cross-device / cross-node
// gaps, node partition, device relabeling and ring reflection.  Each trial draws all of them
// from `seed` (std::mt19937_64) and re-simulates.
Verdict verify_topology_invariance(int depth, int trials, std::uint64_t seed) {
  if (depth < 2 || depth % 2 != 0) return {false, "depth must be even and at least 2"};
  std::mt19937_64 rng(seed);
  auto pick = [&](int lo, int hi) { return lo + static_cast<int>(rng() % static_cast<std::uint64_t>(hi - lo + 1)); };
  auto shuffled = [&]() {
    std::vector<int> v(static_cast<std::size_t>(depth));
    std::iota(v.begin(), v.end(), 0);
    for (std::size_t k = v.size(); k > 1; --k) std::swap(v[k - 1], v[rng() % k]);
    return v;
  };
  for (int trial = 0; trial < trials; ++trial) {
    ClusterSpec cl = ClusterSpec::uniform(depth, depth, Rat(1), Rat(1));
    for (int i = 0; i < depth; ++i) {
      cl.fwd_cost[static_cast<std::size_t>(i)] = Rat(pick(1, 4));
      cl.bwd_cost[static_cast<std::size_t>(i)] = Rat(pick(1, 8));
    }
    cl.comm_cost = Rat(pick(1, 8), pick(1, 4));
    cl.update_cost = Rat(pick(0, 2), 2);
    const std::vector<int> order = shuffled();
    const int nodes = pick(1, 4);
    cl.nodes.assign(static_cast<std::size_t>(std::min(nodes, depth)), {});
    for (std::size_t k = 0; k < order.size(); ++k) cl.nodes[k % cl.nodes.size()].push_back(order[k]);
    cl.inter_node_cost = Rat(pick(1, 6), pick(1, 2));
    PolicyConfig cfg;
    cfg.policy = Policy::AMDP;
    cfg.injection_limit = 2;
    cfg.num_pipelines = depth / 2;
    cfg.accumulation_threshold = depth;
    cfg.num_minibatches = 3 * depth;
    cfg.zero_enabled = rng() % 2 == 0;
    TaskGraph g = build(cfg, cl);
    const std::vector<int> perm = shuffled();
    const bool reflect = rng() % 2 == 1;
    for (Task& task : g.tasks)
      task.device = perm[static_cast<std::size_t>(reflect ? depth - 1 - task.device : task.device)];
    const MismatchReport rep = mismatch_report(simulate(g, cl));
    if (rep.max_overall() > 1) {
      std::ostringstream os;
      os << "trial " << trial << " (seed " << seed << "): max mismatch " << rep.max_overall() << " with comm_cost "
         << cl.comm_cost.str() << ", reflect " << reflect << ", zero " << cfg.zero_enabled << ", perm";
      for (int v : perm) os << ' ' << v;
      return {false, os.str()};
    }
    if (!rep.missing.empty()) return {false, "trial " + std::to_string(trial) + ": incomplete forward/backward pairs"};
  }
  return {true, std::to_string(trials) + " perturbed runs kept max mismatch <= 1"};
}

std::string timeline_csv(const Timeline& t) {
  std::string s = "device,kind,stage,minibatch,pipeline,window,preloaded,start,duration\n";
  s.reserve(64 * 1024);
  for (std::size_t d = 0; d < t.per_device.size(); ++d)
    for (const auto& e : t.per_device[d]) {
      s += std::to_string(d);
      s += ',';
      s += kind_name(e.kind);
      s += ',' + std::to_string(e.stage) + ',' + std::to_string(e.minibatch) + ',' +
           std::to_string(e.pipeline) + ',' + std::to_string(e.window) + ',';
      s += e.preloaded ? '1' : '0';
      s += ',' + e.start.str() + ',' + e.duration.str() + '\n';
    }
  return s;
}

std::string version_trace_csv(const Timeline& t) {
  const auto ch = changes_by_stage(t);
  std::string s = "device,kind,stage,minibatch,pipeline,window,preloaded,version\n";
  for (std::size_t d = 0; d < t.per_device.size(); ++d)
    for (const auto& e : t.per_device[d]) {
      if (e.kind != Kind::Forward && e.kind != Kind::Backward) continue;
      int ver = 0;
      if (e.stage < static_cast<int>(ch.size()))
        for (const Change& c : ch[static_cast<std::size_t>(e.stage)])
          if ((c.all_replicas || c.pipeline == e.pipeline) && c.when <= e.start) ++ver;
      s += std::to_string(d) + ',' + kind_name(e.kind) + ',' + std::to_string(e.stage) + ',' +
           std::to_string(e.minibatch) + ',' + std::to_string(e.pipeline) + ',' +
           std::to_string(e.window) + ',' + (e.preloaded ? '1' : '0') + ',' + std::to_string(ver) + '\n';
    }
  return s;
}

namespace {
std::string rat_j(const Rat& r) { return r.den() == 1 ? std::to_string(r.num()) : "\"" + r.str() + "\""; }
}  // namespace

std::string timeline_json_text(const Timeline& t) {
  std::string s = "{\"policy\":\"" + std::string(policy_name(t.policy)) +
                  "\",\"depth\":" + std::to_string(t.depth) + ",\"devices\":" + std::to_string(t.devices) +
                  ",\"threshold\":" + std::to_string(t.threshold) + ",\"makespan\":" + rat_j(t.makespan) +
                  ",\"per_device\":[";
  for (std::size_t d = 0; d < t.per_device.size(); ++d) {
    s += d ? ",[" : "[";
    bool first = true;
    for (const auto& e : t.per_device[d]) {
      s += first ? "{" : ",{";
      first = false;
      s += "\"kind\":\"" + std::string(kind_name(e.kind)) + "\",\"stage\":" + std::to_string(e.stage) +
           ",\"minibatch\":" + std::to_string(e.minibatch) + ",\"pipeline\":" + std::to_string(e.pipeline) +
           ",\"window\":" + std::to_string(e.window) + ",\"preloaded\":" + (e.preloaded ? "true" : "false") +
           ",\"start\":" + rat_j(e.start) + ",\"duration\":" + rat_j(e.duration) + "}";
    }
    s += "]";
  }
  return s + "]}";
}

}  // namespace ppsim
