// Configuration rules and the schedule builder (the AMDP partition config -> task DAG).
//
// Restates the reference's contract: validate.hpp:12-113 (rules and messages, returned
// as data), builder.hpp:81-104 (placement / pipeline count / preload), builder.hpp:145-385
// (task set, causal + injection-pacing + window edges, per-replica lanes for the
// baseline policies).  The trace this produces must equal the reference's byte-for-byte
// (tests/test_sched_oracle.py against oracle/_ref).
#include <algorithm>
#include <climits>
#include <stdexcept>
#include <tuple>

#include "ppsim/ppsim.hpp"

namespace ppsim {

const char* kind_name(Kind k) {
  static const char* names[] = {"Forward", "Backward", "Reduce", "Broadcast", "Update"};
  const auto i = static_cast<unsigned>(k);
  return i < 5 ? names[i] : "?";
}

const char* policy_name(Policy p) {
  static const char* names[] = {"AMDP", "DAPPLE", "GPipe", "Interleaved1F1B", "Chimera",
                                "PipeDreamAsync"};
  const auto i = static_cast<unsigned>(p);
  return i < 6 ? names[i] : "?";
}

std::optional<Policy> policy_from_name(const std::string& s) {
  for (int i = 0; i < 6; ++i)
    if (s == policy_name(static_cast<Policy>(i))) return static_cast<Policy>(i);
  return std::nullopt;
}

// ------------------------------------------------------------------ ClusterSpec
ClusterSpec ClusterSpec::uniform(int depth, int devices, Rat fwd, Rat bwd, Rat update, Rat comm) {
  ClusterSpec c;
  c.depth = depth;
  c.devices = devices;
  c.fwd_cost = std::vector<Rat>(static_cast<std::size_t>(depth), fwd);
  c.bwd_cost = std::vector<Rat>(static_cast<std::size_t>(depth), bwd);
  c.update_cost = update;
  c.comm_cost = comm;
  return c;
}

int ClusterSpec::node_of(int device) const {
  for (std::size_t g = 0; g < nodes.size(); ++g)
    if (std::find(nodes[g].begin(), nodes[g].end(), device) != nodes[g].end())
      return static_cast<int>(g);
  return 0;
}

Rat ClusterSpec::gap(int from_device, int to_device) const {
  if (from_device == to_device) return Rat(0);
  const bool cross_node =
      !nodes.empty() && inter_node_cost.has_value() && node_of(from_device) != node_of(to_device);
  return cross_node ? *inter_node_cost : comm_cost;
}

static Rat mean_of(const std::vector<Rat>& v) {
  Rat s(0);
  for (const Rat& r : v) s += r;
  return s / Rat(static_cast<std::int64_t>(v.size()));
}
Rat ClusterSpec::mean_fwd() const { return mean_of(fwd_cost); }
Rat ClusterSpec::mean_bwd() const { return mean_of(bwd_cost); }

std::vector<TaskEvent> Timeline::flat() const {
  std::vector<TaskEvent> all;
  for (const auto& d : per_device) all.insert(all.end(), d.begin(), d.end());
  return all;
}

int MismatchReport::max_overall() const {
  int m = 0;
  for (const auto& kv : entries) m = std::max(m, kv.second);
  return m;
}

// ------------------------------------------------------------------ validation
std::vector<std::string> validate_cluster(const ClusterSpec& c) {
  std::vector<std::string> out;
  if (c.depth < 2) out.push_back("depth: must be >= 2 (got " + std::to_string(c.depth) + ")");
  if (c.devices < 1) out.push_back("devices: must be >= 1 (got " + std::to_string(c.devices) + ")");
  if (static_cast<int>(c.fwd_cost.size()) != c.depth)
    out.push_back("fwd_cost: expected one entry per stage");
  if (static_cast<int>(c.bwd_cost.size()) != c.depth)
    out.push_back("bwd_cost: expected one entry per stage");
  for (std::size_t i = 0; i < c.fwd_cost.size(); ++i)
    if (c.fwd_cost[i] <= Rat(0))
      out.push_back("fwd_cost[" + std::to_string(i) + "]: must be strictly positive");
  for (std::size_t i = 0; i < c.bwd_cost.size(); ++i)
    if (c.bwd_cost[i] <= Rat(0))
      out.push_back("bwd_cost[" + std::to_string(i) + "]: must be strictly positive");
  if (c.update_cost < Rat(0)) out.push_back("update_cost: must be nonnegative");
  if (c.comm_cost < Rat(0)) out.push_back("comm_cost: must be nonnegative");
  if (c.inter_node_cost && *c.inter_node_cost < Rat(0))
    out.push_back("inter_node_cost: must be nonnegative");
  if (!c.nodes.empty()) {
    std::vector<int> hits(static_cast<std::size_t>(std::max(c.devices, 0)), 0);
    bool partition = true;
    for (const auto& group : c.nodes)
      for (int d : group) {
        if (d < 0 || d >= c.devices) partition = false;
        else ++hits[static_cast<std::size_t>(d)];
      }
    if (std::any_of(hits.begin(), hits.end(), [](int h) { return h != 1; })) partition = false;
    if (!partition) out.push_back("nodes: must partition the device set");
  }
  return out;
}

std::vector<std::string> validate_policy(const PolicyConfig& p, const ClusterSpec& c) {
  std::vector<std::string> out;
  auto bad = [&](std::string s) { out.push_back(std::move(s)); };
  if (p.injection_limit < 1) bad("injection_limit: must be >= 1");
  if (p.accumulation_threshold < 1) bad("accumulation_threshold: must be >= 1");
  if (p.num_minibatches < 1) bad("num_minibatches: must be >= 1");
  if (p.num_pipelines < 1) bad("num_pipelines: must be >= 1");
  if (p.zero_enabled && p.policy != Policy::AMDP) bad("zero_enabled: only supported for AMDP");
  const std::string pn = policy_name(p.policy);
  switch (p.policy) {
    case Policy::AMDP:
      if (c.depth % 2 != 0) bad("AMDP: depth must be even");
      if (c.devices != c.depth) bad("AMDP: devices must equal depth");
      if (!p.injection_override && p.injection_limit != 2)
        bad("AMDP: injection_limit is fixed to 2 (set injection_override to sweep)");
      if (c.depth % 2 == 0 && p.num_pipelines != c.depth / 2)
        bad("AMDP: num_pipelines must equal depth/2");
      if (p.num_pipelines >= 1) {
        if (p.accumulation_threshold % p.num_pipelines != 0)
          bad("AMDP: accumulation_threshold must be a multiple of num_pipelines");
        else if (p.accumulation_threshold / p.num_pipelines < p.injection_limit)
          bad("AMDP: accumulation_threshold must give each pipeline at least injection_limit "
              "minibatches per window");
      }
      break;
    case Policy::Chimera:
      if (c.depth % 2 != 0) bad("Chimera: depth must be even");
      if (c.devices != c.depth) bad("Chimera: devices must equal depth");
      if (p.num_pipelines != 2) bad("Chimera: num_pipelines must be 2");
      if (p.accumulation_threshold != p.injection_limit)
        bad("Chimera: accumulation_threshold must equal injection_limit");
      if (p.injection_limit % 2 != 0)
        bad("Chimera: injection_limit must be even (split across two pipelines)");
      break;
    case Policy::DAPPLE:
    case Policy::GPipe:
      if (c.devices != c.depth) bad(pn + ": devices must equal depth");
      if (p.num_pipelines != 1) bad(pn + ": num_pipelines must be 1");
      if (p.accumulation_threshold != p.injection_limit)
        bad(pn + ": accumulation_threshold must equal injection_limit");
      break;
    case Policy::Interleaved1F1B:
      if (c.depth != 2 * c.devices)
        bad("Interleaved1F1B: depth must equal 2*devices (two chunks per device)");
      if (p.num_pipelines != 1) bad("Interleaved1F1B: num_pipelines must be 1");
      if (p.accumulation_threshold != p.injection_limit)
        bad("Interleaved1F1B: accumulation_threshold must equal injection_limit");
      break;
    case Policy::PipeDreamAsync:
      if (c.devices != c.depth) bad("PipeDreamAsync: devices must equal depth");
      if (p.num_pipelines != 1) bad("PipeDreamAsync: num_pipelines must be 1");
      if (p.injection_limit > c.depth) bad("PipeDreamAsync: injection_limit must be <= depth");
      break;
  }
  return out;
}

// ------------------------------------------------------------------ placement
int map_stage_to_device(int pipeline, int stage, int depth) {
  if (depth < 2 || depth % 2 != 0)
    throw std::invalid_argument("stage mapping requires even depth >= 2");
  if (stage < 0 || stage >= depth || pipeline < 0 || pipeline >= depth / 2)
    throw std::invalid_argument("stage mapping: index out of range");
  // even pipelines walk the device ring upward from 2p, odd ones downward from 2p+1
  const int origin = 2 * pipeline;
  return (pipeline % 2 == 0) ? (origin + stage) % depth : (origin + 1 - stage + depth) % depth;
}

int default_num_pipelines(int depth) {
  if (depth < 2 || depth % 2 != 0)
    throw std::invalid_argument("pipeline count requires even depth >= 2; got " +
                                std::to_string(depth));
  return depth / 2;
}

Rat active_ratio(int injection_limit, int depth) { return Rat(injection_limit, depth); }

int preload_count(const Rat& bwd, const Rat& fwd) {
  if (fwd <= Rat(0)) throw std::invalid_argument("preload_count: fwd must be positive");
  return static_cast<int>((bwd / fwd).floor());
}

// ------------------------------------------------------------------ builder
namespace {

using Shares = std::vector<std::vector<int>>;  // [window] -> minibatches of one pipeline

// One-forward-one-backward program of a stage replica across windows (the lane of a
// non-AMDP policy): at most `cap` in flight, `preload` next-window forwards pulled into
// each window's drain.
std::vector<std::pair<Kind, int>> replica_program(const Shares& wins, int cap, int preload) {
  std::vector<std::pair<Kind, int>> prog;
  const std::size_t W = wins.size();
  std::vector<std::size_t> carried(W + 1, 0);
  int live = 0;
  for (std::size_t w = 0; w < W; ++w) {
    std::vector<int> fwd(wins[w].begin() + static_cast<std::ptrdiff_t>(carried[w]), wins[w].end());
    if (w + 1 < W) {
      const std::size_t k = std::min<std::size_t>(static_cast<std::size_t>(std::max(preload, 0)),
                                                  wins[w + 1].size());
      carried[w + 1] = k;
      fwd.insert(fwd.end(), wins[w + 1].begin(), wins[w + 1].begin() + static_cast<std::ptrdiff_t>(k));
    }
    std::size_t f = 0;
    for (std::size_t b = 0; b < wins[w].size();) {
      if (f < fwd.size() && live < cap) {
        prog.emplace_back(Kind::Forward, fwd[f++]);
        ++live;
      } else {
        prog.emplace_back(Kind::Backward, wins[w][b++]);
        --live;
      }
    }
    for (; f < fwd.size(); ++f) {
      prog.emplace_back(Kind::Forward, fwd[f]);
      ++live;
    }
  }
  return prog;
}

struct Builder {
  const PolicyConfig& cfg;
  const ClusterSpec& cl;
  TaskGraph g;
  int depth = 0, M = 0, thr = 1, W = 1, P = 1, preload = 0;
  bool windowed = true;
  std::vector<Shares> shares;  // [pipeline]
  std::vector<char> pre;       // [minibatch]
  std::vector<int> fid, bid;   // [stage * M + minibatch]

  Builder(const PolicyConfig& c, const ClusterSpec& k) : cfg(c), cl(k) {}

  int device_of(int p, int i) const {
    switch (cfg.policy) {
      case Policy::AMDP: return map_stage_to_device(p, i, depth);
      case Policy::Chimera: return p == 0 ? i : depth - 1 - i;
      case Policy::Interleaved1F1B: return i % cl.devices;
      default: return i;
    }
  }
  int cap_of(int i) const {
    if (cfg.policy == Policy::GPipe) return INT_MAX;
    if (cfg.policy == Policy::Chimera) return std::min(depth / 2, depth - i);
    return std::min(cfg.injection_limit, depth - i);
  }
  int task(Kind k, int stage, int mb, int pipe, int dev, Rat dur, int win, bool is_pre = false) {
    g.tasks.push_back(Task{k, stage, mb, pipe, dev, dur, win, is_pre});
    return static_cast<int>(g.tasks.size()) - 1;
  }
  void edge(int a, int b) { g.deps.emplace_back(a, b); }
  std::size_t at(int i, int j) const {
    return static_cast<std::size_t>(i) * static_cast<std::size_t>(M) + static_cast<std::size_t>(j);
  }

  void plan() {
    depth = cl.depth;
    M = cfg.num_minibatches;
    thr = cfg.accumulation_threshold;
    W = (M + thr - 1) / thr;
    windowed = cfg.policy != Policy::PipeDreamAsync;
    P = cfg.policy == Policy::AMDP ? cfg.num_pipelines : (cfg.policy == Policy::Chimera ? 2 : 1);
    preload = cfg.policy == Policy::AMDP
                  ? std::min(preload_count(cl.mean_bwd(), cl.mean_fwd()), cfg.injection_limit)
                  : 0;
    g.policy = cfg.policy;
    g.depth = depth;
    g.devices = cl.devices;
    g.threshold = thr;
    shares.assign(static_cast<std::size_t>(P), Shares(static_cast<std::size_t>(windowed ? W : 1)));
    for (int j = 0; j < M; ++j)
      shares[static_cast<std::size_t>(j % P)][static_cast<std::size_t>(windowed ? j / thr : 0)]
          .push_back(j);
    pre.assign(static_cast<std::size_t>(M), 0);
    if (preload > 0)
      for (const Shares& s : shares)
        for (std::size_t w = 1; w < s.size(); ++w)
          for (std::size_t k = 0; k < std::min<std::size_t>(static_cast<std::size_t>(preload), s[w].size()); ++k)
            pre[static_cast<std::size_t>(s[w][k])] = 1;
  }

  void compute_tasks() {
    fid.assign(static_cast<std::size_t>(depth) * static_cast<std::size_t>(M), -1);
    bid.assign(fid.size(), -1);
    for (int j = 0; j < M; ++j) {
      const int p = j % P, w = j / thr;
      for (int i = 0; i < depth; ++i) {
        const int dv = device_of(p, i);
        const auto si = static_cast<std::size_t>(i);
        fid[at(i, j)] = task(Kind::Forward, i, j, p, dv, cl.fwd_cost[si], w, pre[static_cast<std::size_t>(j)] != 0);
        bid[at(i, j)] = task(Kind::Backward, i, j, p, dv, cl.bwd_cost[si], w);
      }
    }
    for (int j = 0; j < M; ++j)
      for (int i = 0; i < depth; ++i) {
        edge(fid[at(i, j)], bid[at(i, j)]);
        if (i + 1 < depth) edge(fid[at(i, j)], fid[at(i + 1, j)]);
        if (i > 0) edge(bid[at(i, j)], bid[at(i - 1, j)]);
      }
  }

  // Entry admission: the k-th entry forward of a pipeline waits for the backward of its
  // (k - n)-th minibatch at stage 1 (the signal reaching the entry stage).
  void injection_pacing() {
    if (cfg.policy != Policy::AMDP) return;
    const int n = cfg.injection_limit;
    const int sig = depth > 1 ? 1 : 0;
    for (const Shares& s : shares) {
      std::vector<int> seq;
      for (const auto& w : s) seq.insert(seq.end(), w.begin(), w.end());
      for (std::size_t k = static_cast<std::size_t>(n); k < seq.size(); ++k)
        edge(bid[at(sig, seq[k - static_cast<std::size_t>(n)])], fid[at(0, seq[k])]);
    }
  }

  void per_backward_updates() {  // PipeDreamAsync: one update per backward, chained
    for (int i = 0; i < depth; ++i) {
      int last = -1;
      for (int j = 0; j < M; ++j) {
        const int u = task(Kind::Update, i, j, 0, i, cl.update_cost, j / thr);
        edge(bid[at(i, j)], u);
        if (last >= 0) edge(last, u);
        last = u;
      }
    }
  }

  void sharded_window_updates() {  // ZeRO: Reduce(w,i) -> Broadcast(w,i) at owner i
    std::vector<int> red(static_cast<std::size_t>(W * depth)), bc(red.size());
    auto u = [&](int w, int i) { return static_cast<std::size_t>(w * depth + i); };
    for (int w = 0; w < W; ++w)
      for (int i = 0; i < depth; ++i) {
        red[u(w, i)] = task(Kind::Reduce, i, w, 0, i, cl.update_cost, w);
        bc[u(w, i)] = task(Kind::Broadcast, i, w, 0, i, cl.update_cost, w);
        edge(red[u(w, i)], bc[u(w, i)]);
        if (w > 0) edge(bc[u(w - 1, i)], red[u(w, i)]);
      }
    for (int j = 0; j < M; ++j) {
      const int w = j / thr;
      const bool is_pre = pre[static_cast<std::size_t>(j)] != 0;
      for (int i = 0; i < depth; ++i) {
        edge(bid[at(i, j)], red[u(w, i)]);
        if (is_pre) {
          edge(fid[at(i, j)], red[u(w - 1, i)]);  // forward reads version w-1
          edge(bc[u(w - 1, i)], bid[at(i, j)]);   // backward reads version w
          if (w >= 2) edge(bc[u(w - 2, i)], fid[at(i, j)]);
        } else if (w > 0) {
          edge(bc[u(w - 1, i)], fid[at(i, j)]);
        }
      }
    }
  }

  void replicated_window_updates() {  // every replica updates after all window backwards
    std::vector<int> up(static_cast<std::size_t>(W * depth * P));
    auto u = [&](int w, int i, int p) { return static_cast<std::size_t>((w * depth + i) * P + p); };
    for (int w = 0; w < W; ++w)
      for (int i = 0; i < depth; ++i)
        for (int p = 0; p < P; ++p) {
          up[u(w, i, p)] = task(Kind::Update, i, w, p, device_of(p, i), cl.update_cost, w);
          if (w > 0) edge(up[u(w - 1, i, p)], up[u(w, i, p)]);
        }
    for (int j = 0; j < M; ++j) {
      const int w = j / thr, jp = j % P;
      const bool is_pre = pre[static_cast<std::size_t>(j)] != 0;
      for (int i = 0; i < depth; ++i) {
        for (int p = 0; p < P; ++p) edge(bid[at(i, j)], up[u(w, i, p)]);
        if (is_pre) {
          edge(fid[at(i, j)], up[u(w - 1, i, jp)]);
          edge(up[u(w - 1, i, jp)], bid[at(i, j)]);
          if (w >= 2) edge(up[u(w - 2, i, jp)], fid[at(i, j)]);
        } else if (w > 0) {
          edge(up[u(w - 1, i, jp)], fid[at(i, j)]);
        }
      }
    }
  }

  // Chimera replica order: the zero-queue reference schedule (builder.hpp:306-335).
  std::vector<std::pair<Kind, int>> chimera_program(int p, int i) const {
    const Rat tf = cl.mean_fwd(), tb = cl.mean_bwd(), unit = tf + tb;
    const int half = depth / 2;
    std::vector<std::pair<Kind, int>> prog;
    for (const auto& share : shares[static_cast<std::size_t>(p)]) {
      std::vector<std::tuple<Rat, int, int>> keyed;
      for (std::size_t k = 0; k < share.size(); ++k) {
        const int kk = static_cast<int>(k);
        const Rat inject = unit * Rat(kk % half) + unit * Rat(depth) * Rat(kk / half);
        keyed.emplace_back(inject + tf * Rat(i), 1, share[k]);
        keyed.emplace_back(inject + tf * Rat(depth) + tb * Rat(depth - 1 - i), 0, share[k]);
      }
      std::sort(keyed.begin(), keyed.end());
      for (const auto& [t, fwd, j] : keyed) prog.emplace_back(fwd ? Kind::Forward : Kind::Backward, j);
    }
    return prog;
  }

  void lanes() {
    if (cfg.policy == Policy::AMDP) return;  // order comes from edges + dispatch only
    for (int p = 0; p < P; ++p)
      for (int i = 0; i < depth; ++i) {
        const auto prog = cfg.policy == Policy::Chimera
                              ? chimera_program(p, i)
                              : replica_program(shares[static_cast<std::size_t>(p)], cap_of(i), preload);
        std::vector<int> lane;
        lane.reserve(prog.size());
        for (const auto& [k, j] : prog) lane.push_back(k == Kind::Forward ? fid[at(i, j)] : bid[at(i, j)]);
        if (!lane.empty()) g.lanes.push_back(std::move(lane));
      }
  }

  TaskGraph run() {
    auto v = validate_cluster(cl);
    auto vp = validate_policy(cfg, cl);
    v.insert(v.end(), vp.begin(), vp.end());
    if (!v.empty()) throw std::invalid_argument("invalid configuration: " + v.front());
    plan();
    compute_tasks();
    injection_pacing();
    if (cfg.policy == Policy::PipeDreamAsync) per_backward_updates();
    else if (cfg.zero_enabled) sharded_window_updates();
    else replicated_window_updates();
    lanes();
    return std::move(g);
  }
};

}  // namespace

TaskGraph build(const PolicyConfig& cfg, const ClusterSpec& cl) { return Builder(cfg, cl).run(); }

std::vector<std::vector<int>> TaskGraph::fifo_hint() const {
  using Key = std::tuple<int, int, int, int, int, int>;
  auto key = [&](int id) {
    const Task& t = tasks[static_cast<std::size_t>(id)];
    return Key{t.window, t.minibatch, t.pipeline, kind_rank(t.kind), t.stage, id};
  };
  std::vector<std::vector<std::vector<int>>> per_dev(static_cast<std::size_t>(devices));
  std::vector<char> laned(tasks.size(), 0);
  for (const auto& lane : lanes) {
    if (lane.empty()) continue;
    per_dev[static_cast<std::size_t>(tasks[static_cast<std::size_t>(lane[0])].device)].push_back(lane);
    for (int t : lane) laned[static_cast<std::size_t>(t)] = 1;
  }
  for (std::size_t t = 0; t < tasks.size(); ++t)
    if (!laned[t]) per_dev[static_cast<std::size_t>(tasks[t].device)].push_back({static_cast<int>(t)});
  std::vector<std::vector<int>> out(static_cast<std::size_t>(devices));
  for (int d = 0; d < devices; ++d) {
    auto& ls = per_dev[static_cast<std::size_t>(d)];
    std::vector<std::size_t> head(ls.size(), 0);
    for (;;) {
      int pick = -1;
      std::size_t pick_lane = 0;
      for (std::size_t l = 0; l < ls.size(); ++l) {
        if (head[l] >= ls[l].size()) continue;
        const int c = ls[l][head[l]];
        if (pick < 0 || key(c) < key(pick)) {
          pick = c;
          pick_lane = l;
        }
      }
      if (pick < 0) break;
      out[static_cast<std::size_t>(d)].push_back(pick);
      ++head[pick_lane];
    }
  }
  return out;
}

}  // namespace ppsim
