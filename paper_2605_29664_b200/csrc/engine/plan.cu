// Planning half of the stage executor (see executor.hpp): the constructor (schedule, partition,
// fold within replica groups, hosting, ZeRO shards), the communication / activation-slot /
// boundary-buffer plan, the compute-stream hazard plan, and the plan / memory / version
// reports.
#include "executor.hpp"

namespace amdp {

// Balanced contiguous partition of L layers over `depth` stages.  The LM head (+ final LN and
// cross-entropy) on the last stage costs 6hV training flops per token against a layer's
// 6(4h^2 + 2h ffn) + 6 s h (causal attention), i.e. ~1.9 layer-equivalents for GPT-1.3B
// (measured on B200: 1.7).  Among partitions with the smallest maximum stage cost, take the
// one with the fewest stages at that maximum: the AMDP projection from measured stage costs
// (profiles/r01_sweep) gives [4,3,3,3,3,3,3,2] 9.7% bubble vs 11.5% for [4,4,3,3,3,3,3,1].
std::vector<int> balance_layers(int L, int depth, int h, int V, int ffn, int seq, bool causal) {
  const double layer = 6.0 * (4.0 * h * h + 2.0 * h * ffn) + (causal ? 6.0 : 12.0) * seq * h;
  const double head = 6.0 * h * static_cast<double>(V) / layer;
  std::vector<int> best;
  double best_max = 1e300;
  int best_at_max = 1 << 30;
  // last stage gets k layers, the rest spread as evenly as possible
  for (int k = 0; k <= L; ++k) {
    const int rest = L - k;
    if (depth > 1 && rest < depth - 1) continue;
    std::vector<int> p(static_cast<size_t>(depth), 0);
    if (depth == 1) {
      p[0] = L;
    } else {
      for (int i = 0; i < depth - 1; ++i) p[static_cast<size_t>(i)] = rest / (depth - 1) + (i < rest % (depth - 1) ? 1 : 0);
      p[static_cast<size_t>(depth - 1)] = k;
    }
    std::vector<double> c(static_cast<size_t>(depth));
    double mx = 0;
    for (int i = 0; i < depth; ++i) {
      c[static_cast<size_t>(i)] = p[static_cast<size_t>(i)] + (i == depth - 1 ? head : 0.0);
      mx = std::max(mx, c[static_cast<size_t>(i)]);
    }
    int at_max = 0;
    for (double x : c) at_max += x > mx - 1e-9 ? 1 : 0;
    if (k >= 1 && (mx < best_max - 1e-9 || (mx < best_max + 1e-9 && at_max < best_at_max))) {
      best_max = mx;
      best_at_max = at_max;
      best = p;
    }
  }
  return best;
}

Engine::Engine(const amdp_model_config& mc, const amdp_run_config& rc, const uint8_t* nccl_id)
    : mc_(mc), rc_(rc) {
  depth_ = rc.depth > 0 ? rc.depth : rc.policy.num_pipelines * 2;
  world_ = std::max(1, rc.world_size);
  rank_ = rc.rank;
  policy_ = static_cast<ppsim::Policy>(rc.policy.policy);
  zero_ = rc.policy.zero_enabled != 0;
  // logical devices: Interleaved1F1B places two stage chunks per device (validate.hpp:96-98)
  devices_ = policy_ == ppsim::Policy::Interleaved1F1B ? depth_ / 2 : depth_;
  switch (policy_) {
    case ppsim::Policy::AMDP:
      if (depth_ != 2 * rc.policy.num_pipelines)
        throw std::invalid_argument("engine: AMDP runs depth = 2 x num_pipelines stages");
      P_ = rc.policy.num_pipelines;
      break;
    case ppsim::Policy::Chimera:
      P_ = 2;
      break;
    case ppsim::Policy::DAPPLE:
    case ppsim::Policy::GPipe:
    case ppsim::Policy::Interleaved1F1B:
    case ppsim::Policy::PipeDreamAsync:
      P_ = 1;
      break;
    default:
      throw std::invalid_argument("engine: unknown policy");
  }
  versioned_ = !zero_ && P_ > 1;
  if (devices_ < 1 || devices_ % world_ != 0)
    throw std::invalid_argument("engine: logical devices must be a multiple of world_size");
  per_rank_ = devices_ / world_;
  M_ = rc.policy.num_minibatches;
  thr_ = rc.policy.accumulation_threshold;
  if (M_ % thr_ != 0) throw std::invalid_argument("engine: num_minibatches must be a multiple of accumulation_threshold");
  // PipeDreamAsync updates after every backward (builder.hpp:260-270): one minibatch per step
  update_div_ = policy_ == ppsim::Policy::PipeDreamAsync ? 1.f : static_cast<float>(thr_);
  W_ = M_ / thr_;

  dm.L = mc.layers;
  dm.h = mc.hidden;
  dm.heads = mc.heads;
  dm.hd = mc.hidden / mc.heads;
  dm.ffn = mc.ffn;
  dm.V = mc.vocab;
  dm.S = mc.seq;
  dm.B = mc.seqs_per_minibatch;
  dm.T = dm.B * dm.S;
  dm.causal = mc.causal != 0;
  dm.ln_eps = mc.ln_eps > 0 ? mc.ln_eps : 1e-5f;
  dm.recompute = mc.recompute != 0;
  dm.fp32 = mc.fp32_validation != 0;
  dm.pad_token = dm.causal ? 0 : std::max(0, mc.pad_token);
  if (mc.pad_token > 0 && dm.causal) throw std::invalid_argument("engine: pad_token is for bidirectional models");
  if (dm.fp32 && dm.recompute) throw std::invalid_argument("engine: fp32 validation mode stores every activation (no recompute)");
  if (dm.h % dm.heads != 0) throw std::invalid_argument("engine: hidden must divide into heads");
  if (!dm.fp32 && (amdp_attention_impl(dm.S, dm.hd, 0) < 0 || amdp_attention_impl(dm.S, dm.hd, 1) < 0))
    throw std::invalid_argument("engine: no tensor-core attention kernel for seq " + std::to_string(dm.S) +
                                ", head_dim " + std::to_string(dm.hd) +
                                " (seq % 256 == 0 with head_dim 64 / 80 / 128, or seq <= 128 with head_dim 32 / 64)");

  // schedule: build + order on the declared cost model
  ppsim::ClusterSpec cl = ppsim::ClusterSpec::uniform(depth_, devices_, from_c(rc.declared_fwd),
                                                      from_c(rc.declared_bwd));
  ppsim::PolicyConfig pc = policy_from_c(&rc.policy);
  sched.cl = cl;
  sched.cfg = pc;
  sched.g = ppsim::build(pc, cl);
  sched.tl = ppsim::simulate_with_order(sched.g, cl, &sched.order);
  sched.has_graph = sched.has_timeline = true;

  // partition
  if (mc.layers_per_stage) {
    part.assign(mc.layers_per_stage, mc.layers_per_stage + depth_);
    int s = 0;
    for (int x : part) s += x;
    if (s != dm.L) throw std::invalid_argument("engine: layers_per_stage must sum to layers");
  } else {
    part = balance_layers(dm.L, depth_, dm.h, dm.V, dm.ffn, dm.S, dm.causal);
    if (part.empty()) throw std::invalid_argument("engine: cannot partition layers over stages");
  }
  int l = 0;
  for (int i = 0; i < depth_; ++i) {
    stages.emplace_back(new GptStage(dm, i, depth_, l, l + part[static_cast<size_t>(i)]));
    l += part[static_cast<size_t>(i)];
  }

  // fold logical devices onto ranks within replica groups: devices running a common stage
  // form one component (union-find); devices ordered by (component's smallest device,
  // device) are cut into world_ contiguous chunks of per_rank_.  AMDP D=8: components
  // {0,3,4,7} and {1,2,5,6} (map_stage_to_device, H/builder.hpp:81-88), so N=2 needs no
  // collective and N=4 pairs {0,3},{4,7},{1,2},{5,6}; DAPPLE / GPipe (stage i on device i)
  // fold contiguously.
  {
    std::vector<int> up(static_cast<size_t>(devices_));
    for (int d = 0; d < devices_; ++d) up[static_cast<size_t>(d)] = d;
    auto find = [&](int d) {
      while (up[static_cast<size_t>(d)] != d) d = up[static_cast<size_t>(d)] = up[static_cast<size_t>(up[static_cast<size_t>(d)])];
      return d;
    };
    std::vector<int> first_dev(static_cast<size_t>(depth_), -1);
    for (const auto& t : sched.g.tasks) {
      if (t.kind != ppsim::Kind::Forward && t.kind != ppsim::Kind::Backward) continue;
      int& f = first_dev[static_cast<size_t>(t.stage)];
      if (f < 0) {
        f = t.device;
        continue;
      }
      const int a = find(f), b = find(t.device);
      if (a != b) up[static_cast<size_t>(std::max(a, b))] = std::min(a, b);
    }
    std::vector<int> ord(static_cast<size_t>(devices_));
    for (int d = 0; d < devices_; ++d) ord[static_cast<size_t>(d)] = d;
    if (per_rank_ > 1)  // one device per rank: rank r runs logical device r
      std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return find(a) < find(b); });
    dev_rank_.assign(static_cast<size_t>(devices_), 0);
    for (int k = 0; k < devices_; ++k) dev_rank_[static_cast<size_t>(ord[static_cast<size_t>(k)])] = k / per_rank_;
  }

  // hosting
  hosted.assign(static_cast<size_t>(depth_), false);
  owned.assign(static_cast<size_t>(depth_), false);
  group_ranks_.assign(static_cast<size_t>(depth_), {});
  // replica group of stage i: the ranks whose devices run a Forward / Backward of stage i
  // (AMDP: map_stage_to_device over the d/2 pipelines, builder.hpp:81-88; Chimera: i and d-1-i;
  // Interleaved1F1B: i mod devices; the others: device i).  ZeRO: the owner (device i) keeps the
  // optimizer state; otherwise every hosting rank does (replicated update).
  for (const auto& t : sched.g.tasks) {
    if (t.kind != ppsim::Kind::Forward && t.kind != ppsim::Kind::Backward) continue;
    auto& gr = group_ranks_[static_cast<size_t>(t.stage)];
    const int r = rank_of_dev(t.device);
    if (std::find(gr.begin(), gr.end(), r) == gr.end()) gr.push_back(r);
  }
  for (int i = 0; i < depth_; ++i) {
    std::sort(group_ranks_[static_cast<size_t>(i)].begin(), group_ranks_[static_cast<size_t>(i)].end());
    hosted[static_cast<size_t>(i)] = std::count(group_ranks_[static_cast<size_t>(i)].begin(),
                                                group_ranks_[static_cast<size_t>(i)].end(), rank_) > 0;
    owned[static_cast<size_t>(i)] = zero_ ? owner_rank(i) == rank_ : hosted[static_cast<size_t>(i)];
  }
  // ZeRO shards: every parameter segment split over the replica group in 64-element-aligned
  // parts, part j to member j (sharded(i) groups only; otherwise the owner holds everything)
  shard_.assign(static_cast<size_t>(depth_), {});
  opt_off_.assign(static_cast<size_t>(depth_), {});
  opt_numel_.assign(static_cast<size_t>(depth_), 0);
  for (int i = 0; i < depth_; ++i) {
    const int64_t n = stages[static_cast<size_t>(i)]->numel();
    if (!sharded(i)) {
      if (owned[static_cast<size_t>(i)]) opt_numel_[static_cast<size_t>(i)] = n;
      continue;
    }
    const size_t G = group_ranks_[static_cast<size_t>(i)].size();
    auto& sh = shard_[static_cast<size_t>(i)];
    sh.assign(G, {});
    for (const auto& [off, len] : stages[static_cast<size_t>(i)]->segments()) {
      const int64_t q = ((len + static_cast<int64_t>(G) - 1) / static_cast<int64_t>(G) + 63) / 64 * 64;
      for (size_t j = 0; j < G; ++j) {
        const int64_t lo = std::min(len, q * static_cast<int64_t>(j)), hi = std::min(len, lo + q);
        sh[j].emplace_back(static_cast<size_t>(off + lo), static_cast<size_t>(off + hi));
      }
    }
    owned[static_cast<size_t>(i)] = hosted[static_cast<size_t>(i)];
    if (hosted[static_cast<size_t>(i)]) {
      int64_t c = 0;
      for (const auto& [lo, hi] : sh[static_cast<size_t>(member(i))]) {
        opt_off_[static_cast<size_t>(i)].push_back(c);
        c += static_cast<int64_t>(hi - lo);
      }
      opt_numel_[static_cast<size_t>(i)] = c;
    }
  }

  make_plan();
  if (rc.plan_only) {  // host-side planning only (multi-rank consistency tests on CPU)
    plan_only_ = true;
    return;
  }
  CUDA_OK(cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking));
  // the window machinery and the data plane run at the highest stream priority: their few,
  // short kernels (optimizer step, transposes, peer reductions, flag signals) then take SMs
  // as the persistent stage GEMMs retire instead of queueing behind the next ones, which is
  // what keeps a Broadcast's latency — the one the gated forwards wait for — short
  int prio_lo = 0, prio_hi = 0;
  CUDA_OK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  static const bool no_prio = getenv("AMDP_NO_UPDATE_PRIORITY") != nullptr;
  const int hi = no_prio ? prio_lo : prio_hi;
  CUDA_OK(cudaStreamCreateWithPriority(&us_, cudaStreamNonBlocking, hi));
  if (!getenv("AMDP_NO_SIDE_STREAM")) {
    CUDA_OK(cudaStreamCreateWithFlags(&side_.side, cudaStreamNonBlocking));
    for (auto& e : side_.ev) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  if (world_ > 1) {
    if (rc.comm_backend == AMDP_COMM_NCCL)
      comm_ = make_nccl_comm(world_, rank_, nccl_id, group_ranks_);
    else
      comm_ = make_ipc_comm(world_, rank_, nmsg_, ncoll_);
    if (comm_->single_stream()) {
      CUDA_OK(cudaStreamCreateWithPriority(&rs_, cudaStreamNonBlocking, hi));
      ss_ = ks_ = rs_;
    } else {
      CUDA_OK(cudaStreamCreateWithPriority(&rs_, cudaStreamNonBlocking, hi));
      CUDA_OK(cudaStreamCreateWithPriority(&ss_, cudaStreamNonBlocking, hi));
      CUDA_OK(cudaStreamCreateWithPriority(&ks_, cudaStreamNonBlocking, hi));
    }
  }
  ev_pool_.resize(64);
  for (auto& e : ev_pool_) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  size_t free0 = 0, free1 = 0, total = 0;
  CUDA_OK(cudaMemGetInfo(&free0, &total));
  allocate();
  CUDA_OK(cudaStreamSynchronize(cs_));
  CUDA_OK(cudaMemGetInfo(&free1, &total));
  measured_alloc_bytes_ = static_cast<int64_t>(free0) - static_cast<int64_t>(free1);
  init_weights();
}

void Engine::make_plan() {
  const auto& g = sched.g;
  const auto& order = sched.order;
  const int N = static_cast<int>(order.size());
  nmsg_ = ncoll_ = 0;
  planned_sends_.clear();
  plan_.assign(static_cast<size_t>(N), TaskPlan{});
  comm_at_.assign(static_cast<size_t>(N), {});
  std::vector<int> pos_of(g.tasks.size());
  for (int k = 0; k < N; ++k) pos_of[static_cast<size_t>(order[static_cast<size_t>(k)])] = k;
  // task ids of F(i,j) / B(i,j)
  std::map<std::pair<int, int>, int> F, B;
  for (std::size_t t = 0; t < g.tasks.size(); ++t) {
    const auto& k = g.tasks[t];
    if (k.kind == ppsim::Kind::Forward) F[{k.stage, k.minibatch}] = static_cast<int>(t);
    if (k.kind == ppsim::Kind::Backward) B[{k.stage, k.minibatch}] = static_cast<int>(t);
  }
  auto rank_of_task = [&](int t) { return rank_of_dev(g.tasks[static_cast<size_t>(t)].device); };

  // activation slots per stage (local tasks only)
  slots_per_stage.assign(static_cast<size_t>(depth_), 0);
  std::vector<std::vector<int>> free_slots(static_cast<size_t>(depth_));
  std::map<std::pair<int, int>, int> slot_of;
  // boundary buffers: interval allocation over positions on this rank
  std::vector<int> free_bufs;
  std::vector<std::vector<int>> release_at(static_cast<size_t>(N));  // buffers freed after position
  // Reuse prefers a free buffer / slot whose last user ran on the same logical device: with
  // concurrent compute streams (one per logical device) the reuse then needs no cross-stream
  // wait; the counts are those of plain LIFO reuse (a free entry is always taken).
  std::map<int, int> buf_dev;                      // buffer -> device of its last use
  std::map<std::pair<int, int>, int> slot_dev;     // (stage, slot) -> device of its last use
  auto take_pref = [](std::vector<int>& fl, const std::function<bool(int)>& same) {
    for (size_t q = fl.size(); q-- > 0;)
      if (same(fl[q])) {
        const int v = fl[q];
        fl.erase(fl.begin() + static_cast<std::ptrdiff_t>(q));
        return v;
      }
    const int v = fl.back();
    fl.pop_back();
    return v;
  };
  int cur_dev = -1;  // device of the task being planned
  auto alloc_buf = [&]() {
    if (!free_bufs.empty())
      return take_pref(free_bufs, [&](int b) { auto it = buf_dev.find(b); return it != buf_dev.end() && it->second == cur_dev; });
    return nbuf++;
  };
  // F boundary (i -> i+1, j): receiver buffer lives [pos F(i,j), pos B(i+1,j)];
  //   on the producer rank (if different) a send buffer lives [pos F(i,j), pos F(i,j)].
  // B boundary (i+1 -> i, j): [pos B(i+1,j), pos B(i,j)] likewise.
  std::map<std::pair<int, int>, int> fbuf_recv, bbuf_recv;  // key (boundary stage i, j)
  std::map<std::pair<int, int>, int> updates_seen;          // key (stage, Update's window / mb)
  for (int k = 0; k < N; ++k) {
    const int t = order[static_cast<size_t>(k)];
    const auto& task = g.tasks[static_cast<size_t>(t)];
    TaskPlan& tp = plan_[static_cast<size_t>(k)];
    const int me = rank_of_task(t);
    tp.local = me == rank_;
    cur_dev = task.device;
    // release buffers whose last use was an earlier position
    if (task.kind == ppsim::Kind::Forward) {
      const int i = task.stage, j = task.minibatch;
      if (tp.local) {
        auto& fl = free_slots[static_cast<size_t>(i)];
        int s;
        if (!fl.empty()) {
          s = take_pref(fl, [&](int x) { auto it = slot_dev.find({i, x}); return it != slot_dev.end() && it->second == cur_dev; });
        } else {
          s = slots_per_stage[static_cast<size_t>(i)]++;
        }
        slot_of[{i, j}] = s;
        tp.slot = s;
        if (i > 0) tp.in_buf = fbuf_recv.at({i - 1, j});
      }
      if (i + 1 < depth_) {
        const int cons = F.at({i + 1, j});
        const int cr = rank_of_task(cons);
        const int last_use = pos_of[static_cast<size_t>(B.at({i + 1, j}))];
        const int msg = cr != me ? nmsg_++ : -1;  // numbered on every rank alike
        if (tp.local) {
          const int b = alloc_buf();
          tp.out_buf = b;
          if (cr == rank_) {
            fbuf_recv[{i, j}] = b;
            release_at[static_cast<size_t>(last_use)].push_back(b);
          } else {
            tp.send_to = cr;
            comm_at_[static_cast<size_t>(k)].push_back({CommOp::Send, cr, b, -1, k, msg});
            planned_sends_.emplace_back(msg, b);
            release_at[static_cast<size_t>(k)].push_back(b);
          }
        } else if (cr == rank_) {
          const int b = alloc_buf();
          fbuf_recv[{i, j}] = b;
          comm_at_[static_cast<size_t>(k)].push_back({CommOp::Recv, me, b, -1, -1, msg});
          release_at[static_cast<size_t>(last_use)].push_back(b);
        }
      }
    } else if (task.kind == ppsim::Kind::Backward) {
      const int i = task.stage, j = task.minibatch;
      if (tp.local) {
        tp.slot = slot_of.at({i, j});
        free_slots[static_cast<size_t>(i)].push_back(tp.slot);
        slot_dev[{i, tp.slot}] = task.device;
        if (i > 0) tp.in_buf = fbuf_recv.at({i - 1, j});
        if (i + 1 < depth_) tp.gin_buf = bbuf_recv.at({i, j});
      }
      if (i > 0) {
        const int cons = B.at({i - 1, j});
        const int cr = rank_of_task(cons);
        const int last_use = pos_of[static_cast<size_t>(cons)];
        const int msg = cr != me ? nmsg_++ : -1;
        if (tp.local) {
          const int b = alloc_buf();
          tp.gout_buf = b;
          if (cr == rank_) {
            bbuf_recv[{i - 1, j}] = b;
            release_at[static_cast<size_t>(last_use)].push_back(b);
          } else {
            tp.send_to = cr;
            comm_at_[static_cast<size_t>(k)].push_back({CommOp::Send, cr, b, -1, k, msg});
            planned_sends_.emplace_back(msg, b);
            release_at[static_cast<size_t>(k)].push_back(b);
          }
        } else if (cr == rank_) {
          const int b = alloc_buf();
          bbuf_recv[{i - 1, j}] = b;
          comm_at_[static_cast<size_t>(k)].push_back({CommOp::Recv, me, b, -1, -1, msg});
          release_at[static_cast<size_t>(last_use)].push_back(b);
        }
      }
    } else if (task.kind == ppsim::Kind::Reduce) {
      const int i = task.stage;
      if (group_ranks_[static_cast<size_t>(i)].size() > 1) {
        const int c = ncoll_++;
        if (hosted[static_cast<size_t>(i)]) comm_at_[static_cast<size_t>(k)].push_back({CommOp::Reduce, -1, -1, i, k, c});
      }
    } else if (task.kind == ppsim::Kind::Broadcast) {
      const int i = task.stage;
      if (group_ranks_[static_cast<size_t>(i)].size() > 1) {  // one collective per parameter segment
        const int c = ncoll_;
        ncoll_ += static_cast<int>(stages[static_cast<size_t>(i)]->segments().size());
        if (hosted[static_cast<size_t>(i)]) comm_at_[static_cast<size_t>(k)].push_back({CommOp::Bcast, -1, -1, i, k, c});
      }
    } else if (task.kind == ppsim::Kind::Update) {
      // Update(w, i, p) (minibatch field = w; PipeDreamAsync: = j).  The first one in the global
      // order steps the optimizer on every rank hosting stage i, after an all-reduce of the
      // window gradient over the replica group (the reference's "all-reduce-equivalent
      // barrier", builder.hpp:306-308): all of the window's backwards precede it.
      const int i = task.stage;
      tp.first_update = updates_seen[{i, task.minibatch}]++ == 0;
      if (tp.first_update && group_ranks_[static_cast<size_t>(i)].size() > 1) {
        const int c = ncoll_++;
        if (hosted[static_cast<size_t>(i)]) comm_at_[static_cast<size_t>(k)].push_back({CommOp::Allreduce, -1, -1, i, k, c});
      }
    }
    for (int b : release_at[static_cast<size_t>(k)]) {
      free_bufs.push_back(b);
      buf_dev[b] = task.device;  // the buffer's last use: this position's task
    }
  }
}

// Cross-stream hazards of the concurrent compute streams, from the resources each local F/B
// task touches in dispatch order: its activation slot (stage, slot), its boundary buffers
// (which also carries the producer -> consumer edge: F(i-1,j) -> F(i,j), B(i+1,j) -> B(i,j)),
// and for a Backward its stage's fp32 window gradient (so the B tasks of a stage accumulate in
// the global order: the same fp32 sums as one stream).  A task waits for the previous user of
// each resource when that ran on another stream.  With one stream the lists only feed the
// window machinery (stage_last_), which then waits for just that stage's last task.
void Engine::plan_streams() {
  const auto& g = sched.g;
  const int N = static_cast<int>(sched.order.size());
  dev_stream_.assign(static_cast<size_t>(devices_), 0);
  {
    int k = 0;
    for (int d = 0; d < devices_; ++d)
      if (rank_of_dev(d) == rank_) dev_stream_[static_cast<size_t>(d)] = (k++) % active_streams_;
  }
  waits_.assign(static_cast<size_t>(N), {});
  stage_last_.assign(static_cast<size_t>(N), {});
  loss_tasks_.assign(static_cast<size_t>(W_), {});
  std::map<std::pair<int, int>, int> slot_last;  // (stage, slot) -> position
  std::map<int, int> buf_last, grad_last;
  std::vector<std::vector<int>> stage_stream_last(static_cast<size_t>(depth_), std::vector<int>(static_cast<size_t>(active_streams_), -1));
  auto stream_at = [&](int q) {
    return dev_stream_[static_cast<size_t>(g.tasks[static_cast<size_t>(sched.order[static_cast<size_t>(q)])].device)];
  };
  for (int k = 0; k < N; ++k) {
    const auto& t = g.tasks[static_cast<size_t>(sched.order[static_cast<size_t>(k)])];
    const TaskPlan& tp = plan_[static_cast<size_t>(k)];
    if (t.kind == ppsim::Kind::Reduce || t.kind == ppsim::Kind::Broadcast || t.kind == ppsim::Kind::Update) {
      stage_last_[static_cast<size_t>(k)] = stage_stream_last[static_cast<size_t>(t.stage)];
      continue;
    }
    if (!tp.local) continue;
    const int me = stream_at(k);
    auto use = [&](int& last) {
      if (last >= 0 && stream_at(last) != me &&
          std::find(waits_[static_cast<size_t>(k)].begin(), waits_[static_cast<size_t>(k)].end(), last) ==
              waits_[static_cast<size_t>(k)].end())
        waits_[static_cast<size_t>(k)].push_back(last);
      last = k;
    };
    auto it = slot_last.emplace(std::make_pair(t.stage, tp.slot), -1).first;
    use(it->second);
    for (int b : {tp.in_buf, tp.out_buf, tp.gin_buf, tp.gout_buf})
      if (b >= 0) use(buf_last.emplace(b, -1).first->second);
    if (t.kind == ppsim::Kind::Backward) use(grad_last.emplace(t.stage, -1).first->second);
    stage_stream_last[static_cast<size_t>(t.stage)][static_cast<size_t>(me)] = k;
    if (t.kind == ppsim::Kind::Forward && t.stage == depth_ - 1) loss_tasks_[static_cast<size_t>(t.window)].push_back(k);
  }
  ln_flush_.assign(static_cast<size_t>(N), 0);
  std::vector<int> pending(static_cast<size_t>(depth_), -1);
  for (int k = 0; k < N; ++k) {
    const auto& t = g.tasks[static_cast<size_t>(sched.order[static_cast<size_t>(k)])];
    int& p = pending[static_cast<size_t>(t.stage)];
    if (t.kind == ppsim::Kind::Reduce || t.kind == ppsim::Kind::Broadcast || t.kind == ppsim::Kind::Update) {
      if (p >= 0) ln_flush_[static_cast<size_t>(p)] = 1;
      p = -1;
    } else if (t.kind == ppsim::Kind::Backward && plan_[static_cast<size_t>(k)].local) {
      p = k;
    }
  }
  for (int p : pending)
    if (p >= 0) ln_flush_[static_cast<size_t>(p)] = 1;
}

namespace {
std::string json_escape(const std::string& in) {
  std::string o;
  for (char c : in) {
    if (c == '"' || c == '\\') o += '\\';
    if (static_cast<unsigned char>(c) >= 0x20) o += c;
  }
  return o;
}
std::string fmt_units(double u) {  // shards of 64-aligned segments: round to 1e-3 of a stage
  char b[32];
  std::snprintf(b, sizeof(b), "%.3f", u);
  std::string s(b);
  while (!s.empty() && s.back() == '0') s.pop_back();
  if (!s.empty() && s.back() == '.') s.pop_back();
  return s;
}
}  // namespace

std::string Engine::plan_json() const {
  std::string s = "{\"depth\":" + std::to_string(depth_) + ",\"world_size\":" + std::to_string(world_) +
                  ",\"rank\":" + std::to_string(rank_) + ",\"tokens_per_minibatch\":" + std::to_string(dm.T) +
                  ",\"comm_backend\":\"" + (world_ == 1 ? "none" : rc_.comm_backend == AMDP_COMM_NCCL ? "nccl" : "ipc") +
                  "\",\"graph_error\":\"" + json_escape(graph_error_) + "\",\"messages\":" + std::to_string(nmsg_) + ",\"collectives\":" + std::to_string(ncoll_) +
                  ",\"compute_streams\":" + std::to_string(active_streams_) + ",\"compute_streams_allocated\":" +
                  std::to_string(nstreams_) + ",\"device_rank\":[";
  for (size_t d = 0; d < dev_rank_.size(); ++d) s += (d ? "," : "") + std::to_string(dev_rank_[d]);
  s += "],\"partition\":[";
  for (size_t i = 0; i < part.size(); ++i) s += (i ? "," : "") + std::to_string(part[i]);
  s += "],\"stages\":[";
  for (int i = 0; i < depth_; ++i) {
    const GptStage& st = *stages[static_cast<size_t>(i)];
    s += std::string(i ? ",{" : "{") + "\"stage\":" + std::to_string(i) + ",\"hosted\":" +
         (hosted[static_cast<size_t>(i)] ? "true" : "false") + ",\"owner\":" +
         (owned[static_cast<size_t>(i)] ? "true" : "false") + ",\"numel\":" + std::to_string(st.numel()) +
         ",\"owner_rank\":" + std::to_string(owner_rank(i)) + ",\"opt_numel\":" +
         std::to_string(opt_numel_[static_cast<size_t>(i)]) + ",\"shard\":[" + shard_json(i) + "]" +
         ",\"slots\":" + std::to_string(slots_per_stage[static_cast<size_t>(i)]) +
         ",\"slot_bytes\":" + std::to_string(st.slot_bytes()) + ",\"group\":[";
    const auto& gr = group_ranks_[static_cast<size_t>(i)];
    for (size_t k = 0; k < gr.size(); ++k) s += (k ? "," : "") + std::to_string(gr[k]);
    s += "],\"params\":[";
    const auto& ps = st.params();
    for (size_t k = 0; k < ps.size(); ++k)
      s += std::string(k ? ",{" : "{") + "\"name\":\"" + ps[k].name + "\",\"offset\":" + std::to_string(ps[k].off) +
           ",\"rows\":" + std::to_string(ps[k].rows) + ",\"cols\":" + std::to_string(ps[k].cols) +
           ",\"global_index\":" + std::to_string(ps[k].global_index) + ",\"init\":" + std::to_string(ps[k].init) +
           ",\"std\":" + std::to_string(ps[k].std) + "}";
    s += "]}";
  }
  s += "],\"memory\":" + memory_json();
  s += ",\"boundary_buffers\":" + std::to_string(nbuf) + ",\"activation_bytes\":" + std::to_string(slot_total_) +
       ",\"workspace_bytes\":" + std::to_string(GptStage::workspace_bytes(dm)) + ",\"comm_ops\":[";
  bool first = true;
  for (size_t k = 0; k < comm_at_.size(); ++k)
    for (const CommOp& op : comm_at_[k]) {
      static const char* names[] = {"send", "recv", "reduce", "bcast", "allreduce"};
      s += std::string(first ? "[" : ",[") + std::to_string(k) + ",\"" + names[op.kind] + "\"," +
           std::to_string(op.peer) + "," + std::to_string(op.stage) + "," + std::to_string(op.id) + "]";
      first = false;
    }
  return s + "]}";
}

std::string Engine::memory_json() const {
  const int64_t T = dm.T, h = dm.h;
  int64_t w = 0, wt = 0, wver = 0, master = 0, grad = 0, opt = 0, act = 0;
  int hosted_n = 0, slots = 0;
  double owned_units = 0;  // optimizer state in stage-weight units (m + v = 2 per full stage)
  for (int i = 0; i < depth_; ++i) {
    if (!hosted[static_cast<size_t>(i)]) continue;
    const int64_t n = stages[static_cast<size_t>(i)]->numel();
    ++hosted_n;
    w += 2 * n;
    wt += 2 * n;
    if (versioned_) wver += 4 * n;
    master += 4 * n;
    grad += 4 * n;
    if (owned[static_cast<size_t>(i)]) {
      opt += 8 * opt_numel_[static_cast<size_t>(i)];
      owned_units += 2.0 * static_cast<double>(opt_numel_[static_cast<size_t>(i)]) / static_cast<double>(n);
    }
    slots += slots_per_stage[static_cast<size_t>(i)];
    act += static_cast<int64_t>(slots_per_stage[static_cast<size_t>(i)]) *
           static_cast<int64_t>(stages[static_cast<size_t>(i)]->slot_bytes());
  }
  const int64_t bounds = static_cast<int64_t>(nbuf) * T * h * static_cast<int64_t>(dm.act_bytes());
  const int64_t wsb = static_cast<int64_t>(GptStage::workspace_bytes(dm)) * std::max(1, nstreams_);
  const int64_t io = static_cast<int64_t>(M_) * T * 8 + static_cast<int64_t>(M_) * 4;
  const int64_t total = w + wt + wver + master + grad + opt + act + bounds + wsb + io;
  auto kv = [](const char* k, int64_t v) { return std::string("\"") + k + "\":" + std::to_string(v); };
  return "{" + kv("weights_bf16", w) + "," + kv("weights_transposed_bf16", wt) + "," + kv("weight_versions_bf16", wver) +
         "," + kv("master_fp32", master) + "," + kv("gradient_fp32", grad) + "," + kv("optimizer_state_fp32", opt) +
         "," + kv("activations", act) + "," + kv("boundary_buffers", bounds) + "," + kv("workspace", wsb) + "," +
         kv("token_io", io) + "," + kv("total", total) + "," + kv("measured_device_bytes", measured_alloc_bytes_) +
         "," + kv("weight_units", hosted_n) + "," + kv("gradient_units", hosted_n) + "," +
         "\"optimizer_state_units\":" + fmt_units(owned_units) + "," + kv("activation_slots", slots) + "}";
}

std::string Engine::version_csv() const {
  std::string s = "device,kind,stage,minibatch,pipeline,window,preloaded,version\n";
  std::vector<std::vector<int>> per_dev(static_cast<size_t>(devices_));
  for (size_t k = 0; k < sched.order.size(); ++k) {
    const int t = sched.order[k];
    const auto& task = sched.g.tasks[static_cast<size_t>(t)];
    if ((task.kind == ppsim::Kind::Forward || task.kind == ppsim::Kind::Backward) && plan_[k].local)
      per_dev[static_cast<size_t>(task.device)].push_back(t);
  }
  for (int d = 0; d < devices_; ++d)
    for (int t : per_dev[static_cast<size_t>(d)]) {
      const auto& e = sched.g.tasks[static_cast<size_t>(t)];
      s += std::to_string(d) + ',' + ppsim::kind_name(e.kind) + ',' + std::to_string(e.stage) + ',' +
           std::to_string(e.minibatch) + ',' + std::to_string(e.pipeline) + ',' + std::to_string(e.window) + ',' +
           (e.preloaded ? '1' : '0') + ',' +
           std::to_string(version_seen.empty() ? -1 : version_seen[static_cast<size_t>(t)]) + '\n';
    }
  return s;
}

}  // namespace amdp
