// AMDP stage executor: replays the reference dispatch order (ppsim::simulate_with_order on
// the declared ClusterSpec) on this process's GPU and returns the measured Timeline.
//
//  * Planning (host, once): logical devices are folded onto ranks WITHIN replica groups
//    (devices that share a stage land on the same rank first: AMDP D=8 on 2 GPUs puts
//    {0,3,4,7} / {1,2,5,6} together, so every stage lives on one GPU and no collective is
//    needed), activation slots per (stage, minibatch) from the order, boundary buffers for
//    stage-to-stage activations/gradients with exact liveness, the communication program
//    (send/recv at the producer's position in the global order on both ranks; message and
//    collective ids numbered identically on every rank), and the replica groups of every
//    stage (owner = the rank of logical device i, H/builder.hpp:273).
//  * Streams: compute (stage kernels, in dispatch order), weight-gradient side stream,
//    receive, send, collective and update streams.  Each wait names the one event it needs
//    (a buffer's last compute use, a message's arrival, a stage's new weights), so a stage's
//    window machinery never blocks the compute of other stages.
//  * Window machinery (ZeRO, H/builder.hpp:272-304): Reduce -> the stage's fp32 window
//    gradients summed onto the owner (collective stream; a no-op when every replica is on
//    this GPU: co-resident replicas accumulate into one buffer); Broadcast -> on the update
//    stream, after the compute that read the old weights: the owner's fused optimizer step,
//    then the bf16 weights + fp32 LayerNorm parameters pulled by the other replicas (half of
//    the fp32-master bytes), which refresh their transposed copies.  Only the tasks the
//    reference gates on the Broadcast (BC(w-1,i) -> F / preloaded B, builder.hpp:289-304)
//    wait for it.  Replicated updates (every other schedule): the first Update(w,i,.)
//    all-reduces the window gradient over the stage's ranks and steps the optimizer.
//  * Exchanges go through Comm (comm.hpp): this library's CUDA-IPC peer-memory data plane
//    (default; also runs several ranks on ONE GPU) or NCCL.
//    Parameter versions are exactly the trace's (F sees w - preloaded, B sees w): a
//    device-side counter per stage records what each task actually read.
#include <cuda_runtime.h>

#include <chrono>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "amdp_engine.h"
#include "../kernels/common.cuh"
#include "../sched/sched_handle.hpp"
#include "comm.hpp"
#include "gpt_stage.hpp"
#include "ktimer.hpp"
#include "ppsim/ppsim.hpp"

namespace amdp {

namespace {

__global__ void record_version_kernel(const int* ver, int stage, int* trace, int idx) {
  trace[idx] = ver[stage];
}
__global__ void bump_version_kernel(int* ver, int first, int count) {
  for (int k = 0; k < count; ++k) ver[first + k] += 1;
}
__global__ void cast_f32_bf16_kernel(const float* __restrict__ src, bf16* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

#define CUDA_OK(x)                                                                 \
  do {                                                                             \
    cudaError_t _e = (x);                                                          \
    if (_e != cudaSuccess)                                                         \
      throw std::runtime_error(std::string(#x) + ": " + cudaGetErrorString(_e));   \
  } while (0)

uint64_t tensor_seed(uint64_t model_seed, int gidx) {
  return model_seed * 1000003ull + static_cast<uint64_t>(gidx);
}

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

struct BoundaryBuf {
  uint16_t* ptr = nullptr;
  cudaEvent_t comm_done = nullptr;  // last communication use (send / recv) of this buffer
  bool comm_pending = false;
  cudaEvent_t used = nullptr;       // last compute use (a recv into it waits for this)
  bool use_recorded = false;
};

struct TaskPlan {
  int slot = -1;            // activation slot (F/B)
  int in_buf = -1;          // F: boundary buffer holding the stage input (stages > 0)
  int out_buf = -1;         // F: boundary buffer receiving the stage output (stages < d-1)
  int gin_buf = -1;         // B: incoming gradient buffer (stages < d-1)
  int gout_buf = -1;        // B: outgoing gradient buffer (stages > 0)
  int send_to = -1;         // rank to send out/gout to after this task (-1: none)
  bool local = false;       // executed by this rank
  bool first_update = false;  // Update: the first of its (stage, window) -> the optimizer step
};

struct CommOp {           // issued at a position in the global order
  enum Kind { Send, Recv, Reduce, Bcast, Allreduce } kind;
  int peer = -1;          // send/recv peer rank
  int buf = -1;           // boundary buffer (send/recv)
  int stage = -1;         // reduce/bcast stage
  int after_task = -1;    // order position whose compute it must follow (send/reduce)
  int id = -1;            // message id (send/recv) or collective id, same on every rank
};

}  // namespace

class Engine {
 public:
  Engine(const amdp_model_config& mc, const amdp_run_config& rc, const uint8_t* nccl_id);
  ~Engine();
  void run(const int32_t* inputs, const int32_t* labels, float* losses_out, int max_window = -1,
           bool resident = false);
  void stage_tokens(const int32_t* inputs, const int32_t* labels);
  void set_kernel_timing(bool on) {
    ktimer_.enabled = on;
    for (auto& s : stages) s->kt = on ? &ktimer_ : nullptr;
  }
  KTimer ktimer_;
  std::string plan_json() const;
  std::string shard_json(int i) const {  // this rank's ZeRO ranges of stage i ([] if unsharded)
    std::string r;
    if (!sharded(i) || !hosted[static_cast<size_t>(i)]) return r;
    for (const auto& [lo, hi] : shard_[static_cast<size_t>(i)][static_cast<size_t>(member(i))])
      r += (r.empty() ? "[" : ",[") + std::to_string(lo) + "," + std::to_string(hi) + "]";
    return r;
  }
  std::string version_csv() const;
  int64_t stage_numel(int stage) const;
  void copy_params(int stage, float* host, int64_t n, bool to_host);

  // results
  amdp_run_stats stats{};
  std::vector<ppsim::TaskEvent> events;  // measured, this rank's logical devices
  std::vector<ppsim::TaskEvent> lane_events;  // Reduce / Broadcast on their own streams
  std::vector<int> version_seen;         // per task id (-1 if not local)
  SchedHandle sched;                     // declared graph + timeline + order
  std::vector<std::unique_ptr<GptStage>> stages;
  std::vector<bool> hosted, owned;
  std::vector<int> slots_per_stage;
  int nbuf = 0;
  Dims dm{};
  std::vector<int> part;

 private:
  amdp_model_config mc_;
  amdp_run_config rc_;
  int depth_ = 0, devices_ = 0, world_ = 1, rank_ = 0, per_rank_ = 1, M_ = 0, thr_ = 1, W_ = 1;
  ppsim::Policy policy_ = ppsim::Policy::AMDP;
  bool zero_ = true;  // ZeRO Reduce/Broadcast (AMDP) vs Update tasks (every other schedule)
  int P_ = 1;         // pipelines: version counters are per (stage, pipeline replica)
  // Update-task schedules with several pipelines (AMDP without ZeRO, Chimera): replica p of
  // stage i advances at its own Update(w, i, p) (builder.hpp:306-336), but every replica's k-th
  // update applies the same all-reduced window gradient, so the k-th weights are identical
  // across replicas.  One optimizer state per rank; the first Update(w, i, .) in the global
  // order takes the step into the other of two bf16 weight buffers, and each replica switches
  // buffers at its own Update.  (At most two versions are live: no replica's Update(w + 1)
  // can precede another's Update(w).)
  bool versioned_ = false;
  std::vector<std::array<uint16_t*, 2>> wbuf_, wtbuf_;  // per stage
  std::vector<int> cur_buf_;                             // per stage: newest weights
  std::vector<std::vector<int>> rep_buf_;                // per stage, pipeline
  float update_div_ = 1.f;                               // minibatches per optimizer step
  void use_replica_weights(int stage, int pipeline);
  void optimizer_step(int stage, int step, cudaStream_t st);  // whole stage + transposed copies
  // m_off: where parameter `off`'s optimizer state lives in the stage's m / v (= off unless sharded)
  void optimizer_range(int stage, int step, int64_t off, int64_t n, cudaStream_t st, int64_t m_off = -1);
  std::vector<int> pending_ag_;  // per stage: first collective id of an all-gather not yet confirmed
  // ZeRO within a multi-rank replica group: member j of stage i's group steps the optimizer on
  // shard_[i][j] (its part of every parameter segment) and keeps m / v for those ranges only,
  // packed (opt_off_[i][k]: packed offset of this rank's k-th range)
  bool sharded(int i) const { return zero_ && group_ranks_[static_cast<size_t>(i)].size() > 1; }
  int member(int i) const {
    const auto& g = group_ranks_[static_cast<size_t>(i)];
    return static_cast<int>(std::find(g.begin(), g.end(), rank_) - g.begin());
  }
  std::vector<std::vector<Comm::Ranges>> shard_;
  std::vector<std::vector<int64_t>> opt_off_;
  std::vector<int64_t> opt_numel_;  // per stage: optimizer-state elements on this rank
  int cur_pos_ = 0;  // order position being issued
  int64_t comm_launches_seen_ = 0;
  std::vector<TaskPlan> plan_;               // per order position
  std::vector<std::vector<CommOp>> comm_at_; // per order position
  std::vector<std::vector<uint8_t*>> slot_mem_;
  std::vector<std::vector<SlotActs>> slot_acts_;
  std::vector<BoundaryBuf> bufs_;
  std::vector<std::vector<int>> group_ranks_; // per stage: ranks hosting it
  std::vector<int> dev_rank_;                 // logical device -> rank (fold within replica groups)
  std::unique_ptr<Comm> comm_;                // world_size > 1
  int nmsg_ = 0, ncoll_ = 0;                  // message / collective ids of the global plan
  // compute, receive, send, collective, window-update streams (NCCL: one stream for all comm)
  cudaStream_t cs_ = nullptr, rs_ = nullptr, ss_ = nullptr, ks_ = nullptr, us_ = nullptr;
  std::vector<cudaEvent_t> wready_;   // per stage: new weights in place (update stream)
  std::vector<char> wpending_;        // per (stage, compute stream): next B must wait wready_
  std::vector<char> fpending_;        // per (stage, compute stream): next F waits the segment events
  std::vector<std::vector<std::pair<int64_t, int64_t>>> segs_;  // per stage: GptStage::segments()
  std::vector<std::vector<cudaEvent_t>> seg_ev_;               // per stage, segment: weights in place
  std::vector<cudaEvent_t> reduced_;  // per stage: window gradient reduced (collective stream)
  std::vector<cudaEvent_t> ev_pool_;  // cross-stream hand-offs (recycled round robin)
  size_t ev_next_ = 0;
  cudaEvent_t handoff(cudaStream_t from);  // event recorded on `from` now
  // Timing records: under CUDA-graph capture they become event-record nodes (external), so a
  // replay timestamps them like an eager run.
  bool capturing_ = false;
  void rec(cudaEvent_t e, cudaStream_t s) {
    CUDA_OK(capturing_ ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal) : cudaEventRecord(e, s));
  }
  // CUDA graphs of whole runs (one GPU): a run is a fixed sequence of launches, so after one
  // eager run (lazy initialisation) each new configuration is captured once (streams, events,
  // PDL edges, copies) and replayed: one launch instead of ~17k host API calls per window.
  struct GraphKey {
    int max_window;
    bool resident;
    const void *in, *lab, *loss;
    uint64_t scale_hash;
    bool operator<(const GraphKey& o) const {
      return std::tie(max_window, resident, in, lab, loss, scale_hash) <
             std::tie(o.max_window, o.resident, o.in, o.lab, o.loss, o.scale_hash);
    }
  };
  struct GraphRun {
    cudaGraphExec_t exec = nullptr;
    amdp_run_stats stats{};
    std::vector<char> lane_rec;
  };
  int eager_runs_ = 0;
  std::string graph_error_;  // why capture was abandoned (plan_json "graph_error")
  std::map<GraphKey, GraphRun> graphs_;

 public:
  bool graphs_enabled_ = true;

 private:
  void issue(int max_window, bool resident, const int32_t* h_in, const int32_t* h_lab, float* losses_out);
  uint16_t* bounds_arena_ = nullptr;
  std::vector<std::pair<int, int>> planned_sends_;  // (message id, boundary buffer)
  uint8_t* ws_ = nullptr;
  // Concurrent compute streams (ZeRO AMDP, any rank hosting several logical devices): logical
  // device d's Forward / Backward tasks run in dispatch order on compute stream
  // dev_stream_[d] (cstreams_[0] = cs_), each with its own weight-gradient side stream and
  // workspace, so tasks of different logical
  // devices overlap on the SMs as they would on separate GPUs.  Every cross-stream hazard is
  // an event wait computed at plan time from the resources the tasks touch (activation slots,
  // boundary buffers, a stage's window gradient: B tasks of a stage keep their global order,
  // so the fp32 sums - and the bits - are those of the serial run).
  int nstreams_ = 1;       // compute streams allocated (workspaces, side streams)
  int active_streams_ = 1;  // compute streams the plan uses (<= nstreams_; amdp_engine_set_streams)
  std::vector<cudaStream_t> cstreams_;
  std::vector<SideStream> sides_;
  std::vector<uint8_t*> wss_;
  std::vector<int> dev_stream_;             // per logical device
  std::vector<std::vector<int>> waits_;     // per position: earlier positions (other streams)
  std::vector<std::vector<int>> stage_last_;  // per R / BC position: last local F/B of the stage per stream
  std::vector<std::vector<int>> loss_tasks_;  // per window: local last-stage Forward positions
  std::vector<cudaEvent_t> done_;           // per position: the F/B task complete on its stream
  std::vector<int> tok_loader_;             // per window: position whose stream copied the tokens (run)
  std::vector<char> issued_;                // per position: issued in the current run
  int sidx(int pos) const {                 // compute-stream index of a local F/B position
    if (ktimer_.enabled) return 0;          // kernel timing: everything serial on cs_
    const auto& t = sched.g.tasks[static_cast<size_t>(sched.order[static_cast<size_t>(pos)])];
    return dev_stream_[static_cast<size_t>(t.device)];
  }
  void plan_streams();
  void wait_stage_tasks(int pos, cudaStream_t st);  // st waits for stage's earlier tasks
  int32_t *d_inputs_ = nullptr, *d_labels_ = nullptr;
  float* d_loss_ = nullptr;
  int *d_ver_ = nullptr, *d_trace_ = nullptr;
  std::vector<cudaEvent_t> ev_start_, ev_end_;
  // window machinery's own intervals on the collective / update streams (Reduce, Broadcast);
  // the Timeline shows those tasks where the compute stream passed them (the reference's
  // one-task-at-a-time device model), lane_events their real extent
  std::vector<cudaEvent_t> ev_lstart_, ev_lend_;
  std::vector<char> lane_rec_;
  cudaEvent_t run_begin_ = nullptr, run_end_ = nullptr;
  size_t slot_total_ = 0;
  int64_t measured_alloc_bytes_ = -1;  // cudaMemGetInfo delta across allocate() (-1: plan only)
  std::string memory_json() const;
  bool plan_only_ = false;
  std::vector<float> loss_scale_;  // per minibatch: 1 / number of labelled tokens
  SideStream side_;                // weight-gradient GEMM stream + events

  int rank_of_dev(int dev) const { return dev_rank_[static_cast<size_t>(dev)]; }
  int owner_rank(int stage) const { return rank_of_dev(stage); }
  void make_plan();
  void allocate();
  void init_weights();
  void exec_task(int pos, const int32_t* h_in, const int32_t* h_lab, std::vector<int>& window_tokens_loaded,
                 std::vector<int>& window_last_left, float* losses_out);
  void exec_comm(int pos);
  void zero_broadcast(int stage, int window);

 public:
  std::string comm_export() { return comm_ ? comm_->export_blob() : std::string(); }
  // Use the first n allocated compute streams (1 = the serial executor: isolated per-task
  // times, what the multi-GPU projection needs); recomputes the hazard plan and drops the
  // captured graphs (they encode the previous stream assignment).
  int set_streams(int n) {
    if (plan_only_) return 0;
    active_streams_ = std::max(1, std::min(n, nstreams_));
    CUDA_OK(cudaDeviceSynchronize());
    for (auto& kv : graphs_)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    graphs_.clear();
    plan_streams();
    return active_streams_;
  }
  void comm_connect(const std::vector<std::string>& blobs) {
    if (comm_) comm_->import_blobs(blobs);
  }
};

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
  if (dm.fp32 && dm.recompute) throw std::invalid_argument("engine: fp32 validation mode stores every activation (no recompute)");
  if (dm.h % dm.heads != 0) throw std::invalid_argument("engine: hidden must divide into heads");

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

// An event recorded on `from` now, for an immediate cudaStreamWaitEvent (which binds the
// event's record at call time, so recycling the small pool is safe).
cudaEvent_t Engine::handoff(cudaStream_t from) {
  cudaEvent_t e = ev_pool_[ev_next_++ % ev_pool_.size()];
  CUDA_OK(cudaEventRecord(e, from));
  return e;
}

Engine::~Engine() {
  if (plan_only_) return;
  for (cudaStream_t st : {cs_, rs_, ss_, ks_, us_, side_.side})
    if (st) cudaStreamSynchronize(st);
  comm_.reset();  // unmaps peers' memory before our own buffers go away
  for (auto& [k, g] : graphs_)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  for (auto& s : stages) {
    cudaFree(s->master);
    cudaFree(s->m);
    cudaFree(s->v);
    cudaFree(s->grad);
    cudaFree(s->w);
    cudaFree(s->wt);
  }
  for (size_t i = 0; i < wbuf_.size(); ++i)  // the replica buffer the stage does not point at
    for (int b = 0; b < 2; ++b) {
      if (wbuf_[i][static_cast<size_t>(b)] != stages[i]->w) cudaFree(wbuf_[i][static_cast<size_t>(b)]);
      if (wtbuf_[i][static_cast<size_t>(b)] != stages[i]->wt) cudaFree(wtbuf_[i][static_cast<size_t>(b)]);
    }
  for (auto& v : slot_mem_)
    for (auto* p : v) cudaFree(p);
  for (auto& b : bufs_) {
    if (b.comm_done) cudaEventDestroy(b.comm_done);
    if (b.used) cudaEventDestroy(b.used);
  }
  cudaFree(bounds_arena_);
  cudaFree(ws_);
  cudaFree(d_inputs_);
  cudaFree(d_labels_);
  cudaFree(d_loss_);
  cudaFree(d_ver_);
  cudaFree(d_trace_);
  for (auto e : ev_start_) cudaEventDestroy(e);
  for (auto e : ev_end_) cudaEventDestroy(e);
  for (auto e : ev_lstart_)
    if (e) cudaEventDestroy(e);
  for (auto e : ev_lend_)
    if (e) cudaEventDestroy(e);
  for (auto e : wready_) cudaEventDestroy(e);
  for (auto e : reduced_) cudaEventDestroy(e);
  for (auto& v : seg_ev_)
    for (auto e : v) cudaEventDestroy(e);
  for (auto e : ev_pool_) cudaEventDestroy(e);
  if (run_begin_) cudaEventDestroy(run_begin_);
  if (run_end_) cudaEventDestroy(run_end_);
  for (size_t k = 0; k < sides_.size(); ++k) {  // sides_[0] is side_
    if (sides_[k].side) {
      cudaStreamSynchronize(sides_[k].side);
      for (auto e : sides_[k].ev) cudaEventDestroy(e);
      cudaStreamDestroy(sides_[k].side);
    }
  }
  if (sides_.empty() && side_.side) {
    for (auto e : side_.ev) cudaEventDestroy(e);
    cudaStreamDestroy(side_.side);
  }
  for (size_t k = 1; k < cstreams_.size(); ++k) {
    cudaStreamSynchronize(cstreams_[k]);
    cudaStreamDestroy(cstreams_[k]);
  }
  for (size_t k = 1; k < wss_.size(); ++k) cudaFree(wss_[k]);
  for (auto e : done_) cudaEventDestroy(e);
  if (ss_ && ss_ != rs_) cudaStreamDestroy(ss_);
  if (ks_ && ks_ != rs_) cudaStreamDestroy(ks_);
  if (rs_) cudaStreamDestroy(rs_);
  cudaStreamDestroy(us_);
  cudaStreamDestroy(cs_);
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
}

// `st` waits for every local Forward / Backward of the stage of the window task at `pos` that
// precedes it in the dispatch order (the last one per compute stream): after them nothing
// reads the stage's old weights or adds to its window gradient.
void Engine::wait_stage_tasks(int pos, cudaStream_t st) {
  for (int q : stage_last_[static_cast<size_t>(pos)])
    if (q >= 0 && issued_[static_cast<size_t>(q)]) CUDA_OK(cudaStreamWaitEvent(st, done_[static_cast<size_t>(q)], 0));
}

void Engine::allocate() {
  const size_t T = static_cast<size_t>(dm.T), h = static_cast<size_t>(dm.h);
  wbuf_.assign(static_cast<size_t>(depth_), {nullptr, nullptr});
  wtbuf_.assign(static_cast<size_t>(depth_), {nullptr, nullptr});
  cur_buf_.assign(static_cast<size_t>(depth_), 0);
  rep_buf_.assign(static_cast<size_t>(depth_), std::vector<int>(static_cast<size_t>(P_), 0));
  for (int i = 0; i < depth_; ++i) {
    if (!hosted[static_cast<size_t>(i)]) continue;
    GptStage& st = *stages[static_cast<size_t>(i)];
    const size_t n = static_cast<size_t>(st.numel());
    CUDA_OK(cudaMalloc(&st.master, n * sizeof(float)));
    CUDA_OK(cudaMalloc(&st.grad, n * sizeof(float)));
    CUDA_OK(cudaMalloc(&st.w, n * sizeof(uint16_t)));
    CUDA_OK(cudaMalloc(&st.wt, n * sizeof(uint16_t)));
    CUDA_OK(cudaMemsetAsync(st.grad, 0, n * sizeof(float), cs_));
    if (versioned_) {
      auto& wb = wbuf_[static_cast<size_t>(i)];
      auto& wtb = wtbuf_[static_cast<size_t>(i)];
      wb[0] = st.w;
      wtb[0] = st.wt;
      CUDA_OK(cudaMalloc(&wb[1], n * sizeof(uint16_t)));
      CUDA_OK(cudaMalloc(&wtb[1], n * sizeof(uint16_t)));
    }
    if (owned[static_cast<size_t>(i)]) {  // the optimizer state this rank keeps (its shard under ZeRO)
      const size_t no = static_cast<size_t>(std::max<int64_t>(opt_numel_[static_cast<size_t>(i)], 64));
      CUDA_OK(cudaMalloc(&st.m, no * sizeof(float)));
      CUDA_OK(cudaMalloc(&st.v, no * sizeof(float)));
      CUDA_OK(cudaMemsetAsync(st.m, 0, no * sizeof(float), cs_));
      CUDA_OK(cudaMemsetAsync(st.v, 0, no * sizeof(float), cs_));
    }
  }
  slot_mem_.assign(static_cast<size_t>(depth_), {});
  slot_acts_.assign(static_cast<size_t>(depth_), {});
  for (int i = 0; i < depth_; ++i) {
    const size_t bytes = stages[static_cast<size_t>(i)]->slot_bytes();
    for (int s = 0; s < slots_per_stage[static_cast<size_t>(i)]; ++s) {
      uint8_t* p = nullptr;
      CUDA_OK(cudaMalloc(&p, bytes));
      slot_total_ += bytes;
      slot_mem_[static_cast<size_t>(i)].push_back(p);
      slot_acts_[static_cast<size_t>(i)].push_back(stages[static_cast<size_t>(i)]->carve_slot(p));
    }
  }
  // boundary buffers: one arena (one IPC export), buffer b at b * T * h elements
  bufs_.resize(static_cast<size_t>(nbuf));
  const size_t ab = dm.act_bytes();
  if (nbuf > 0) CUDA_OK(cudaMalloc(&bounds_arena_, static_cast<size_t>(nbuf) * T * h * ab));
  for (size_t k = 0; k < bufs_.size(); ++k) {
    BoundaryBuf& b = bufs_[k];
    b.ptr = bounds_arena_ + k * T * h * (ab / 2);
    CUDA_OK(cudaEventCreateWithFlags(&b.comm_done, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&b.used, cudaEventDisableTiming));
  }
  CUDA_OK(cudaMalloc(&ws_, GptStage::workspace_bytes(dm)));
  CUDA_OK(cudaMalloc(&d_inputs_, static_cast<size_t>(M_) * T * sizeof(int32_t)));
  CUDA_OK(cudaMalloc(&d_labels_, static_cast<size_t>(M_) * T * sizeof(int32_t)));
  CUDA_OK(cudaMalloc(&d_loss_, static_cast<size_t>(M_) * sizeof(float)));
  CUDA_OK(cudaMalloc(&d_ver_, static_cast<size_t>(depth_ * P_) * sizeof(int)));
  CUDA_OK(cudaMalloc(&d_trace_, sched.g.tasks.size() * sizeof(int)));
  wready_.resize(static_cast<size_t>(depth_));
  reduced_.resize(static_cast<size_t>(depth_));
  wpending_.assign(static_cast<size_t>(depth_), 0);
  fpending_.assign(static_cast<size_t>(depth_), 0);
  pending_ag_.assign(static_cast<size_t>(depth_), -1);
  segs_.resize(static_cast<size_t>(depth_));
  seg_ev_.resize(static_cast<size_t>(depth_));
  for (int i = 0; i < depth_; ++i) {
    segs_[static_cast<size_t>(i)] = stages[static_cast<size_t>(i)]->segments();
    for (size_t k = 0; k < segs_[static_cast<size_t>(i)].size(); ++k) {
      cudaEvent_t e;
      CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      seg_ev_[static_cast<size_t>(i)].push_back(e);
    }
  }
  for (auto& e : wready_) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : reduced_) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (comm_) {  // what peers may read: boundary arena, and per hosted stage grad / w / master
    if (bounds_arena_) comm_->register_region(REG_BOUNDS, 0, bounds_arena_, static_cast<size_t>(nbuf) * T * h * ab);
    for (const auto& [msg, b] : planned_sends_) comm_->plan_send(msg, static_cast<size_t>(b) * T * h * ab);
    for (int i = 0; i < depth_; ++i) {
      if (!hosted[static_cast<size_t>(i)] || group_ranks_[static_cast<size_t>(i)].size() < 2) continue;
      GptStage& st = *stages[static_cast<size_t>(i)];
      const size_t n = static_cast<size_t>(st.numel());
      comm_->register_region(REG_GRAD, i, st.grad, n * 4);
      comm_->register_region(REG_MASTER, i, st.master, n * 4);
      comm_->register_region(REG_W, i, st.w, n * 2);
    }
  }
  CUDA_OK(cudaEventCreate(&run_begin_));
  CUDA_OK(cudaEventCreate(&run_end_));
  // concurrent compute streams: as many as this rank's logical devices (ZeRO AMDP; the NCCL
  // backend keeps one), within what the extra workspaces leave of HBM (a 6 GiB margin);
  // AMDP_STREAMS overrides the count
  cstreams_.assign(1, cs_);
  sides_.assign(1, side_);
  wss_.assign(1, ws_);
  nstreams_ = 1;
  int local_devices = 0;
  for (int d = 0; d < devices_; ++d) local_devices += rank_of_dev(d) == rank_ ? 1 : 0;
  const bool nccl = comm_ && comm_->single_stream();  // NCCL: one stream for all its ops
  if (zero_ && local_devices > 1 && !nccl && !getenv("AMDP_SINGLE_STREAM")) {
    size_t fr = 0, tot = 0;
    CUDA_OK(cudaMemGetInfo(&fr, &tot));
    const size_t wsb = GptStage::workspace_bytes(dm);
    int want = getenv("AMDP_STREAMS") ? std::max(1, atoi(getenv("AMDP_STREAMS"))) : local_devices;
    want = std::min(want, local_devices);
    while (want > 1 && static_cast<size_t>(want - 1) * wsb + (6ull << 30) > fr) --want;
    for (int k = 1; k < want; ++k) {
      cudaStream_t st;
      CUDA_OK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      cstreams_.push_back(st);
      SideStream sd;
      if (side_.side) {
        CUDA_OK(cudaStreamCreateWithFlags(&sd.side, cudaStreamNonBlocking));
        for (auto& e : sd.ev) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      }
      sides_.push_back(sd);
      uint8_t* w = nullptr;
      CUDA_OK(cudaMalloc(&w, wsb));
      wss_.push_back(w);
    }
    nstreams_ = want;
  }
  wpending_.assign(static_cast<size_t>(depth_ * nstreams_), 0);
  fpending_.assign(static_cast<size_t>(depth_ * nstreams_), 0);
  active_streams_ = nstreams_;
  plan_streams();
}

void Engine::init_weights() {
  for (int i = 0; i < depth_; ++i) {
    if (!hosted[static_cast<size_t>(i)]) continue;
    GptStage& st = *stages[static_cast<size_t>(i)];
    CUDA_OK(cudaMemsetAsync(st.master, 0, static_cast<size_t>(st.numel()) * sizeof(float), cs_));
    for (const auto& p : st.params()) {
      float* dst = st.master + p.off;
      int rc = 0;
      if (p.init == 0)
        rc = amdp_fill_normal_bf16_f32(nullptr, dst, p.numel(), tensor_seed(mc_.seed, p.global_index), p.std,
                                       reinterpret_cast<amdp_stream_t>(cs_));
      else
        rc = amdp_fill_const_f32(dst, p.numel(), p.init == 1 ? 1.0f : 0.0f, reinterpret_cast<amdp_stream_t>(cs_));
      if (rc != 0) throw std::runtime_error("weight init failed");
    }
    const int64_t n = st.numel();
    cast_f32_bf16_kernel<<<std::min<int64_t>((n + 255) / 256, 4 * 148), 256, 0, cs_>>>(
        st.master, reinterpret_cast<bf16*>(st.w), n);
    CUDA_OK(cudaGetLastError());
    if (st.refresh_transposed(cs_) < 0) throw std::runtime_error("weight transpose failed");
  }
  CUDA_OK(cudaStreamSynchronize(cs_));
}

// Point-to-point ops placed at order position `pos`, and the Reduce of a window.  Sends run
// on the send stream after this position's compute; a receive waits only for the last
// compute use of its destination buffer (not for all earlier compute of the rank).
void Engine::exec_comm(int pos) {
  for (const CommOp& op : comm_at_[static_cast<size_t>(pos)]) {
    const size_t bytes = static_cast<size_t>(dm.T) * static_cast<size_t>(dm.h) * dm.act_bytes();
    switch (op.kind) {
      case CommOp::Send: {
        BoundaryBuf& b = bufs_[static_cast<size_t>(op.buf)];
        // after the producing task (this position) on its compute stream
        CUDA_OK(cudaStreamWaitEvent(ss_, issued_[static_cast<size_t>(pos)] ? done_[static_cast<size_t>(pos)] : handoff(cs_), 0));
        comm_->send(op.id, op.peer, b.ptr, bytes, ss_);
        CUDA_OK(cudaEventRecord(b.comm_done, ss_));
        b.comm_pending = true;
        stats.p2p_bytes_sent += static_cast<int64_t>(bytes);
        break;
      }
      case CommOp::Recv: {
        BoundaryBuf& b = bufs_[static_cast<size_t>(op.buf)];
        if (b.use_recorded) CUDA_OK(cudaStreamWaitEvent(rs_, b.used, 0));
        if (b.comm_pending) CUDA_OK(cudaStreamWaitEvent(rs_, b.comm_done, 0));  // NCCL: same stream
        comm_->recv(op.id, op.peer, b.ptr, bytes, rs_);
        CUDA_OK(cudaEventRecord(b.comm_done, rs_));
        b.comm_pending = true;
        break;
      }
      case CommOp::Reduce: {
        GptStage& st = *stages[static_cast<size_t>(op.stage)];
        wait_stage_tasks(pos, ks_);  // the window's backwards of this stage on this rank
        // ZeRO within the group: member j ends with the group's sum over its shard
        comm_->reduce_scatter_f32(op.id, group_ranks_[static_cast<size_t>(op.stage)], op.stage, st.grad,
                                  shard_[static_cast<size_t>(op.stage)], ks_);
        CUDA_OK(cudaEventRecord(reduced_[static_cast<size_t>(op.stage)], ks_));
        stats.collective_bytes += st.numel() * 4;
        break;
      }
      case CommOp::Bcast:
      case CommOp::Allreduce:
        break;  // issued from exec_task (ordered with the optimizer step)
    }
  }
}

// ZeRO Broadcast(w, i) (H/builder.hpp:289-304) on the update stream, after this rank's compute
// up to this order position (every read of the old weights and, through reduced_, the
// reduced window gradient): the owner steps the optimizer (bf16 copy + transposed copy
// rewritten, gradient zeroed); replicas on other ranks clear their gradient and pull the
// owner's bf16 weights + fp32 LayerNorm parameters, then refresh their transposed copy.
// The next F/B of stage i waits for wready_[i]; nothing else does.
void Engine::zero_broadcast(int i, int window) {
  GptStage& S = *stages[static_cast<size_t>(i)];
  const auto& gr = group_ranks_[static_cast<size_t>(i)];
  const bool multi = sharded(i);
  wait_stage_tasks(cur_pos_, us_);  // every earlier reader of the old weights / window gradient
  if (multi) CUDA_OK(cudaStreamWaitEvent(us_, reduced_[static_cast<size_t>(i)], 0));
  // every replica of stage i reads the next version from its next task on (those wait for
  // this stream's segment events / wready_, recorded after this bump)
  bump_version_kernel<<<1, 1, 0, us_>>>(d_ver_, i * P_, P_);
  stats.kernels_launched += 1;
  // the update stream's interval of this Broadcast (a lane event: it overlaps other stages'
  // compute on this GPU; projection.py models the update lane separately)
  if (rc_.record_events) {
    rec(ev_lstart_[static_cast<size_t>(cur_pos_)], us_);
    lane_rec_[static_cast<size_t>(cur_pos_)] = 1;
  }
  const auto& segs = segs_[static_cast<size_t>(i)];
  if (!multi) {
    // every replica of stage i is on this GPU (they share one set of buffers): the owner
    // steps segment by segment in the forward's reading order (embeddings, layers, head), so
    // a gated Forward starts on its first layer while later layers are still being stepped
    for (size_t k = 0; k < segs.size(); ++k) {
      optimizer_range(i, window + 1, segs[k].first, segs[k].second, us_);
      CUDA_OK(cudaEventRecord(seg_ev_[static_cast<size_t>(i)][k], us_));
    }
  } else {
    // ZeRO within the replica group: after the reduce-scatter (collective stream) each member
    // steps its shard of every segment and the group all-gathers the bf16 weights + fp32
    // LayerNorm parameters (fp32 validation mode: the fp32 master), segment by segment.
    // NCCL: the collectives of one communicator share its stream, so this runs there.
    int coll0 = -1;
    for (const CommOp& op : comm_at_[static_cast<size_t>(cur_pos_)])
      if (op.kind == CommOp::Bcast && op.stage == i) coll0 = op.id;
    cudaStream_t st = comm_->single_stream() ? ks_ : us_;
    if (st != us_) CUDA_OK(cudaStreamWaitEvent(st, handoff(us_), 0));
    // the previous window's gather of these weights must be complete everywhere before the
    // optimizer overwrites this rank's shard
    if (pending_ag_[static_cast<size_t>(i)] >= 0) {
      for (size_t k = 0; k < segs.size(); ++k)
        comm_->allgather_wait(pending_ag_[static_cast<size_t>(i)] + static_cast<int>(k), gr, st);
      pending_ag_[static_cast<size_t>(i)] = -1;
    }
    const auto& sh = shard_[static_cast<size_t>(i)];
    const int me = member(i);
    int64_t moved = 0;
    for (size_t k = 0; k < segs.size(); ++k) {
      const auto [lo, hi] = sh[static_cast<size_t>(me)][k];
      if (hi > lo)
        optimizer_range(i, window + 1, static_cast<int64_t>(lo), static_cast<int64_t>(hi - lo), st,
                        opt_off_[static_cast<size_t>(i)][k]);
      std::vector<std::vector<Span>> spans(gr.size());
      for (size_t j = 0; j < gr.size(); ++j) {
        const auto [a, b] = sh[j][k];
        if (b <= a) continue;
        if (dm.fp32) {  // fp32 validation mode: the kernels read the fp32 master itself
          spans[j].push_back(Span{REG_MASTER, i, a * 4, (b - a) * 4});
        } else {  // bf16 working weights + the fp32 LayerNorm parameters the kernels read
          spans[j].push_back(Span{REG_W, i, a * 2, (b - a) * 2});
          for (const auto& p : S.params()) {
            const size_t p0 = static_cast<size_t>(p.off), p1 = p0 + static_cast<size_t>(p.numel());
            if (p.rows == 1 && p1 > a && p0 < b)
              spans[j].push_back(Span{REG_MASTER, i, std::max(p0, a) * 4, (std::min(p1, b) - std::max(p0, a)) * 4});
          }
        }
        if (j != static_cast<size_t>(me))
          for (const Span& sp : spans[j]) moved += static_cast<int64_t>(sp.bytes);
      }
      comm_->allgather(coll0 + static_cast<int>(k), gr, i, spans, st);
      CUDA_OK(cudaEventRecord(seg_ev_[static_cast<size_t>(i)][k], st));
    }
    pending_ag_[static_cast<size_t>(i)] = coll0;
    stats.collective_bytes += moved;
    // the optimizer zeroed this rank's shard of the window gradient; the rest was consumed by
    // the reduce-scatter
    CUDA_OK(cudaMemsetAsync(S.grad, 0, static_cast<size_t>(S.numel()) * sizeof(float), st));
    if (st != us_) CUDA_OK(cudaStreamWaitEvent(us_, handoff(st), 0));
  }
  const int nt = S.refresh_transposed(us_);  // the backward's K-major weight copies
  if (nt < 0) throw std::runtime_error("weight transpose failed");
  stats.kernels_launched += nt;
  CUDA_OK(cudaEventRecord(wready_[static_cast<size_t>(i)], us_));
  if (rc_.record_events) rec(ev_lend_[static_cast<size_t>(cur_pos_)], us_);
  for (int k = 0; k < nstreams_; ++k) {  // the first F / B of the stage on each compute stream waits
    wpending_[static_cast<size_t>(i * nstreams_ + k)] = 1;
    fpending_[static_cast<size_t>(i * nstreams_ + k)] = 1;
  }
}

void Engine::exec_task(int pos, const int32_t* h_in, const int32_t* h_lab, std::vector<int>& loaded,
                       std::vector<int>& last_left, float* losses_out) {
  const auto& g = sched.g;
  const int t = sched.order[static_cast<size_t>(pos)];
  const auto& task = g.tasks[static_cast<size_t>(t)];
  const TaskPlan& tp = plan_[static_cast<size_t>(pos)];
  const size_t T = static_cast<size_t>(dm.T);
  int rc = 0;
  cur_pos_ = pos;

  if (task.kind == ppsim::Kind::Forward || task.kind == ppsim::Kind::Backward) {
    if (!tp.local) {
      exec_comm(pos);
      return;
    }
    const int i = task.stage, j = task.minibatch;
    GptStage& S = *stages[static_cast<size_t>(i)];
    const SlotActs& A = slot_acts_[static_cast<size_t>(i)][static_cast<size_t>(tp.slot)];
    const int w = j / thr_;
    const int si = sidx(pos);
    cudaStream_t cs = cstreams_[static_cast<size_t>(si)];  // this task's compute stream
    for (int q : waits_[static_cast<size_t>(pos)])      // hazards with other compute streams
      if (issued_[static_cast<size_t>(q)]) CUDA_OK(cudaStreamWaitEvent(cs, done_[static_cast<size_t>(q)], 0));
    if (task.kind == ppsim::Kind::Forward && !loaded[static_cast<size_t>(w)]) {
      const size_t off = static_cast<size_t>(w) * thr_ * T;
      CUDA_OK(cudaMemcpyAsync(d_inputs_ + off, h_in + off, thr_ * T * sizeof(int32_t), cudaMemcpyHostToDevice, cs));
      CUDA_OK(cudaMemcpyAsync(d_labels_ + off, h_lab + off, thr_ * T * sizeof(int32_t), cudaMemcpyHostToDevice, cs));
      stats.h2d_bytes += static_cast<int64_t>(2 * thr_ * T * sizeof(int32_t));
      loaded[static_cast<size_t>(w)] = 1;
      tok_loader_[static_cast<size_t>(w)] = pos;
    } else if (task.kind == ppsim::Kind::Forward && (S.first() || S.last()) && tok_loader_[static_cast<size_t>(w)] >= 0 &&
               sidx(tok_loader_[static_cast<size_t>(w)]) != si) {  // tokens copied on another stream
      CUDA_OK(cudaStreamWaitEvent(cs, done_[static_cast<size_t>(tok_loader_[static_cast<size_t>(w)])], 0));
    }
    auto wait_buf = [&](int b) {
      if (b >= 0 && bufs_[static_cast<size_t>(b)].comm_pending) {
        CUDA_OK(cudaStreamWaitEvent(cs, bufs_[static_cast<size_t>(b)].comm_done, 0));
      }
    };
    wait_buf(tp.in_buf);
    wait_buf(tp.gin_buf);
    wait_buf(tp.out_buf);
    wait_buf(tp.gout_buf);
    // the stage's new weights (Broadcast on the update stream): a Forward waits segment by
    // segment inside its body, a Backward (transposed copies, cleared gradient) for all of it
    const cudaEvent_t* seg_wait = nullptr;
    const size_t pk = static_cast<size_t>(i * nstreams_ + si);  // (stage, compute stream)
    if (task.kind == ppsim::Kind::Forward && fpending_[pk]) {
      seg_wait = seg_ev_[static_cast<size_t>(i)].data();
      fpending_[pk] = 0;
    } else if (task.kind == ppsim::Kind::Backward && wpending_[pk]) {
      CUDA_OK(cudaStreamWaitEvent(cs, wready_[static_cast<size_t>(i)], 0));
      wpending_[pk] = fpending_[pk] = 0;
    }
    // the version this task reads: after the Broadcast's counter bump, which precedes its first
    // segment event (the body then waits for the later segments as it reaches them)
    if (seg_wait) CUDA_OK(cudaStreamWaitEvent(cs, seg_wait[0], 0));
    if (rc_.record_events) rec(ev_start_[static_cast<size_t>(pos)], cs);
    record_version_kernel<<<1, 1, 0, cs>>>(d_ver_, i * P_ + task.pipeline, d_trace_, t);
    use_replica_weights(i, task.pipeline);
    stats.kernels_launched += 1;
    const int32_t* tok = d_inputs_ + static_cast<size_t>(j) * T;
    const int32_t* lab = d_labels_ + static_cast<size_t>(j) * T;
    const uint16_t* in = tp.in_buf >= 0 ? bufs_[static_cast<size_t>(tp.in_buf)].ptr : nullptr;
    int launched;
    if (task.kind == ppsim::Kind::Forward) {
      uint16_t* out = tp.out_buf >= 0 ? bufs_[static_cast<size_t>(tp.out_buf)].ptr : nullptr;
      launched = S.forward(A, tok, lab, in, out, d_loss_ + j, loss_scale_[static_cast<size_t>(j)],
                           wss_[static_cast<size_t>(si)], cs, &rc, seg_wait);
    } else {
      const uint16_t* gin = tp.gin_buf >= 0 ? bufs_[static_cast<size_t>(tp.gin_buf)].ptr : nullptr;
      uint16_t* gout = tp.gout_buf >= 0 ? bufs_[static_cast<size_t>(tp.gout_buf)].ptr : nullptr;
      // the kernel-timing run serialises the streams so per-launch event spans are exact
      launched = S.backward(A, tok, in, gin, gout, wss_[static_cast<size_t>(si)], cs,
                            ktimer_.enabled ? SideStream{} : sides_[static_cast<size_t>(si)], &rc);
    }
    stats.kernels_launched += launched;
    if (rc != 0) throw std::runtime_error("stage kernel failed with code " + std::to_string(rc));
    if (rc_.record_events) rec(ev_end_[static_cast<size_t>(pos)], cs);
    CUDA_OK(cudaEventRecord(done_[static_cast<size_t>(pos)], cs));
    issued_[static_cast<size_t>(pos)] = 1;
    stats.tasks_executed += 1;
    if (comm_) {  // last compute use of the buffers this task touched (a later recv waits for it)
      for (int b : {tp.in_buf, tp.gin_buf, tp.out_buf, tp.gout_buf})
        if (b >= 0) {
          CUDA_OK(cudaEventRecord(bufs_[static_cast<size_t>(b)].used, cs));
          bufs_[static_cast<size_t>(b)].use_recorded = true;
        }
    }
    exec_comm(pos);  // sends of this task's output, recvs placed at this position
    // D2H of a window's losses once its last-stage forwards are all issued
    if (task.kind == ppsim::Kind::Forward && S.last() && losses_out) {
      if (--last_left[static_cast<size_t>(w)] == 0) {
        for (int q : loss_tasks_[static_cast<size_t>(w)])  // the window's other last-stage forwards
          if (q != pos && issued_[static_cast<size_t>(q)] && sidx(q) != si)
            CUDA_OK(cudaStreamWaitEvent(cs, done_[static_cast<size_t>(q)], 0));
        CUDA_OK(cudaMemcpyAsync(losses_out + static_cast<size_t>(w) * thr_, d_loss_ + static_cast<size_t>(w) * thr_,
                                thr_ * sizeof(float), cudaMemcpyDeviceToHost, cs));
        stats.d2h_bytes += thr_ * static_cast<int64_t>(sizeof(float));
      }
    }
    return;
  }

  // window machinery
  const int i = task.stage;
  if (!hosted[static_cast<size_t>(i)]) {
    exec_comm(pos);
    return;
  }
  GptStage& S = *stages[static_cast<size_t>(i)];
  // the marker events of a window task: where its logical device's compute stream passed it
  cudaStream_t ms = cstreams_[ktimer_.enabled ? 0 : static_cast<size_t>(dev_stream_[static_cast<size_t>(task.device)])];
  if (task.kind == ppsim::Kind::Reduce) {
    // the reduction runs on the collective stream (its measured interval); the update stream's
    // Broadcast waits for it
    const bool lane = !comm_at_[static_cast<size_t>(pos)].empty();
    if (rc_.record_events) rec(ev_start_[static_cast<size_t>(pos)], ms);
    if (rc_.record_events && lane) {
      wait_stage_tasks(pos, ks_);
      rec(ev_lstart_[static_cast<size_t>(pos)], ks_);
      lane_rec_[static_cast<size_t>(pos)] = 1;
    }
    exec_comm(pos);
    if (rc_.record_events && lane) rec(ev_lend_[static_cast<size_t>(pos)], ks_);
    if (rc_.record_events) rec(ev_end_[static_cast<size_t>(pos)], ms);
    stats.tasks_executed += 1;
    return;
  }
  if (task.kind == ppsim::Kind::Update) {  // replicated update (every schedule but ZeRO AMDP)
    if (rc_.record_events) rec(ev_start_[static_cast<size_t>(pos)], ms);
    if (tp.first_update) {
      if (group_ranks_[static_cast<size_t>(i)].size() > 1) {  // sum the replicas' window gradients
        int coll = -1;
        for (const CommOp& op : comm_at_[static_cast<size_t>(pos)])
          if (op.kind == CommOp::Allreduce && op.stage == i) coll = op.id;
        CUDA_OK(cudaStreamWaitEvent(ks_, handoff(cs_), 0));
        comm_->allreduce_f32(coll, group_ranks_[static_cast<size_t>(i)], i, S.grad, static_cast<size_t>(S.numel()),
                             ks_);
        stats.collective_bytes += 2 * S.numel() * 4;
        CUDA_OK(cudaStreamWaitEvent(cs_, handoff(ks_), 0));
      }
      optimizer_step(i, task.minibatch + 1, cs_);  // Update's minibatch field: window (PipeDream: j)
    }
    if (rank_of_dev(task.device) == rank_) {  // this replica now reads the newest weights
      if (versioned_) rep_buf_[static_cast<size_t>(i)][static_cast<size_t>(task.pipeline)] = cur_buf_[static_cast<size_t>(i)];
      bump_version_kernel<<<1, 1, 0, cs_>>>(d_ver_, i * P_ + task.pipeline, 1);
      stats.kernels_launched += 1;
    }
    if (rc_.record_events) rec(ev_end_[static_cast<size_t>(pos)], ms);
    stats.tasks_executed += 1;
    return;
  }
  if (task.kind == ppsim::Kind::Broadcast) {
    if (rc_.record_events) rec(ev_start_[static_cast<size_t>(pos)], ms);
    zero_broadcast(i, task.minibatch);  // Broadcast's minibatch field: the window
    if (rc_.record_events) rec(ev_end_[static_cast<size_t>(pos)], ms);
    stats.tasks_executed += 1;
    return;
  }
  exec_comm(pos);
}

void Engine::stage_tokens(const int32_t* h_in, const int32_t* h_lab) {
  const size_t n = static_cast<size_t>(M_) * static_cast<size_t>(dm.T) * sizeof(int32_t);
  CUDA_OK(cudaMemcpy(d_inputs_, h_in, n, cudaMemcpyHostToDevice));
  CUDA_OK(cudaMemcpy(d_labels_, h_lab, n, cudaMemcpyHostToDevice));
}

// Everything a run puts on the GPU, in the global dispatch order (eager, or under capture).
void Engine::issue(int max_window, bool resident, const int32_t* h_in, const int32_t* h_lab, float* losses_out) {
  const int N = static_cast<int>(sched.order.size());
  const auto& g = sched.g;
  if (done_.empty()) {
    done_.resize(static_cast<size_t>(N));
    for (auto& e : done_) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  issued_.assign(static_cast<size_t>(N), 0);
  tok_loader_.assign(static_cast<size_t>(W_), -1);
  CUDA_OK(cudaMemsetAsync(d_ver_, 0, static_cast<size_t>(depth_ * P_) * sizeof(int), cs_));
  CUDA_OK(cudaMemsetAsync(d_loss_, 0, static_cast<size_t>(M_) * sizeof(float), cs_));
  CUDA_OK(cudaMemsetAsync(d_trace_, 0xff, g.tasks.size() * sizeof(int), cs_));
  std::vector<int> loaded(static_cast<size_t>(W_), resident ? 1 : 0), last_left(static_cast<size_t>(W_), 0);
  for (int k = 0; k < N; ++k) {
    const auto& t = g.tasks[static_cast<size_t>(sched.order[static_cast<size_t>(k)])];
    if (t.kind == ppsim::Kind::Forward && t.stage == depth_ - 1 && plan_[static_cast<size_t>(k)].local)
      ++last_left[static_cast<size_t>(t.window)];
  }
  for (auto& b : bufs_) b.comm_pending = b.use_recorded = false;  // the previous run fully drained
  lane_rec_.assign(static_cast<size_t>(N), 0);
  std::fill(wpending_.begin(), wpending_.end(), 0);
  std::fill(fpending_.begin(), fpending_.end(), 0);
  rec(run_begin_, cs_);
  {  // every other stream starts after the run's initialisation (counters, losses, trace)
    const cudaEvent_t e = handoff(cs_);
    CUDA_OK(cudaStreamWaitEvent(us_, e, 0));
    for (size_t k = 1; k < cstreams_.size(); ++k) CUDA_OK(cudaStreamWaitEvent(cstreams_[k], e, 0));
  }
  for (int k = 0; k < N; ++k)
    if (g.tasks[static_cast<size_t>(sched.order[static_cast<size_t>(k)])].window < max_window)
      exec_task(k, h_in, h_lab, loaded, last_left, losses_out);
  for (int i = 0; i < depth_; ++i)  // the last window's gathers have completed everywhere
    if (pending_ag_[static_cast<size_t>(i)] >= 0) {
      cudaStream_t st = comm_ && comm_->single_stream() ? ks_ : us_;
      for (size_t k = 0; k < segs_[static_cast<size_t>(i)].size(); ++k)
        comm_->allgather_wait(pending_ag_[static_cast<size_t>(i)] + static_cast<int>(k), group_ranks_[static_cast<size_t>(i)],
                              st);
      pending_ag_[static_cast<size_t>(i)] = -1;
    }
  for (cudaStream_t st : {rs_, ss_, ks_, us_})  // join every stream: the run ends when all are idle
    if (st) CUDA_OK(cudaStreamWaitEvent(cs_, handoff(st), 0));
  for (size_t k = 1; k < cstreams_.size(); ++k) CUDA_OK(cudaStreamWaitEvent(cs_, handoff(cstreams_[k]), 0));
  rec(run_end_, cs_);
}

void Engine::run(const int32_t* h_in, const int32_t* h_lab, float* losses_out, int max_window, bool resident) {
  const int N = static_cast<int>(sched.order.size());
  const auto& g = sched.g;
  if (max_window < 0 || max_window > W_) max_window = W_;
  stats = amdp_run_stats{};
  // loss = mean over the minibatch's labelled tokens (all of them for GPT; the masked
  // positions for MLM), so the CE gradient and the reported loss use 1 / count
  loss_scale_.assign(static_cast<size_t>(M_), 1.f / static_cast<float>(dm.T));
  if (h_lab)
    for (int j = 0; j < M_; ++j) {
      int64_t cnt = 0;
      const int32_t* lj = h_lab + static_cast<size_t>(j) * dm.T;
      for (int t = 0; t < dm.T; ++t) cnt += lj[t] >= 0;
      loss_scale_[static_cast<size_t>(j)] = 1.f / static_cast<float>(cnt > 0 ? cnt : 1);
    }
  ktimer_.reset();
  if (rc_.record_events && ev_start_.empty()) {
    ev_start_.resize(static_cast<size_t>(N));
    ev_end_.resize(static_cast<size_t>(N));
    ev_lstart_.assign(static_cast<size_t>(N), nullptr);
    ev_lend_.assign(static_cast<size_t>(N), nullptr);
    for (int k = 0; k < N; ++k) {
      CUDA_OK(cudaEventCreate(&ev_start_[static_cast<size_t>(k)]));
      CUDA_OK(cudaEventCreate(&ev_end_[static_cast<size_t>(k)]));
      const auto kind = g.tasks[static_cast<size_t>(sched.order[static_cast<size_t>(k)])].kind;
      if (kind == ppsim::Kind::Reduce || kind == ppsim::Kind::Broadcast) {
        CUDA_OK(cudaEventCreate(&ev_lstart_[static_cast<size_t>(k)]));
        CUDA_OK(cudaEventCreate(&ev_lend_[static_cast<size_t>(k)]));
      }
    }
  }
  if (comm_) {
    if (!comm_->connected())
      throw std::runtime_error("engine: world_size > 1 needs the communication descriptors exchanged "
                               "(amdp_engine_comm_export / amdp_engine_comm_connect) before run");
    comm_->begin_run();
  }
  // CUDA graph of the whole run: one GPU (peer flags carry a per-run epoch), no kernel timing,
  // no replica weight versions (their buffer rotation is host state), pinned host buffers
  auto pinned = [](const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  };
  const bool can_graph = graphs_enabled_ && !comm_ && !ktimer_.enabled && !versioned_ &&
                         (resident || (pinned(h_in) && pinned(h_lab))) && (!losses_out || pinned(losses_out));
  uint64_t sh = 1469598103934665603ull;
  for (float f : loss_scale_) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    sh = (sh ^ u) * 1099511628211ull;
  }
  const GraphKey key{max_window, resident, h_in, h_lab, losses_out, sh};
  const auto t_issue0 = std::chrono::steady_clock::now();
  auto it = can_graph ? graphs_.find(key) : graphs_.end();
  if (it != graphs_.end()) {  // replay
    CUDA_OK(cudaGraphLaunch(it->second.exec, cs_));
    stats = it->second.stats;
    lane_rec_ = it->second.lane_rec;
    stats.graph_replayed = 1;
  } else if (can_graph && eager_runs_ >= 1) {  // a new configuration after an eager run (which did
                                                 // every lazy initialisation): capture
    capturing_ = true;
    cudaGraph_t graph = nullptr;
    try {
      CUDA_OK(cudaStreamBeginCapture(cs_, cudaStreamCaptureModeRelaxed));
      const cudaEvent_t e0 = handoff(cs_);  // pull the other streams into the capture
      CUDA_OK(cudaStreamWaitEvent(us_, e0, 0));
      for (size_t k = 0; k < cstreams_.size(); ++k) {
        if (k) CUDA_OK(cudaStreamWaitEvent(cstreams_[k], e0, 0));
        // the stage bodies wait on side-stream events recorded by the previous task; a wait on
        // a record from outside the capture would invalidate it, so re-record them inside
        if (sides_[k].side) {
          CUDA_OK(cudaStreamWaitEvent(sides_[k].side, e0, 0));
          for (cudaEvent_t e : sides_[k].ev) CUDA_OK(cudaEventRecord(e, sides_[k].side));
        }
      }
      issue(max_window, resident, h_in, h_lab, losses_out);
      CUDA_OK(cudaStreamEndCapture(cs_, &graph));
      capturing_ = false;
      GraphRun gr;
      CUDA_OK(cudaGraphInstantiate(&gr.exec, graph, 0));
      cudaGraphDestroy(graph);
      gr.stats = stats;
      gr.lane_rec = lane_rec_;
      CUDA_OK(cudaGraphLaunch(gr.exec, cs_));
      graphs_[key] = gr;
      stats.graph_replayed = 1;
    } catch (const std::exception& ex) {  // not capturable here: abandon graphs, run eagerly
      graph_error_ = ex.what();
      if (getenv("AMDP_GRAPH_DEBUG")) fprintf(stderr, "amdp: CUDA graph capture failed: %s\n", ex.what());
      cudaStreamCaptureStatus cs;
      if (cudaStreamIsCapturing(cs_, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
        cudaGraph_t g2 = nullptr;
        cudaStreamEndCapture(cs_, &g2);
        if (g2) cudaGraphDestroy(g2);
      }
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      capturing_ = false;
      graphs_enabled_ = false;
      stats = amdp_run_stats{};
      issue(max_window, resident, h_in, h_lab, losses_out);
    }
  } else {
    issue(max_window, resident, h_in, h_lab, losses_out);
    ++eager_runs_;
  }
  stats.host_issue_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_issue0).count();
  CUDA_OK(cudaStreamSynchronize(cs_));
  if (comm_) {
    stats.kernels_launched += comm_->kernel_launches() - comm_launches_seen_;
    comm_launches_seen_ = comm_->kernel_launches();
  }
  float ms = 0.f;
  CUDA_OK(cudaEventElapsedTime(&ms, run_begin_, run_end_));
  stats.device_ms = ms;
  ktimer_.collect();
  if (losses_out)
    for (int j = 0; j < max_window * thr_; ++j) losses_out[j] *= loss_scale_[static_cast<size_t>(j)];

  // measured timeline + observed versions
  std::vector<int> trace(g.tasks.size());
  CUDA_OK(cudaMemcpy(trace.data(), d_trace_, trace.size() * sizeof(int), cudaMemcpyDeviceToHost));
  version_seen = trace;
  events.clear();
  lane_events.clear();
  double busy = 0;
  if (rc_.record_events) {
    for (int k = 0; k < N; ++k) {
      const TaskPlan& tp = plan_[static_cast<size_t>(k)];
      const auto& t = g.tasks[static_cast<size_t>(sched.order[static_cast<size_t>(k)])];
      const bool fb = t.kind == ppsim::Kind::Forward || t.kind == ppsim::Kind::Backward;
      if (t.window >= max_window) continue;
      if (fb ? !tp.local : !hosted[static_cast<size_t>(t.stage)] || rank_of_dev(t.device) != rank_) continue;
      float a = 0.f, b = 0.f;
      CUDA_OK(cudaEventElapsedTime(&a, run_begin_, ev_start_[static_cast<size_t>(k)]));
      CUDA_OK(cudaEventElapsedTime(&b, run_begin_, ev_end_[static_cast<size_t>(k)]));
      const int64_t s_ns = std::llround(static_cast<double>(a) * 1e6);
      int64_t e_ns = std::llround(static_cast<double>(b) * 1e6);
      if (e_ns < s_ns) e_ns = s_ns;
      ppsim::TaskEvent ev;
      ev.kind = t.kind;
      ev.stage = t.stage;
      ev.minibatch = t.minibatch;
      ev.pipeline = t.pipeline;
      ev.device = t.device;
      ev.window = t.window;
      ev.preloaded = t.preloaded;
      ev.start = ppsim::Rat(s_ns);
      ev.duration = ppsim::Rat(e_ns - s_ns);
      busy += static_cast<double>(e_ns - s_ns) * 1e-6;
      events.push_back(ev);
      if (lane_rec_[static_cast<size_t>(k)]) {  // the task's own interval on its stream
        CUDA_OK(cudaEventElapsedTime(&a, run_begin_, ev_lstart_[static_cast<size_t>(k)]));
        CUDA_OK(cudaEventElapsedTime(&b, run_begin_, ev_lend_[static_cast<size_t>(k)]));
        const int64_t ls = std::llround(static_cast<double>(a) * 1e6);
        const int64_t le = std::max(ls, static_cast<int64_t>(std::llround(static_cast<double>(b) * 1e6)));
        ev.start = ppsim::Rat(ls);
        ev.duration = ppsim::Rat(le - ls);
        lane_events.push_back(ev);
      }
    }
  }
  stats.busy_ms = busy;
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

// What this rank allocates, by category (allocate() below, the same formulas), in the units of
// the reference's memory model (H/analysis.hpp:226-330: stage replicas, gradient buffers,
// optimizer-state multiples, live per-stage activations), plus the measured cudaMemGetInfo
// delta across allocate().  Co-resident replicas of one stage share one set of buffers.

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

int64_t Engine::stage_numel(int stage) const { return stages.at(static_cast<size_t>(stage))->numel(); }

void Engine::use_replica_weights(int stage, int pipeline) {
  if (!versioned_) return;
  GptStage& S = *stages[static_cast<size_t>(stage)];
  const int b = rep_buf_[static_cast<size_t>(stage)][static_cast<size_t>(pipeline)];
  S.w = wbuf_[static_cast<size_t>(stage)][static_cast<size_t>(b)];
  S.wt = wtbuf_[static_cast<size_t>(stage)][static_cast<size_t>(b)];
}

// The optimizer step of stage i (detail::apply_update H/optim.hpp:234-268 / AdamW) on this
// rank's state: g / update_div -> master, m, v; bf16 working copy + transposed copy rewritten
// (versioned: into the buffer no replica reads yet); the gradient is zeroed.
void Engine::optimizer_step(int stage, int step, cudaStream_t st) {
  GptStage& S = *stages[static_cast<size_t>(stage)];
  if (versioned_) {
    int& cur = cur_buf_[static_cast<size_t>(stage)];
    cur ^= 1;
    S.w = wbuf_[static_cast<size_t>(stage)][static_cast<size_t>(cur)];
    S.wt = wtbuf_[static_cast<size_t>(stage)][static_cast<size_t>(cur)];
  }
  optimizer_range(stage, step, 0, S.numel(), st);
  const int nt = S.refresh_transposed(st);
  if (nt < 0) throw std::runtime_error("weight transpose failed");
  stats.kernels_launched += nt;
}

// The optimizer step of parameters [off, off + n) of stage i (detail::apply_update
// H/optim.hpp:234-268 / AdamW): g / update_div -> master, m, v; bf16 working copy; gradient
// zeroed.  Elementwise, so any split into ranges gives the same bits as one call.
void Engine::optimizer_range(int stage, int step, int64_t off, int64_t n, cudaStream_t st, int64_t m_off) {
  GptStage& S = *stages[static_cast<size_t>(stage)];
  if (m_off < 0) m_off = off;
  amdp_opt_args o = rc_.optimizer;
  o.step = step;
  o.grad_scale = rc_.optimizer.grad_scale * (1.0f / update_div_);
  ktimer_.begin(K_OPTIM, 0, 34.0 * static_cast<double>(n), st);
  const int rc = amdp_optimizer_step(&o, S.master + off, S.m + m_off, S.v ? S.v + m_off : nullptr, S.grad + off,
                                     S.w + off, n, reinterpret_cast<amdp_stream_t>(st));
  ktimer_.end(st);
  if (rc != 0) throw std::runtime_error("optimizer step failed");
  stats.kernels_launched += 1;
}

void Engine::copy_params(int stage, float* host, int64_t n, bool to_host) {
  GptStage& st = *stages.at(static_cast<size_t>(stage));
  if (!hosted[static_cast<size_t>(stage)]) throw std::invalid_argument("stage not hosted on this rank");
  if (n != st.numel()) throw std::invalid_argument("parameter count mismatch");
  CUDA_OK(cudaStreamSynchronize(cs_));
  if (to_host) {
    CUDA_OK(cudaMemcpy(host, st.master, static_cast<size_t>(n) * sizeof(float), cudaMemcpyDeviceToHost));
  } else {
    if (versioned_) {  // every replica reads the newly written weights
      for (int& b : rep_buf_[static_cast<size_t>(stage)]) b = cur_buf_[static_cast<size_t>(stage)];
      use_replica_weights(stage, 0);
    }
    CUDA_OK(cudaMemcpy(st.master, host, static_cast<size_t>(n) * sizeof(float), cudaMemcpyHostToDevice));
    cast_f32_bf16_kernel<<<std::min<int64_t>((n + 255) / 256, 4 * 148), 256, 0, cs_>>>(
        st.master, reinterpret_cast<bf16*>(st.w), n);
    if (st.refresh_transposed(cs_) < 0) throw std::runtime_error("weight transpose failed");
    CUDA_OK(cudaStreamSynchronize(cs_));
  }
}

}  // namespace amdp

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
