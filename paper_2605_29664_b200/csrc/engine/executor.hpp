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
//
// Files: executor.hpp (this class), plan.cu (construction: partition, fold, hosting, the
// communication / activation / stream plans, plan and memory reports), executor.cu (device
// buffers, task bodies, window machinery, runs and CUDA graphs), capi.cu (the C-ABI of
// amdp_engine.h and ppsim::execute).
#pragma once

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

#define CUDA_OK(x)                                                                 \
  do {                                                                             \
    cudaError_t _e = (x);                                                          \
    if (_e != cudaSuccess)                                                         \
      throw std::runtime_error(std::string(#x) + ": " + cudaGetErrorString(_e));   \
  } while (0)

inline uint64_t tensor_seed(uint64_t model_seed, int gidx) {
  return model_seed * 1000003ull + static_cast<uint64_t>(gidx);
}

std::vector<int> balance_layers(int L, int depth, int h, int V, int ffn, int seq, bool causal);

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
  // per position: 1 = a local Backward after which the stage's deferred LayerNorm gradients are
  // folded into its window gradient (the last local Backward of the stage before each of its
  // Reduce / Broadcast / Update tasks, and before the end of the run)
  std::vector<char> ln_flush_;
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
  // key padding (dm.pad_token): valid length per (minibatch, sequence), pinned host -> device
  int32_t *d_lens_ = nullptr, *h_lens_ = nullptr;
  void set_lengths(const int32_t* h_in);
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

}  // namespace amdp
