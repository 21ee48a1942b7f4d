// Execution half of the stage executor (see executor.hpp): device buffers and weight init,
// the data-plane and window-machinery operations, the Forward / Backward task bodies on their
// compute streams, eager runs and CUDA-graph capture / replay, the optimizer step.
#include "executor.hpp"

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
}  // namespace

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
    cudaFree(s->ln_part);
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
  cudaFree(d_lens_);
  if (h_lens_) cudaFreeHost(h_lens_);
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
    // deferred LayerNorm parameter gradients (bf16 path; AMDP_LN_DEFER=0 reduces per backward)
    static const bool ln_defer = !getenv("AMDP_LN_DEFER") || atoi(getenv("AMDP_LN_DEFER")) != 0;
    if (ln_defer && !dm.fp32 && st.ln_parts() > 0) {
      CUDA_OK(cudaMalloc(&st.ln_part, st.ln_part_floats() * sizeof(float)));
      CUDA_OK(cudaMemsetAsync(st.ln_part, 0, st.ln_part_floats() * sizeof(float), cs_));
    }
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
  if (dm.pad_token > 0) {
    CUDA_OK(cudaMalloc(&d_lens_, static_cast<size_t>(M_) * dm.B * sizeof(int32_t)));
    CUDA_OK(cudaHostAlloc(&h_lens_, static_cast<size_t>(M_) * dm.B * sizeof(int32_t), cudaHostAllocDefault));
    std::fill(h_lens_, h_lens_ + static_cast<size_t>(M_) * dm.B, dm.S);
  }
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
    const int32_t* klen = d_lens_ ? d_lens_ + static_cast<size_t>(j) * dm.B : nullptr;  // key padding
    const int32_t* lab = d_labels_ + static_cast<size_t>(j) * T;
    const uint16_t* in = tp.in_buf >= 0 ? bufs_[static_cast<size_t>(tp.in_buf)].ptr : nullptr;
    int launched;
    if (task.kind == ppsim::Kind::Forward) {
      uint16_t* out = tp.out_buf >= 0 ? bufs_[static_cast<size_t>(tp.out_buf)].ptr : nullptr;
      launched = S.forward(A, tok, lab, in, out, d_loss_ + j, loss_scale_[static_cast<size_t>(j)],
                           wss_[static_cast<size_t>(si)], cs, &rc, seg_wait, klen);
    } else {
      const uint16_t* gin = tp.gin_buf >= 0 ? bufs_[static_cast<size_t>(tp.gin_buf)].ptr : nullptr;
      uint16_t* gout = tp.gout_buf >= 0 ? bufs_[static_cast<size_t>(tp.gout_buf)].ptr : nullptr;
      // the kernel-timing run serialises the streams so per-launch event spans are exact
      launched = S.backward(A, tok, in, gin, gout, wss_[static_cast<size_t>(si)], cs,
                            ktimer_.enabled ? SideStream{} : sides_[static_cast<size_t>(si)], &rc, klen);
      if (rc == 0 && ln_flush_[static_cast<size_t>(pos)]) launched += S.flush_ln_grads(cs, &rc);
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

// key padding: each sequence's valid length = position of its first pad token (>= 1)
void Engine::set_lengths(const int32_t* h_in) {
  if (!h_lens_) return;
  for (int j = 0; j < M_; ++j)
    for (int b = 0; b < dm.B; ++b) {
      const int32_t* sq = h_in + static_cast<size_t>(j) * dm.T + static_cast<size_t>(b) * dm.S;
      int len = dm.S;
      for (int p = 0; p < dm.S; ++p)
        if (sq[p] == dm.pad_token) {
          len = p;
          break;
        }
      h_lens_[static_cast<size_t>(j) * dm.B + b] = std::max(1, len);
    }
}

void Engine::stage_tokens(const int32_t* h_in, const int32_t* h_lab) {
  set_lengths(h_in);
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
  if (d_lens_)  // the sequences' valid lengths (host-computed in run(), pinned: capturable)
    CUDA_OK(cudaMemcpyAsync(d_lens_, h_lens_, static_cast<size_t>(M_) * dm.B * sizeof(int32_t), cudaMemcpyHostToDevice,
                            cs_));
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
  if (h_in) set_lengths(h_in);  // resident runs keep the lengths stage_tokens() set
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



// What this rank allocates, by category (allocate() below, the same formulas), in the units of
// the reference's memory model (H/analysis.hpp:226-330: stage replicas, gradient buffers,
// optimizer-state multiples, live per-stage activations), plus the measured cudaMemGetInfo
// delta across allocate().  Co-resident replicas of one stage share one set of buffers.



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
