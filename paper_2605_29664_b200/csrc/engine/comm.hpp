// Communication layer of the stage executor: the exchanges the reference models as events —
// the cross-device activation / activation-gradient hop a stage boundary costs
// (H/engine.hpp:119-125) and the window machinery's Reduce / Broadcast / Update
// (H/builder.hpp:272-338) — behind one interface with two backends:
//
//  * IpcComm (default): this library's own data plane over CUDA IPC peer memory.  Every
//    rank exports its boundary-buffer arena, per-stage gradient / weight buffers and a flag
//    array; peers map them (cudaIpcOpenMemHandle) and move data with copy-engine copies and
//    peer-memory reduction kernels, ordered by epoch-valued flags (a one-thread signal kernel
//    stores into the peer's flag array; the waiter blocks its stream on its own flag with
//    cuStreamWaitValue32, or a polling kernel where stream memory operations are
//    unavailable).  The same code runs between GPUs of one NVLink/NVSwitch box (peer
//    mappings over NVLink) and between several processes sharing ONE GPU, which is how the
//    multi-rank data plane is exercised on the single-GPU pool.
//  * NcclComm: ncclSend / ncclRecv and per-stage replica communicators (ncclCommSplit) on one
//    communication stream.
//
// Both give NCCL's completion semantics: when an operation completes on the calling stream,
// every transfer that touches this rank's buffers is finished (a send's buffer may be
// reused, a reduce's root holds the sum, a broadcast's receivers hold the data).  Message
// and collective ids are assigned from the global dispatch order identically on every rank.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

namespace amdp {

// Regions a rank exposes to its peers (IPC backend); `index` = stage (or 0 for the arena).
enum RegionKind : int { REG_BOUNDS = 0, REG_GRAD = 1, REG_W = 2, REG_MASTER = 3, REG_NUM };

struct Span {  // a byte range of a region (same layout on every rank hosting the stage)
  int kind, index;
  size_t offset, bytes;
};

class Comm {
 public:
  virtual ~Comm() = default;
  virtual const char* name() const = 0;

  // ---- setup: regions to expose, then (IPC) one exchange of descriptors through the host
  virtual void register_region(int kind, int index, void* base, size_t bytes) = 0;
  // producer side of message `msg`: its payload lives at `offset` in the boundary arena
  virtual void plan_send(int msg, size_t offset) = 0;
  virtual std::string export_blob() = 0;
  virtual void import_blobs(const std::vector<std::string>& per_rank) = 0;
  virtual bool connected() const = 0;
  virtual void begin_run() = 0;  // new epoch (every rank calls it once per run)

  // ---- point to point (stage boundary hops); `s` orders the call after prior work
  virtual void send(int msg, int peer, const void* buf, size_t bytes, cudaStream_t s) = 0;
  virtual void recv(int msg, int peer, void* dst, size_t bytes, cudaStream_t s) = 0;

  // ---- replica-group collectives (group = sorted ranks hosting the stage; members indexed
  // by their position in it).  ZeRO within the replica group: the window gradient is
  // reduce-scattered (member j ends with the group sum over ranges[j]), each member steps the
  // optimizer on its ranges, and the updated weights are all-gathered.
  using Ranges = std::vector<std::pair<size_t, size_t>>;  // element [lo, hi)
  virtual void reduce_scatter_f32(int coll, const std::vector<int>& group, int stage, float* buf,
                                  const std::vector<Ranges>& ranges, cudaStream_t s) = 0;
  // every member's spans[j] (its own, freshly written) -> all other members.  Returns once this
  // rank has copied everyone's spans; before a member next modifies its own spans it calls
  // allgather_wait(coll, ...) (every other member has copied them).
  virtual void allgather(int coll, const std::vector<int>& group, int stage,
                         const std::vector<std::vector<Span>>& spans, cudaStream_t s) = 0;
  virtual void allgather_wait(int coll, const std::vector<int>& group, cudaStream_t s) = 0;
  // replicated updates: the whole window gradient summed on every member
  virtual void allreduce_f32(int coll, const std::vector<int>& group, int stage, float* buf, size_t n,
                             cudaStream_t s) = 0;

  // this library's kernels launched by the backend (signal / wait / sum), bytes pulled in
  virtual int64_t kernel_launches() const { return 0; }
  virtual int64_t bytes_received() const { return 0; }
  // true: every operation must be issued on one stream (NCCL ops of one communicator)
  virtual bool single_stream() const { return false; }
};

// world/rank: the job; messages / collectives: ids the plan assigned (flag-array sizing).
std::unique_ptr<Comm> make_ipc_comm(int world, int rank, int messages, int collectives);
std::unique_ptr<Comm> make_nccl_comm(int world, int rank, const uint8_t* nccl_id,
                                     const std::vector<std::vector<int>>& stage_groups);

}  // namespace amdp
