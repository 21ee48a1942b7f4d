// NcclComm: the executor's exchanges through NCCL (see comm.hpp) — ncclSend / ncclRecv on the
// world communicator for stage-boundary hops, and per-stage replica communicators
// (ncclCommSplit, color = stage, over the ranks hosting it) for Reduce / Broadcast /
// all-reduce.  All operations go to one stream (single_stream()): NCCL kernels of one
// communicator issued from several streams can interleave differently on different ranks.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "amdp_engine.h"
#include "comm.hpp"

namespace amdp {
namespace {

#define NCCL_OK(x)                                                                 \
  do {                                                                             \
    ncclResult_t _r = (x);                                                         \
    if (_r != ncclSuccess)                                                         \
      throw std::runtime_error(std::string(#x) + ": " + ncclGetErrorString(_r));   \
  } while (0)

class NcclComm final : public Comm {
 public:
  NcclComm(int world, int rank, const uint8_t* id_bytes, const std::vector<std::vector<int>>& groups)
      : rank_(rank) {
    if (!id_bytes) throw std::invalid_argument("engine: nccl_id required for the NCCL backend");
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, sizeof(id));
    NCCL_OK(ncclCommInitRank(&world_comm_, world, id, rank));
    stage_comm_.assign(groups.size(), nullptr);
    for (size_t i = 0; i < groups.size(); ++i) {  // collective over all ranks, same order
      const auto& g = groups[i];
      const bool in = std::find(g.begin(), g.end(), rank) != g.end();
      ncclComm_t c = nullptr;
      NCCL_OK(ncclCommSplit(world_comm_, in ? static_cast<int>(i) : NCCL_SPLIT_NOCOLOR, rank, &c, nullptr));
      if (c && in && g.size() > 1) stage_comm_[i] = c;
      else if (c) ncclCommDestroy(c);
    }
  }
  ~NcclComm() override {
    for (auto c : stage_comm_)
      if (c) ncclCommDestroy(c);
    if (world_comm_) ncclCommDestroy(world_comm_);
  }
  const char* name() const override { return "nccl"; }
  bool single_stream() const override { return true; }

  void register_region(int kind, int index, void* base, size_t) override { regions_[{kind, index}] = base; }
  void plan_send(int, size_t) override {}
  std::string export_blob() override { return {}; }
  void import_blobs(const std::vector<std::string>&) override {}
  bool connected() const override { return true; }
  void begin_run() override {}

  void send(int, int peer, const void* buf, size_t bytes, cudaStream_t s) override {
    NCCL_OK(ncclSend(buf, bytes, ncclUint8, peer, world_comm_, s));
  }
  void recv(int, int peer, void* dst, size_t bytes, cudaStream_t s) override {
    NCCL_OK(ncclRecv(dst, bytes, ncclUint8, peer, world_comm_, s));
    bytes_in_ += static_cast<int64_t>(bytes);
  }
  void reduce_scatter_f32(int, const std::vector<int>& group, int stage, float* buf, const std::vector<Ranges>& ranges,
                          cudaStream_t s) override {
    NCCL_OK(ncclGroupStart());
    for (size_t j = 0; j < group.size(); ++j)
      for (const auto& [lo, hi] : ranges[j])
        if (hi > lo)
          NCCL_OK(ncclReduce(buf + lo, buf + lo, hi - lo, ncclFloat32, ncclSum, static_cast<int>(j), comm(stage), s));
    NCCL_OK(ncclGroupEnd());
  }
  void allgather(int, const std::vector<int>& group, int stage, const std::vector<std::vector<Span>>& spans,
                 cudaStream_t s) override {
    NCCL_OK(ncclGroupStart());
    for (size_t j = 0; j < group.size(); ++j)
      for (const Span& sp : spans[j]) {
        if (!sp.bytes) continue;
        char* p = static_cast<char*>(regions_.at({sp.kind, sp.index})) + sp.offset;
        NCCL_OK(ncclBroadcast(p, p, sp.bytes, ncclUint8, static_cast<int>(j), comm(stage), s));
        if (group[j] != rank_) bytes_in_ += static_cast<int64_t>(sp.bytes);
      }
    NCCL_OK(ncclGroupEnd());
  }
  void allgather_wait(int, const std::vector<int>&, cudaStream_t) override {}
  void allreduce_f32(int, const std::vector<int>&, int stage, float* buf, size_t n, cudaStream_t s) override {
    NCCL_OK(ncclAllReduce(buf, buf, n, ncclFloat32, ncclSum, comm(stage), s));
  }
  int64_t bytes_received() const override { return bytes_in_; }

 private:
  ncclComm_t comm(int stage) const {
    ncclComm_t c = stage_comm_.at(static_cast<size_t>(stage));
    if (!c) throw std::runtime_error("nccl: no replica communicator for this stage");
    return c;
  }
  static int index_in(const std::vector<int>& g, int r) {
    return static_cast<int>(std::find(g.begin(), g.end(), r) - g.begin());
  }
  int rank_;
  ncclComm_t world_comm_ = nullptr;
  std::vector<ncclComm_t> stage_comm_;
  std::map<std::pair<int, int>, void*> regions_;
  int64_t bytes_in_ = 0;
};

}  // namespace

std::unique_ptr<Comm> make_nccl_comm(int world, int rank, const uint8_t* nccl_id,
                                     const std::vector<std::vector<int>>& stage_groups) {
  return std::unique_ptr<Comm>(new NcclComm(world, rank, nccl_id, stage_groups));
}

}  // namespace amdp

extern "C" int amdp_nccl_unique_id(uint8_t out[128]) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return -3;
  std::memcpy(out, &id, sizeof(id));
  return 0;
}
