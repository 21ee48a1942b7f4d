// IpcComm: the executor's data plane over CUDA IPC peer memory (see comm.hpp).
//
// Flag array of one rank (int32, waited on by that rank only, written by its peers):
//   [0, M)                 READY(msg)   the producer's payload of message msg is complete
//   [M, 2M)                ACK(msg)     the consumer has copied message msg out
//   2M + 32 c + [0, 8)     collective c: phase-1 arrival of group member k (its data ready)
//   2M + 32 c + [8, 16)    phase-2 arrival (reduce-scatter / all-reduce: its ranges summed;
//                          all-gather: it has copied every other member's spans)
//   2M + 32 c + [16, 24)   phase-3 arrival (all-reduce: member gathered every chunk)
// A flag holds the epoch (run counter) of its last signal; waits are "flag >= epoch", so no
// flag is ever reset and consecutive runs cannot confuse each other.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "comm.hpp"

namespace amdp {
namespace {

#define IPC_OK(x)                                                                  \
  do {                                                                             \
    cudaError_t _e = (x);                                                          \
    if (_e != cudaSuccess)                                                         \
      throw std::runtime_error(std::string("ipc: ") + #x + ": " + cudaGetErrorString(_e)); \
  } while (0)

constexpr int kMaxGroup = 8;
constexpr int kCollStride = 32;

struct SigTargets {
  int* p[kMaxGroup];
  int n;
  int value;
};

// Release-store the epoch into up to 8 peer flags after everything before it on the stream.
__global__ void ipc_signal_kernel(SigTargets t) {
  if (static_cast<int>(threadIdx.x) < t.n) {
    __threadfence_system();
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(t.p[threadIdx.x]), "r"(t.value) : "memory");
  }
}

// Fallback wait where stream memory operations are unavailable: poll with acquire loads.
__global__ void ipc_wait_kernel(const int* f, int value) {
  if (threadIdx.x == 0) {
    int v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if (v - value >= 0) break;
      __nanosleep(200);
    }
  }
}

struct SumSrcs {
  const float* p[kMaxGroup];
  int n;
};

// out[i] = src_0[i] + src_1[i] + ... in group order (out may alias one source): deterministic.
__global__ void __launch_bounds__(256) ipc_sum_kernel(float* out, SumSrcs s, size_t n) {
  const size_t n4 = n / 4;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4; i += stride) {
    float4 a = reinterpret_cast<const float4*>(s.p[0])[i];
    for (int k = 1; k < s.n; ++k) {
      const float4 b = reinterpret_cast<const float4*>(s.p[k])[i];
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    reinterpret_cast<float4*>(out)[i] = a;
  }
  for (size_t i = n4 * 4 + blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    float a = s.p[0][i];
    for (int k = 1; k < s.n; ++k) a += s.p[k][i];
    out[i] = a;
  }
}

using PFN_wait32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct Handle {
  int kind, index;
  uint64_t bytes;
  cudaIpcMemHandle_t h;
};

class IpcComm final : public Comm {
 public:
  IpcComm(int world, int rank, int messages, int collectives)
      : world_(world), rank_(rank), nmsg_(messages), ncoll_(collectives) {
    nflags_ = static_cast<size_t>(2 * nmsg_ + kCollStride * ncoll_ + 1);
    IPC_OK(cudaMalloc(&flags_, nflags_ * sizeof(int)));
    IPC_OK(cudaMemset(flags_, 0, nflags_ * sizeof(int)));
    register_region_raw(-1, 0, flags_, nflags_ * sizeof(int));
    const char* mode = getenv("AMDP_IPC_WAIT");
    if (!(mode && std::strcmp(mode, "kernel") == 0)) {
      cudaDriverEntryPointQueryResult q;
      void* fn = nullptr;
      if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        wait32_ = reinterpret_cast<PFN_wait32>(fn);
    }
    peers_.resize(static_cast<size_t>(world_));
  }

  ~IpcComm() override {
    cudaDeviceSynchronize();
    for (auto& p : peers_)
      for (void* q : p.opened) cudaIpcCloseMemHandle(q);
    cudaFree(flags_);
  }

  const char* name() const override { return "ipc"; }

  void register_region(int kind, int index, void* base, size_t bytes) override {
    register_region_raw(kind, index, base, bytes);
  }
  void plan_send(int msg, size_t offset) override { sends_.emplace_back(msg, offset); }

  std::string export_blob() override {
    std::string b;
    auto put = [&](const void* p, size_t n) { b.append(static_cast<const char*>(p), n); };
    const int hdr[3] = {0x41495043, rank_, static_cast<int>(local_.size())};
    put(hdr, sizeof(hdr));
    for (const auto& r : local_) put(&r, sizeof(r));
    const int ns = static_cast<int>(sends_.size());
    put(&ns, sizeof(ns));
    for (const auto& s : sends_) {
      const int64_t e[2] = {s.first, static_cast<int64_t>(s.second)};
      put(e, sizeof(e));
    }
    return b;
  }

  void import_blobs(const std::vector<std::string>& all) override {
    if (static_cast<int>(all.size()) != world_) throw std::invalid_argument("ipc: one descriptor per rank expected");
    for (int r = 0; r < world_; ++r) {
      if (r == rank_) continue;
      const std::string& b = all[static_cast<size_t>(r)];
      size_t at = 0;
      auto get = [&](void* p, size_t n) {
        if (at + n > b.size()) throw std::invalid_argument("ipc: truncated descriptor");
        std::memcpy(p, b.data() + at, n);
        at += n;
      };
      int hdr[3];
      get(hdr, sizeof(hdr));
      if (hdr[0] != 0x41495043 || hdr[1] != r) throw std::invalid_argument("ipc: bad descriptor");
      Peer& p = peers_[static_cast<size_t>(r)];
      for (int k = 0; k < hdr[2]; ++k) {
        Handle h;
        get(&h, sizeof(h));
        void* ptr = nullptr;
        IPC_OK(cudaIpcOpenMemHandle(&ptr, h.h, cudaIpcMemLazyEnablePeerAccess));
        p.opened.push_back(ptr);
        if (h.kind == -1) p.flags = static_cast<int*>(ptr);
        else p.regions[{h.kind, h.index}] = ptr;
      }
      int ns = 0;
      get(&ns, sizeof(ns));
      for (int k = 0; k < ns; ++k) {
        int64_t e[2];
        get(e, sizeof(e));
        p.send_off[static_cast<int>(e[0])] = static_cast<size_t>(e[1]);
      }
      if (!p.flags) throw std::invalid_argument("ipc: peer exported no flag array");
    }
    connected_ = true;
  }

  bool connected() const override { return connected_ || world_ == 1; }
  void begin_run() override { ++epoch_; }

  void send(int msg, int peer, const void*, size_t, cudaStream_t s) override {
    signal(s, {flag_of(peer, msg)});
    wait(s, nmsg_ + msg);
  }

  void recv(int msg, int peer, void* dst, size_t bytes, cudaStream_t s) override {
    const Peer& p = peers_.at(static_cast<size_t>(peer));
    auto it = p.send_off.find(msg);
    if (it == p.send_off.end()) throw std::runtime_error("ipc: peer has no send planned for this message");
    wait(s, msg);
    IPC_OK(cudaMemcpyAsync(dst, static_cast<const char*>(region(peer, REG_BOUNDS, 0)) + it->second, bytes,
                           cudaMemcpyDeviceToDevice, s));
    signal(s, {flag_of(peer, nmsg_ + msg)});
    bytes_in_ += static_cast<int64_t>(bytes);
  }

  void reduce_scatter_f32(int coll, const std::vector<int>& group, int stage, float* buf,
                          const std::vector<Ranges>& ranges, cudaStream_t s) override {
    const int G = static_cast<int>(group.size()), base = coll_base(coll), me = index_in(group, rank_);
    // 1. every member's window gradient is complete
    signal(s, to_others(group, base + me));
    wait_others(group, base, s);
    // 2. this member sums its ranges over the group (group order: deterministic)
    for (const auto& [lo, hi] : ranges.at(static_cast<size_t>(me))) {
      if (hi <= lo) continue;
      SumSrcs src{};
      src.n = G;
      for (int j = 0; j < G; ++j)
        src.p[j] = (j == me ? buf : static_cast<const float*>(region(group[static_cast<size_t>(j)], REG_GRAD, stage))) + lo;
      launch_sum(buf + lo, src, hi - lo, s);
      bytes_in_ += static_cast<int64_t>((G - 1) * (hi - lo) * sizeof(float));
    }
    // 3. nobody modifies its gradient before every member has read its ranges from it
    signal(s, to_others(group, base + 8 + me));
    wait_others(group, base + 8, s);
  }

  void allgather(int coll, const std::vector<int>& group, int stage, const std::vector<std::vector<Span>>& spans,
                 cudaStream_t s) override {
    (void)stage;
    const int G = static_cast<int>(group.size()), base = coll_base(coll), me = index_in(group, rank_);
    signal(s, to_others(group, base + me));  // my spans are written
    for (int j = 0; j < G; ++j) {
      if (j == me) continue;
      wait(s, base + j);
      for (const Span& sp : spans.at(static_cast<size_t>(j))) {
        if (!sp.bytes) continue;
        char* dst = static_cast<char*>(local_region(sp.kind, sp.index)) + sp.offset;
        const char* src = static_cast<const char*>(region(group[static_cast<size_t>(j)], sp.kind, sp.index)) + sp.offset;
        IPC_OK(cudaMemcpyAsync(dst, src, sp.bytes, cudaMemcpyDeviceToDevice, s));
        bytes_in_ += static_cast<int64_t>(sp.bytes);
      }
    }
    signal(s, to_others(group, base + 8 + me));  // I have copied everyone's
  }

  void allgather_wait(int coll, const std::vector<int>& group, cudaStream_t s) override {
    wait_others(group, coll_base(coll) + 8, s);
  }

  void allreduce_f32(int coll, const std::vector<int>& group, int stage, float* buf, size_t n,
                     cudaStream_t s) override {
    const int G = static_cast<int>(group.size()), base = coll_base(coll), me = index_in(group, rank_);
    auto others = [&](int off) {
      std::vector<int*> t;
      for (int j = 0; j < G; ++j)
        if (j != me) t.push_back(flag_of(group[static_cast<size_t>(j)], base + off + me));
      return t;
    };
    auto wait_others = [&](int off) {
      for (int j = 0; j < G; ++j)
        if (j != me) wait(s, base + off + j);
    };
    auto chunk = [&](int j) {  // 4-float aligned chunk j of G
      const size_t per = ((n + G - 1) / G + 3) / 4 * 4;
      const size_t lo = std::min(n, per * static_cast<size_t>(j)), hi = std::min(n, lo + per);
      return std::make_pair(lo, hi);
    };
    auto peer_grad = [&](int j) {
      return j == me ? buf : static_cast<float*>(region(group[static_cast<size_t>(j)], REG_GRAD, stage));
    };
    // 1. every member's window gradient is complete
    signal(s, others(0));
    wait_others(0);
    // 2. reduce-scatter: this member sums chunk `me` over the group (group order)
    {
      const auto [lo, hi] = chunk(me);
      if (hi > lo) {
        SumSrcs src{};
        src.n = G;
        for (int j = 0; j < G; ++j) src.p[j] = peer_grad(j) + lo;
        launch_sum(buf + lo, src, hi - lo, s);
      }
    }
    signal(s, others(8));
    wait_others(8);
    // 3. all-gather: copy every other member's summed chunk
    for (int j = 0; j < G; ++j) {
      if (j == me) continue;
      const auto [lo, hi] = chunk(j);
      if (hi > lo) {
        IPC_OK(cudaMemcpyAsync(buf + lo, peer_grad(j) + lo, (hi - lo) * sizeof(float), cudaMemcpyDeviceToDevice, s));
        bytes_in_ += static_cast<int64_t>((hi - lo) * sizeof(float));
      }
    }
    // 4. nobody modifies its buffer before every member has gathered from it
    signal(s, others(16));
    wait_others(16);
  }

 private:
  struct Peer {
    int* flags = nullptr;
    std::map<std::pair<int, int>, void*> regions;
    std::unordered_map<int, size_t> send_off;
    std::vector<void*> opened;
  };

  void register_region_raw(int kind, int index, void* base, size_t bytes) {
    Handle h{};
    h.kind = kind;
    h.index = index;
    h.bytes = bytes;
    IPC_OK(cudaIpcGetMemHandle(&h.h, base));
    local_.push_back(h);
    local_ptr_[{kind, index}] = base;
  }
  void* local_region(int kind, int index) const {
    auto it = local_ptr_.find({kind, index});
    if (it == local_ptr_.end()) throw std::runtime_error("ipc: region not registered locally");
    return it->second;
  }
  void* region(int peer, int kind, int index) const {
    const auto& m = peers_.at(static_cast<size_t>(peer)).regions;
    auto it = m.find({kind, index});
    if (it == m.end()) throw std::runtime_error("ipc: peer " + std::to_string(peer) + " exported no region (" +
                                                std::to_string(kind) + "," + std::to_string(index) + ")");
    return it->second;
  }
  int* flag_of(int peer, int idx) const { return peers_.at(static_cast<size_t>(peer)).flags + idx; }
  // flag `idx` of every other group member / wait for flags base + j of every other member j
  std::vector<int*> to_others(const std::vector<int>& group, int idx) const {
    std::vector<int*> t;
    for (int r : group)
      if (r != rank_) t.push_back(flag_of(r, idx));
    return t;
  }
  void wait_others(const std::vector<int>& group, int base, cudaStream_t s) {
    const int me = index_in(group, rank_);
    for (int j = 0; j < static_cast<int>(group.size()); ++j)
      if (j != me) wait(s, base + j);
  }
  int coll_base(int coll) const { return 2 * nmsg_ + kCollStride * coll; }
  static int index_in(const std::vector<int>& g, int r) {
    auto it = std::find(g.begin(), g.end(), r);
    if (it == g.end() || g.size() > static_cast<size_t>(kMaxGroup))
      throw std::runtime_error("ipc: rank not in group (or group larger than 8)");
    return static_cast<int>(it - g.begin());
  }

  void signal(cudaStream_t s, const std::vector<int*>& targets) {
    for (size_t k = 0; k < targets.size(); k += kMaxGroup) {
      SigTargets t{};
      t.n = static_cast<int>(std::min<size_t>(kMaxGroup, targets.size() - k));
      for (int j = 0; j < t.n; ++j) t.p[j] = targets[k + static_cast<size_t>(j)];
      t.value = static_cast<int>(epoch_);
      ipc_signal_kernel<<<1, 32, 0, s>>>(t);
      IPC_OK(cudaGetLastError());
      ++launches_;
    }
  }
  void wait(cudaStream_t s, int idx) {
    int* f = flags_ + idx;
    if (wait32_) {
      const CUresult r = wait32_(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(f),
                                 static_cast<cuuint32_t>(epoch_), CU_STREAM_WAIT_VALUE_GEQ);
      if (r == CUDA_SUCCESS) return;
      wait32_ = nullptr;  // stream memory operations unavailable: poll from a kernel instead
    }
    ipc_wait_kernel<<<1, 32, 0, s>>>(f, static_cast<int>(epoch_));
    IPC_OK(cudaGetLastError());
    ++launches_;
  }
  void launch_sum(float* out, const SumSrcs& src, size_t n, cudaStream_t s) {
    const size_t blocks = std::min<size_t>((n / 4 + 255) / 256 + 1, 4 * 148);
    ipc_sum_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(out, src, n);
    IPC_OK(cudaGetLastError());
    ++launches_;
  }

  int world_, rank_, nmsg_, ncoll_;
  int* flags_ = nullptr;
  size_t nflags_ = 0;
  std::vector<Handle> local_;
  std::map<std::pair<int, int>, void*> local_ptr_;
  std::vector<std::pair<int, size_t>> sends_;
  std::vector<Peer> peers_;
  uint32_t epoch_ = 0;
  bool connected_ = false;
  PFN_wait32 wait32_ = nullptr;

  int64_t bytes_in_ = 0, launches_ = 0;

 public:
  int64_t kernel_launches() const override { return launches_; }
  int64_t bytes_received() const override { return bytes_in_; }
};

}  // namespace

std::unique_ptr<Comm> make_ipc_comm(int world, int rank, int messages, int collectives) {
  return std::unique_ptr<Comm>(new IpcComm(world, rank, messages, collectives));
}

}  // namespace amdp
