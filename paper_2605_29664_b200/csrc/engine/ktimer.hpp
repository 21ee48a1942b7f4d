// Per-kernel-class CUDA-event timing for the executor (bench roofline evidence).
// Events are recorded on the launching stream around each kernel-library call and read
// back once after the run; disabled by default.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <vector>

namespace amdp {

enum KClass : int {
  K_GEMM_FWD = 0,
  K_GEMM_DGRAD,
  K_GEMM_WGRAD,
  K_ATTN_FWD,
  K_ATTN_BWD,
  K_LAYERNORM,
  K_XENT,
  K_EMBED,
  K_OPTIM,
  K_GELU,  // recompute runs only: f = gelu(u) rebuilt by the backward
  K_NUM
};

inline const char* kclass_name(int c) {
  static const char* n[] = {"gemm_fwd", "gemm_dgrad", "gemm_wgrad", "attn_fwd", "attn_bwd",
                            "layernorm", "xent", "embedding", "optimizer", "gelu"};
  return c >= 0 && c < K_NUM ? n[c] : "?";
}

class KTimer {
 public:
  bool enabled = false;
  struct Rec {
    int cls;
    double flops, bytes;
    cudaEvent_t a, b;
  };
  std::array<int64_t, K_NUM> launches{};
  std::array<double, K_NUM> ms{}, flops{}, bytes{};

  void begin(int cls, double fl, double by, cudaStream_t s) {
    if (!enabled) return;
    Rec r{cls, fl, by, ev(), ev()};
    cudaEventRecord(r.a, s);
    open_.push_back(r);
  }
  void end(cudaStream_t s) {
    if (!enabled || open_.empty()) return;
    cudaEventRecord(open_.back().b, s);
    done_.push_back(open_.back());
    open_.pop_back();
  }
  // after the stream is synchronised
  void collect() {
    for (const Rec& r : done_) {
      float t = 0.f;
      cudaEventElapsedTime(&t, r.a, r.b);
      launches[static_cast<size_t>(r.cls)] += 1;
      ms[static_cast<size_t>(r.cls)] += t;
      flops[static_cast<size_t>(r.cls)] += r.flops;
      bytes[static_cast<size_t>(r.cls)] += r.bytes;
      pool_.push_back(r.a);
      pool_.push_back(r.b);
    }
    done_.clear();
  }
  void reset() {
    launches.fill(0);
    ms.fill(0);
    flops.fill(0);
    bytes.fill(0);
  }
  ~KTimer() {
    for (auto e : pool_) cudaEventDestroy(e);
    for (auto& r : done_) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
  }

 private:
  std::vector<Rec> open_, done_;
  std::vector<cudaEvent_t> pool_;
  cudaEvent_t ev() {
    if (!pool_.empty()) {
      cudaEvent_t e = pool_.back();
      pool_.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};

}  // namespace amdp
