// GPT stage model for the AMDP executor: parameter layout of one pipeline stage (a
// contiguous range of transformer layers, plus the embedding on the first stage and the
// final LayerNorm + LM head on the last), its activation slot layout, and the forward /
// backward task bodies as sequences of sm_100a kernel launches (include/amdp_kernels.h).
//
// The reference models a stage only as an opaque cost (ppsim types.hpp:63-64); the
// arithmetic here is this repository's (pre-LN GPT, no linear biases, untied LM head),
// restated on the CPU by oracle/gpt_oracle.py for the loss/weight parity tests.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "amdp_kernels.h"

namespace amdp {

class KTimer;

// Second stream + events for the weight-gradient GEMMs of a backward task.
struct SideStream {
  cudaStream_t side = nullptr;  // nullptr: everything on the main stream
  cudaEvent_t ev[10] = {};
};

struct Dims {
  int L, h, heads, hd, ffn, V, S, B, T;  // T = B * S tokens per minibatch
  bool causal;
  float ln_eps;
  bool recompute = false;  // f and o recomputed in the backward (amdp_model_config.recompute)
  bool fp32 = false;       // fp32 validation mode: activations fp32, amdp_f32_* kernels
  int pad_token = 0;       // > 0: key padding of bidirectional models (amdp_model_config)
  size_t act_bytes() const { return fp32 ? 4 : 2; }  // per activation element
};

struct ParamRef {
  std::string name;
  int64_t off = 0;  // element offset in the stage's flat buffers
  int rows = 0, cols = 0;
  int global_index = 0;  // model-wide tensor id (init seeding, partition-independent)
  int init = 0;          // 0 normal(std), 1 ones, 2 zeros
  float std = 0.f;
  int64_t numel() const { return static_cast<int64_t>(rows) * cols; }
};

struct LayerParams {
  ParamRef ln1_g, ln1_b, qkv, o, ln2_g, ln2_b, fc1, fc2;
};

// Activations of one (stage, minibatch) between its Forward and Backward.
struct LayerActs {
  uint16_t *x = nullptr, *ln1 = nullptr, *qkv = nullptr, *o = nullptr, *hmid = nullptr,
           *ln2 = nullptr, *u = nullptr, *f = nullptr;
  float *ln1_mean = nullptr, *ln1_rstd = nullptr, *ln2_mean = nullptr, *ln2_rstd = nullptr,
        *lse = nullptr;
};
struct SlotActs {
  std::vector<LayerActs> layers;
  uint16_t* x0 = nullptr;      // stage 0: embedding output (layer-0 input)
  uint16_t* xf = nullptr;      // last stage: final residual stream
  uint16_t* lnf = nullptr;     // last stage: final LayerNorm output
  float *lnf_mean = nullptr, *lnf_rstd = nullptr;
  uint16_t* logits = nullptr;  // last stage: [T][V] logits, overwritten by dlogits
};

class GptStage {
 public:
  GptStage(const Dims& d, int stage, int depth, int l0, int l1);

  int stage() const { return stage_; }
  bool first() const { return stage_ == 0; }
  bool last() const { return stage_ == depth_ - 1; }
  int64_t numel() const { return numel_; }
  const std::vector<ParamRef>& params() const { return all_; }
  size_t slot_bytes() const;
  SlotActs carve_slot(uint8_t* base) const;
  // Workspace shared by all tasks on one stream.
  static size_t workspace_bytes(const Dims& d);

  // Buffers of this stage on this GPU.
  float* master = nullptr;  // fp32 weights (owner: updated by the optimizer)
  float* m = nullptr;
  float* v = nullptr;
  float* grad = nullptr;    // fp32 window-accumulated gradient
  uint16_t* w = nullptr;    // bf16 working weights read by the kernels
  // bf16 transposed copies ([in][out], same offsets as `w`) of the matrices the
  // activation-gradient GEMMs read, so dX = dY W runs with a K-major B operand like the
  // forward GEMMs (refresh_transposed() after every write of `w`)
  uint16_t* wt = nullptr;
  int refresh_transposed(cudaStream_t s) const;
  // Deferred LayerNorm parameter gradients (amdp_layernorm_bwd_rows): per-LayerNorm partial
  // rows accumulated over the window's backwards, folded into `grad` by flush_ln_grads() once
  // per window.  Null: every backward reduces its own (amdp_layernorm_bwd).
  float* ln_part = nullptr;
  int ln_count() const { return 2 * (l1_ - l0_) + (last() ? 1 : 0); }
  int ln_parts() const { return amdp_layernorm_bwd_parts(d_.T, d_.h); }
  size_t ln_part_floats() const { return static_cast<size_t>(ln_count()) * ln_parts() * 2 * d_.h; }
  int flush_ln_grads(cudaStream_t s, int* rc) const;
  KTimer* kt = nullptr;     // optional per-kernel-class timing
  double attn_fwd_flops() const {  // algorithmic: QK^T + PV, causal half
    const double f = 4.0 * d_.B * d_.heads * static_cast<double>(d_.S) * d_.S * d_.hd;
    return d_.causal ? f / 2 : f;
  }

  // Task bodies (stream-ordered).  `in`: stage input [T][h] (stages > 0); `out`: stage
  // output [T][h] (stages < depth-1).  Backward: `gin` incoming grad [T][h] (stages <
  // depth-1), `gout` grad w.r.t. the stage input (stages > 0).  Returns the number of
  // kernels launched (>= 0) or a negative/positive error code via `rc`.
  // `seg_ready` (optional, one event per segments() entry): the forward waits for segment k's
  // weights only right before its first use (an optimizer step still running on another
  // stream overlaps the layers already updated).
  int forward(const SlotActs& a, const int32_t* tokens, const int32_t* labels,
              const uint16_t* in, uint16_t* out, float* loss_sum, float loss_scale, uint8_t* ws,
              cudaStream_t s, int* rc, const cudaEvent_t* seg_ready = nullptr,
              const int32_t* key_len = nullptr) const;
  // The stage's parameters as contiguous (offset, numel) segments in the order the forward
  // reads them: [embeddings (stage 0)], one per layer, [final LayerNorm + head (last stage)].
  std::vector<std::pair<int64_t, int64_t>> segments() const;
  // key_len: [seqs_per_minibatch] valid keys per sequence (key padding, bidirectional
  // models), device memory, or null
  int backward(const SlotActs& a, const int32_t* tokens, const uint16_t* in,
               const uint16_t* gin, uint16_t* gout, uint8_t* ws, cudaStream_t s,
               const SideStream& side, int* rc, const int32_t* key_len = nullptr) const;
  // fp32 validation mode bodies (gpt_stage_f32.cu): the same math on float tensors (the
  // activation pointers then address fp32 data), weights read from `master`
  int forward_f32(const SlotActs& a, const int32_t* tokens, const int32_t* labels, const float* in,
                  float* out, float* loss_sum, float loss_scale, uint8_t* ws, cudaStream_t s, int* rc,
                  const cudaEvent_t* seg_ready, const int32_t* key_len) const;
  int backward_f32(const SlotActs& a, const int32_t* tokens, const float* in, const float* gin,
                   float* gout, uint8_t* ws, cudaStream_t s, int* rc, const int32_t* key_len) const;

 private:
  Dims d_;
  int stage_, depth_, l0_, l1_;
  int64_t numel_ = 0;
  std::vector<LayerParams> layers_;
  ParamRef wte_, wpe_, lnf_g_, lnf_b_, head_;
  std::vector<ParamRef> all_;
  ParamRef add(const std::string& name, int rows, int cols, int gidx, int init, float std);
};

}  // namespace amdp
