// Attention entry points of the C-ABI (include/amdp_kernels.h) for the stage executor.
//
// Every supported shape runs on the 5th-generation tensor cores (tcgen05 / TMEM / TMA):
//   * attention_tc.cu / attention_bwd_tc.cu: tiled kernels, forward seq % 256 == 0 and
//     backward seq % 128 == 0, head_dim 64 / 80 / 128 (GPT-350M / 1.3B / 2.7B, BERT-large);
//   * attention_short_tc.cu: one 128 x 128 tile per (sequence, head), seq <= 128, head_dim
//     32 / 64 (the reference's tiny configuration: seq 64, head_dim 32).
// Other shapes return AMDP_ERR_UNSUPPORTED (round 1's mma.sync kernels are gone).  This file
// also holds the backward's delta = rowsum(dO * O) pass for amdp_attention_bwd.
//
// Layout: qkv rows are tokens [batch*seq][3*H*D] = q | k | v, head-major inside each;
// out / dout rows [batch*seq][H*D]; lse/delta [batch][H][seq] fp32 (lse in the log2 domain,
// softmax scale folded in).
#include "common.cuh"

namespace amdp {
namespace {

// Vectorised variant for D in {32, 64, 128}: one thread per 8-element chunk, D/8 lanes per
// (token, head) reduce with shuffles (groups never straddle a warp).
__global__ void attn_bwd_delta_vec_kernel(const bf16* __restrict__ out, const bf16* __restrict__ dout,
                                          float* __restrict__ delta, int ntok, int seq, int H, int D) {
  grid_dep_wait();  // PDL: predecessor's outputs visible from here
  grid_dep_trigger();
  const int G = D / 8;
  const int64_t chunks = static_cast<int64_t>(ntok) * H * G;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < chunks;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float o[8], d[8];
    load8(out + i * 8, o);
    load8(dout + i * 8, d);
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) s += o[e] * d[e];
    for (int m = G >> 1; m > 0; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
    if (i % G == 0) {
      const int64_t th = i / G;  // token * H + head
      const int tok = static_cast<int>(th / H), h = static_cast<int>(th % H);
      delta[(static_cast<size_t>(tok / seq) * H + h) * seq + tok % seq] = s;
    }
  }
}

// delta for head dims whose 8-element chunk count is not a power of two (head_dim 80): one
// thread per (token, head) row, 16-byte loads.
__global__ void attn_bwd_delta_row_kernel(const bf16* __restrict__ out, const bf16* __restrict__ dout,
                                          float* __restrict__ delta, int ntok, int seq, int H, int D) {
  grid_dep_wait();  // PDL: predecessor's outputs visible from here
  grid_dep_trigger();
  const int64_t rows = static_cast<int64_t>(ntok) * H;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < D; c += 8) {
      float o[8], d[8];
      load8(out + i * D + c, o);
      load8(dout + i * D + c, d);
#pragma unroll
      for (int e = 0; e < 8; ++e) s += o[e] * d[e];
    }
    const int tok = static_cast<int>(i / H), h = static_cast<int>(i % H);
    delta[(static_cast<size_t>(tok / seq) * H + h) * seq + tok % seq] = s;
  }
}

}  // namespace
}  // namespace amdp

namespace amdp {
int attention_fwd_tc(const bf16* qkv, bf16* out, float* lse, int B, int S, int H, int D, int causal,
                     const int32_t* key_len, cudaStream_t st);
int attention_bwd_tc(const bf16* qkv, const bf16* dout, const float* lse, const float* delta, bf16* dqkv, int B,
                     int S, int H, int D, int causal, const int32_t* key_len, uint8_t* ds_ws, cudaStream_t st);
size_t attention_bwd_ds_bytes(int B, int S, int H, int causal);
// attention_short_tc.cu: seq <= 128, head_dim 32 / 64 (one 128 x 128 tile per sequence and head)
bool attention_short_supported(int S, int D);
int attention_fwd_short(const bf16* qkv, bf16* out, float* lse, int B, int S, int H, int D, int causal,
                        const int32_t* key_len, cudaStream_t st);
int attention_bwd_short(const bf16* qkv, const bf16* dout, const float* lse, const float* delta, bf16* dqkv, int B,
                        int S, int H, int D, int causal, const int32_t* key_len, cudaStream_t st);
bool attention_tiled_bwd(int S, int D) { return (D == 64 || D == 80 || D == 128) && S % 128 == 0; }
}

using namespace amdp;

extern "C" int amdp_attention_fwd(const uint16_t* qkv, uint16_t* out, float* lse, int batch,
                                  int seq, int heads, int head_dim, int causal, const int32_t* key_len,
                                  amdp_stream_t stream) {
  if (batch <= 0 || seq <= 0 || seq % 64 != 0 || heads <= 0) return AMDP_ERR_INVALID;
  if (causal && key_len) return AMDP_ERR_UNSUPPORTED;  // key padding is for bidirectional models
  auto q = reinterpret_cast<const bf16*>(qkv);
  auto o = reinterpret_cast<bf16*>(out);
  auto s = reinterpret_cast<cudaStream_t>(stream);
  if ((head_dim == 64 || head_dim == 80 || head_dim == 128) && seq % 256 == 0)  // tcgen05 path
    return attention_fwd_tc(q, o, lse, batch, seq, heads, head_dim, causal, key_len, s);
  if (attention_short_supported(seq, head_dim))  // tcgen05, one tile per sequence
    return attention_fwd_short(q, o, lse, batch, seq, heads, head_dim, causal, key_len, s);
  return AMDP_ERR_UNSUPPORTED;
}

namespace {
// workspace = [delta: batch * heads * seq floats, padded to 256 B][dS^T scratch of the tiled path]
size_t delta_bytes(int batch, int seq, int heads) {
  return (static_cast<size_t>(batch) * seq * heads * sizeof(float) + 255) & ~static_cast<size_t>(255);
}
}  // namespace

extern "C" size_t amdp_attention_bwd_scratch_bytes(int batch, int seq, int heads, int head_dim, int causal) {
  // head_dim 80 keeps the dQ kernel that recomputes S / dP (attention_bwd_tc): no scratch
  if (batch <= 0 || seq <= 0 || heads <= 0 || !attention_tiled_bwd(seq, head_dim) || head_dim == 80) return 0;
  return attention_bwd_ds_bytes(batch, seq, heads, causal ? 1 : 0);
}

extern "C" size_t amdp_attention_bwd_workspace_causal(int batch, int seq, int heads, int head_dim, int causal) {
  return delta_bytes(batch, seq, heads) + amdp_attention_bwd_scratch_bytes(batch, seq, heads, head_dim, causal);
}

extern "C" size_t amdp_attention_bwd_workspace(int batch, int seq, int heads, int head_dim) {
  // bidirectional scratch: an upper bound for either value of causal
  return amdp_attention_bwd_workspace_causal(batch, seq, heads, head_dim, 0);
}

extern "C" int amdp_attention_bwd_delta_ws(const uint16_t* qkv, const uint16_t* dout, const float* lse,
                                           const float* delta, uint16_t* dqkv, void* scratch, int batch, int seq,
                                           int heads, int head_dim, int causal, const int32_t* key_len,
                                           amdp_stream_t stream) {
  if (batch <= 0 || seq <= 0 || heads <= 0 || !delta) return AMDP_ERR_INVALID;
  if (causal && key_len) return AMDP_ERR_UNSUPPORTED;
  if (!amdp_attention_bwd_delta_supported(seq, head_dim)) return AMDP_ERR_UNSUPPORTED;
  if (!attention_tiled_bwd(seq, head_dim))
    return attention_bwd_short(reinterpret_cast<const bf16*>(qkv), reinterpret_cast<const bf16*>(dout), lse, delta,
                               reinterpret_cast<bf16*>(dqkv), batch, seq, heads, head_dim, causal, key_len,
                               reinterpret_cast<cudaStream_t>(stream));
  return attention_bwd_tc(reinterpret_cast<const bf16*>(qkv), reinterpret_cast<const bf16*>(dout), lse,
                          const_cast<float*>(delta), reinterpret_cast<bf16*>(dqkv), batch, seq, heads, head_dim,
                          causal, key_len, static_cast<uint8_t*>(scratch), reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int amdp_attention_bwd_delta(const uint16_t* qkv, const uint16_t* dout, const float* lse,
                                        const float* delta, uint16_t* dqkv, int batch, int seq, int heads,
                                        int head_dim, int causal, const int32_t* key_len, amdp_stream_t stream) {
  return amdp_attention_bwd_delta_ws(qkv, dout, lse, delta, dqkv, nullptr, batch, seq, heads, head_dim, causal,
                                     key_len, stream);
}

extern "C" int amdp_attention_impl(int seq, int head_dim, int backward) {
  const bool tc_dim = head_dim == 64 || head_dim == 80 || head_dim == 128;
  if (seq <= 0 || seq % 64 != 0) return -1;
  if (tc_dim && seq % (backward ? 128 : 256) == 0) return AMDP_ATTN_IMPL_TCGEN05;
  if (attention_short_supported(seq, head_dim)) return AMDP_ATTN_IMPL_TCGEN05;
  return -1;
}

extern "C" int amdp_attention_bwd_delta_supported(int seq, int head_dim) {
  return attention_tiled_bwd(seq, head_dim) || attention_short_supported(seq, head_dim);
}



extern "C" int amdp_attention_bwd(const uint16_t* qkv, const uint16_t* out, const uint16_t* dout,
                                  const float* lse, uint16_t* dqkv, void* workspace, int batch,
                                  int seq, int heads, int head_dim, int causal, const int32_t* key_len,
                                  amdp_stream_t stream) {
  if (batch <= 0 || seq <= 0 || seq % 64 != 0 || heads <= 0 || !workspace) return AMDP_ERR_INVALID;
  if (causal && key_len) return AMDP_ERR_UNSUPPORTED;
  auto q = reinterpret_cast<const bf16*>(qkv);
  auto o = reinterpret_cast<const bf16*>(out);
  auto d = reinterpret_cast<const bf16*>(dout);
  auto dq = reinterpret_cast<bf16*>(dqkv);
  auto w = static_cast<float*>(workspace);
  auto s = reinterpret_cast<cudaStream_t>(stream);
  if (attention_tiled_bwd(seq, head_dim) || attention_short_supported(seq, head_dim)) {  // tcgen05 paths
    const int ntok = batch * seq;
    const int64_t chunks = static_cast<int64_t>(ntok) * heads * (head_dim / 8);
    int64_t blocks = (chunks + 255) / 256;
    if (blocks > 16 * num_sms()) blocks = 16 * num_sms();  // grid-stride; multiple of 256 threads
    if ((head_dim / 8) & (head_dim / 8 - 1)) {  // shuffle groups need a power-of-two chunk count
      const int64_t rows = static_cast<int64_t>(ntok) * heads;
      launch_pdl(attn_bwd_delta_row_kernel, dim3(static_cast<int>(std::min<int64_t>((rows + 255) / 256, 16 * num_sms()))), dim3(256), 0, s, 
          o, d, w, ntok, seq, heads, head_dim);
    } else {
      launch_pdl(attn_bwd_delta_vec_kernel, dim3(static_cast<int>(blocks)), dim3(256), 0, s, o, d, w, ntok, seq, heads, head_dim);
    }
    if (!attention_tiled_bwd(seq, head_dim))
      return attention_bwd_short(q, d, lse, w, dq, batch, seq, heads, head_dim, causal, key_len, s);
    return attention_bwd_tc(q, d, lse, w, dq, batch, seq, heads, head_dim, causal, key_len,
                            static_cast<uint8_t*>(workspace) + delta_bytes(batch, seq, heads), s);
  }
  return AMDP_ERR_UNSUPPORTED;
}
