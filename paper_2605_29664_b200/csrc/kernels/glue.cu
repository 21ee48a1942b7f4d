// Memory-bound stage glue: LayerNorm fwd/bwd, token+position embedding fwd/bwd,
// fused softmax cross-entropy (loss + dlogits in one pass pair).
// All are HBM-bound: 16-byte vector accesses, one warp per row (LayerNorm) or one
// CTA per row (cross-entropy over the vocabulary), warp-shuffle reductions, grids
// sized in multiples of the SM count.
#include "common.cuh"

namespace amdp {
namespace {

constexpr int LN_MAX_VEC = 12;  // up to 12 x 256 = 3072 columns held in registers per warp

// ---------------------------------------------------------------- LayerNorm forward
__global__ void __launch_bounds__(256) layernorm_fwd_kernel(
    const bf16* __restrict__ x, const float* __restrict__ gamma, const float* __restrict__ beta,
    bf16* __restrict__ y, float* __restrict__ mean_out, float* __restrict__ rstd_out, int rows,
    int cols, float eps) {
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  for (int row = blockIdx.x * warps + (threadIdx.x >> 5); row < rows; row += gridDim.x * warps) {
    const bf16* xr = x + static_cast<size_t>(row) * cols;
    float v[LN_MAX_VEC][8];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < LN_MAX_VEC; ++i) {
      const int c = (i * 32 + lane) * 8;
      if (c < cols) {
        load8(xr + c, v[i]);
#pragma unroll
        for (int e = 0; e < 8; ++e) s += v[i][e];
      }
    }
    const float mean = warp_sum(s) / cols;
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < LN_MAX_VEC; ++i) {
      const int c = (i * 32 + lane) * 8;
      if (c < cols) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float d = v[i][e] - mean;
          ss += d * d;
        }
      }
    }
    const float rstd = rsqrtf(warp_sum(ss) / cols + eps);
    bf16* yr = y + static_cast<size_t>(row) * cols;
#pragma unroll
    for (int i = 0; i < LN_MAX_VEC; ++i) {
      const int c = (i * 32 + lane) * 8;
      if (c < cols) {
        float o[8];
        const float4 g0 = *reinterpret_cast<const float4*>(gamma + c);
        const float4 g1 = *reinterpret_cast<const float4*>(gamma + c + 4);
        const float4 b0 = *reinterpret_cast<const float4*>(beta + c);
        const float4 b1 = *reinterpret_cast<const float4*>(beta + c + 4);
        const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = (v[i][e] - mean) * rstd * g[e] + b[e];
        store8(yr + c, o);
      }
    }
    if (lane == 0) {
      mean_out[row] = mean;
      rstd_out[row] = rstd;
    }
  }
}

// ---------------------------------------------------------------- LayerNorm backward
// Each CTA handles a strided set of rows; per-column dgamma/dbeta partials are kept in
// registers per lane, reduced across the CTA's warps in shared memory and written to
// workspace[block][2*cols]; a second kernel folds the partials into dgamma/dbeta.
__global__ void __launch_bounds__(256) layernorm_bwd_kernel(
    const bf16* __restrict__ dy, const bf16* __restrict__ x, const float* __restrict__ gamma,
    const float* __restrict__ mean_in, const float* __restrict__ rstd_in,
    const bf16* resid_grad, bf16* dx, float* __restrict__ partial, int rows, int cols) {
  extern __shared__ float red[];  // [warps][2*cols]: per-warp dgamma | dbeta partials
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int warps = blockDim.x >> 5;
  float* mine = red + static_cast<size_t>(warp) * 2 * cols;
  for (int c = lane; c < 2 * cols; c += 32) mine[c] = 0.f;
  __syncwarp();

  for (int row = blockIdx.x * warps + warp; row < rows; row += gridDim.x * warps) {
    const size_t off = static_cast<size_t>(row) * cols;
    const float mean = mean_in[row], rstd = rstd_in[row];
    float s1 = 0.f, s2 = 0.f;
    // pass 1: row statistics of dxhat = dy*gamma, column partials into smem
    for (int c = lane * 8; c < cols; c += 256) {
      float xv[8], dv[8];
      load8(x + off + c, xv);
      load8(dy + off + c, dv);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float xh = (xv[e] - mean) * rstd;
        const float dxh = dv[e] * gamma[c + e];
        s1 += dxh;
        s2 += dxh * xh;
        mine[c + e] += dv[e] * xh;
        mine[cols + c + e] += dv[e];
      }
    }
    s1 = warp_sum(s1) / cols;
    s2 = warp_sum(s2) / cols;
    // pass 2: dx (row re-read hits L1)
    for (int c = lane * 8; c < cols; c += 256) {
      float xv[8], dv[8], o[8];
      float r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      load8(x + off + c, xv);
      load8(dy + off + c, dv);
      if (resid_grad) load8(resid_grad + off + c, r);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float xh = (xv[e] - mean) * rstd;
        const float dxh = dv[e] * gamma[c + e];
        o[e] = r[e] + rstd * (dxh - s1 - xh * s2);
      }
      store8(dx + off + c, o);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 2 * cols; c += blockDim.x) {
    float s = 0.f;
    for (int w = 0; w < warps; ++w) s += red[static_cast<size_t>(w) * 2 * cols + c];
    partial[static_cast<size_t>(blockIdx.x) * 2 * cols + c] = s;
  }
}

__global__ void layernorm_bwd_fold(const float* __restrict__ partial, int nblocks, int cols,
                                   float* dgamma, float* dbeta) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= 2 * cols) return;
  float s = 0.f;
  for (int b = 0; b < nblocks; ++b) s += partial[static_cast<size_t>(b) * 2 * cols + c];
  if (c < cols) dgamma[c] += s;
  else dbeta[c - cols] += s;
}

int ln_bwd_blocks(int rows) {
  const int want = (rows + 7) / 8;  // 8 warps per CTA, >= 1 row per warp
  const int cap = 2 * num_sms();
  return want < cap ? want : cap;
}

// ---------------------------------------------------------------- embedding
__global__ void embedding_fwd_kernel(const int32_t* __restrict__ tok, const bf16* __restrict__ wte,
                                     const bf16* __restrict__ wpe, bf16* __restrict__ x, int ntok,
                                     int seq, int hidden) {
  const int vecs = hidden / 8;
  const int64_t total = static_cast<int64_t>(ntok) * vecs;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(i / vecs);
    const int c = static_cast<int>(i % vecs) * 8;
    float a[8], b[8];
    load8(wte + static_cast<size_t>(tok[t]) * hidden + c, a);
    load8(wpe + static_cast<size_t>(t % seq) * hidden + c, b);
#pragma unroll
    for (int e = 0; e < 8; ++e) a[e] += b[e];
    store8(x + static_cast<size_t>(t) * hidden + c, a);
  }
}

__global__ void embedding_bwd_tok_kernel(const int32_t* __restrict__ tok,
                                         const bf16* __restrict__ dx, float* dwte, int ntok,
                                         int hidden) {
  const int vecs = hidden / 8;
  const int64_t total = static_cast<int64_t>(ntok) * vecs;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(i / vecs);
    const int c = static_cast<int>(i % vecs) * 8;
    float g[8];
    load8(dx + static_cast<size_t>(t) * hidden + c, g);
    float4* dst = reinterpret_cast<float4*>(dwte + static_cast<size_t>(tok[t]) * hidden + c);
    atomicAdd(dst, make_float4(g[0], g[1], g[2], g[3]));
    atomicAdd(dst + 1, make_float4(g[4], g[5], g[6], g[7]));
  }
}

__global__ void embedding_bwd_pos_kernel(const bf16* __restrict__ dx, float* dwpe, int ntok,
                                         int seq, int hidden) {
  const int vecs = hidden / 8;
  const int batch = ntok / seq;
  const int total = seq * vecs;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int p = i / vecs;
    const int c = (i % vecs) * 8;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int b = 0; b < batch; ++b) {
      float g[8];
      load8(dx + (static_cast<size_t>(b) * seq + p) * hidden + c, g);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += g[e];
    }
    float* d = dwpe + static_cast<size_t>(p) * hidden + c;
#pragma unroll
    for (int e = 0; e < 8; ++e) d[e] += acc[e];
  }
}

// ---------------------------------------------------------------- cross-entropy
// One CTA per token row: pass 1 online max/sum-exp over the bf16 row, pass 2 writes
// scale * (softmax - onehot) back in place.  The second read of the row hits L2.
__global__ void __launch_bounds__(512) xent_kernel(bf16* logits, const int32_t* __restrict__ labels,
                                                   float* loss_sum, int vocab, int ld,
                                                   float scale) {
  __shared__ float sm_m[16], sm_s[16];
  __shared__ float row_lse;
  const int row = blockIdx.x;
  bf16* lr = logits + static_cast<size_t>(row) * ld;
  const int label = labels[row];
  float m = -INFINITY, s = 0.f;
  const int nvec = vocab / 8;
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    float f[8];
    load8(lr + v * 8, f);
    float bm = f[0];
#pragma unroll
    for (int e = 1; e < 8; ++e) bm = fmaxf(bm, f[e]);
    const float nm = fmaxf(m, bm);
    float acc = s * __expf(m - nm);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc += __expf(f[e] - nm);
    m = nm;
    s = acc;
  }
  // warp then CTA combine of (m, s)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, m, o);
    const float os = __shfl_xor_sync(0xffffffffu, s, o);
    const float nm = fmaxf(m, om);
    s = (nm == -INFINITY) ? 0.f : s * __expf(m - nm) + os * __expf(om - nm);
    m = nm;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sm_m[warp] = m;
    sm_s[warp] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = -INFINITY, S = 0.f;
    for (int w = 0; w < (blockDim.x >> 5); ++w) {
      const float nm = fmaxf(M, sm_m[w]);
      S = (nm == -INFINITY) ? 0.f : S * __expf(M - nm) + sm_s[w] * __expf(sm_m[w] - nm);
      M = nm;
    }
    const float lse = M + __logf(S);
    row_lse = lse;
    if (label >= 0) atomicAdd(loss_sum, lse - __bfloat162float(lr[label]));
  }
  __syncthreads();
  const float lse = row_lse;
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    float f[8];
    load8(lr + v * 8, f);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int col = v * 8 + e;
      f[e] = (label >= 0) ? scale * (__expf(f[e] - lse) - (col == label ? 1.f : 0.f)) : 0.f;
    }
    store8(lr + v * 8, f);
  }
}

}  // namespace
}  // namespace amdp

using namespace amdp;

extern "C" int amdp_layernorm_fwd(const uint16_t* x, const float* gamma, const float* beta,
                                  uint16_t* y, float* mean, float* rstd, int rows, int cols,
                                  float eps, amdp_stream_t stream) {
  if (rows <= 0 || cols <= 0 || cols % 8 != 0 || cols > LN_MAX_VEC * 256) return AMDP_ERR_INVALID;
  const int warps_needed = rows;
  int blocks = (warps_needed + 7) / 8;
  const int cap = 8 * num_sms();
  if (blocks > cap) blocks = cap;
  layernorm_fwd_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const bf16*>(x), gamma, beta, reinterpret_cast<bf16*>(y), mean, rstd, rows,
      cols, eps);
  return cudaGetLastError();
}

extern "C" size_t amdp_layernorm_bwd_workspace(int rows, int cols) {
  return static_cast<size_t>(ln_bwd_blocks(rows)) * 2 * cols * sizeof(float);
}

extern "C" int amdp_layernorm_bwd(const uint16_t* dy, const uint16_t* x, const float* gamma,
                                  const float* mean, const float* rstd,
                                  const uint16_t* resid_grad, uint16_t* dx, float* dgamma,
                                  float* dbeta, void* workspace, int rows, int cols,
                                  amdp_stream_t stream) {
  if (rows <= 0 || cols <= 0 || cols % 8 != 0 || cols > LN_MAX_VEC * 256 || !workspace)
    return AMDP_ERR_INVALID;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int blocks = ln_bwd_blocks(rows);
  const size_t smem = static_cast<size_t>(8) * 2 * cols * sizeof(float);
  static int smem_attr = 0;
  if (smem > 48 * 1024 && static_cast<int>(smem) > smem_attr) {
    cudaFuncSetAttribute(layernorm_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    smem_attr = static_cast<int>(smem);
  }
  layernorm_bwd_kernel<<<blocks, 256, smem, s>>>(
      reinterpret_cast<const bf16*>(dy), reinterpret_cast<const bf16*>(x), gamma, mean, rstd,
      reinterpret_cast<const bf16*>(resid_grad), reinterpret_cast<bf16*>(dx),
      static_cast<float*>(workspace), rows, cols);
  layernorm_bwd_fold<<<(2 * cols + 255) / 256, 256, 0, s>>>(static_cast<float*>(workspace),
                                                           blocks, cols, dgamma, dbeta);
  return cudaGetLastError();
}

extern "C" int amdp_embedding_fwd(const int32_t* tokens, const uint16_t* wte, const uint16_t* wpe,
                                  uint16_t* x, int ntok, int seq, int hidden,
                                  amdp_stream_t stream) {
  if (ntok <= 0 || seq <= 0 || hidden % 8 != 0) return AMDP_ERR_INVALID;
  const int64_t work = static_cast<int64_t>(ntok) * (hidden / 8);
  int blocks = static_cast<int>((work + 255) / 256);
  if (blocks > 16 * num_sms()) blocks = 16 * num_sms();
  embedding_fwd_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      tokens, reinterpret_cast<const bf16*>(wte), reinterpret_cast<const bf16*>(wpe),
      reinterpret_cast<bf16*>(x), ntok, seq, hidden);
  return cudaGetLastError();
}

extern "C" int amdp_embedding_bwd(const int32_t* tokens, const uint16_t* dx, float* dwte,
                                  float* dwpe, int ntok, int seq, int hidden,
                                  amdp_stream_t stream) {
  if (ntok <= 0 || seq <= 0 || hidden % 8 != 0 || ntok % seq != 0) return AMDP_ERR_INVALID;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t work = static_cast<int64_t>(ntok) * (hidden / 8);
  int blocks = static_cast<int>((work + 255) / 256);
  if (blocks > 16 * num_sms()) blocks = 16 * num_sms();
  embedding_bwd_tok_kernel<<<blocks, 256, 0, s>>>(tokens, reinterpret_cast<const bf16*>(dx), dwte,
                                                  ntok, hidden);
  const int pwork = seq * (hidden / 8);
  embedding_bwd_pos_kernel<<<(pwork + 255) / 256, 256, 0, s>>>(reinterpret_cast<const bf16*>(dx),
                                                               dwpe, ntok, seq, hidden);
  return cudaGetLastError();
}

extern "C" int amdp_xent_fwd_bwd(uint16_t* logits, const int32_t* labels, float* loss_sum,
                                 int ntok, int vocab, int ld, float scale, amdp_stream_t stream) {
  if (ntok <= 0 || vocab % 8 != 0 || ld % 8 != 0 || ld < vocab) return AMDP_ERR_INVALID;
  xent_kernel<<<ntok, 512, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<bf16*>(logits), labels, loss_sum, vocab, ld, scale);
  return cudaGetLastError();
}
