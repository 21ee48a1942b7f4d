// fp32 validation mode (north_star: "tightened for an fp32 validation mode"): the stage math
// of the bf16 production path with every tensor in fp32 and every product accumulated in
// fp32 on the CUDA cores — no bf16 storage, no tensor-core rounding, tanhf / expf / logf
// instead of the SFU approximations.  Against the fp64 CPU oracle (emulate_bf16=False) the
// engine then matches to float rounding, which is what lets the losses / weights tolerance
// tighten from bf16's 1e-3.  These kernels favour clarity and determinism over speed (fixed
// summation orders, no atomics); the production path is the bf16 tcgen05 one.
#include <cmath>

#include "common.cuh"

namespace amdp {
namespace {

constexpr float kGeluK0 = 0.7978845608028654f, kGeluK1 = 0.044715f;
__device__ __forceinline__ float gelu_f32(float x) {
  return 0.5f * x * (1.f + tanhf(kGeluK0 * x * (1.f + kGeluK1 * x * x)));
}
__device__ __forceinline__ float gelu_grad_f32(float x) {
  const float t = tanhf(kGeluK0 * x * (1.f + kGeluK1 * x * x));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * kGeluK0 * (1.f + 3.f * kGeluK1 * x * x);
}

// ---------------------------------------------------------------- GEMM
// C = epi(alpha * A(m,k) B(n,k)), the operand conventions of amdp_gemm: A element (m,k) at
// A[m*lda + k] (K-major) or A[k*lda + m] (MN-major), B element (n,k) at B[n*ldb + k] or
// B[k*ldb + n].  64x64 tiles, K in steps of 16 through shared memory, 4x4 per thread.
constexpr int FT = 64, FK = 16;
template <bool AMN, bool BMN>
__global__ void __launch_bounds__(256) f32_gemm_kernel(int M, int N, int K, const float* __restrict__ A, int lda,
                                                       const float* __restrict__ B, int ldb, float* C, int ldc,
                                                       const float* __restrict__ aux, int ld_aux, float* C2, int ldc2,
                                                       int epi, float alpha) {
  __shared__ float As[FK][FT + 4], Bs[FK][FT + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * FT, n0 = blockIdx.x * FT;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += FK) {
    for (int i = threadIdx.x; i < FT * FK; i += 256) {
      int r, kk;
      if (AMN) {  // coalesced along m
        r = i % FT;
        kk = i / FT;
      } else {
        r = i / FK;
        kk = i % FK;
      }
      const int gm = m0 + r, gk = k0 + kk;
      As[kk][r] = (gm < M && gk < K) ? (AMN ? A[static_cast<size_t>(gk) * lda + gm] : A[static_cast<size_t>(gm) * lda + gk]) : 0.f;
      int c, kb;
      if (BMN) {
        c = i % FT;
        kb = i / FT;
      } else {
        c = i / FK;
        kb = i % FK;
      }
      const int gn = n0 + c, gk2 = k0 + kb;
      Bs[kb][c] = (gn < N && gk2 < K) ? (BMN ? B[static_cast<size_t>(gk2) * ldb + gn] : B[static_cast<size_t>(gn) * ldb + gk2]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < FK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      const float v = alpha * acc[i][j];
      float* c = C + static_cast<size_t>(m) * ldc + n;
      switch (epi) {
        case AMDP_EPI_GELU:
          C2[static_cast<size_t>(m) * ldc2 + n] = v;
          *c = gelu_f32(v);
          break;
        case AMDP_EPI_RESIDUAL:
          *c = v + aux[static_cast<size_t>(m) * ld_aux + n];
          break;
        case AMDP_EPI_GELU_BWD:
          *c = v * gelu_grad_f32(aux[static_cast<size_t>(m) * ld_aux + n]);
          break;
        case AMDP_EPI_ACCUM_F32:
          *c += v;
          break;
        default:
          *c = v;
      }
    }
  }
}

// ---------------------------------------------------------------- LayerNorm (warp per row)
__global__ void f32_ln_fwd_kernel(const float* __restrict__ x, const float* __restrict__ g, const float* __restrict__ b,
                                  float* __restrict__ y, float* __restrict__ mean, float* __restrict__ rstd, int rows,
                                  int cols, float eps) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* xr = x + static_cast<size_t>(row) * cols;
  float s = 0.f;
  for (int c = lane; c < cols; c += 32) s += xr[c];
  const float mu = warp_sum(s) / cols;
  float v = 0.f;
  for (int c = lane; c < cols; c += 32) v += (xr[c] - mu) * (xr[c] - mu);
  const float r = rsqrtf(warp_sum(v) / cols + eps);
  for (int c = lane; c < cols; c += 32) y[static_cast<size_t>(row) * cols + c] = (xr[c] - mu) * r * g[c] + b[c];
  if (lane == 0) {
    mean[row] = mu;
    rstd[row] = r;
  }
}

__global__ void f32_ln_bwd_dx_kernel(const float* __restrict__ dy, const float* __restrict__ x, const float* __restrict__ g,
                                     const float* __restrict__ mean, const float* __restrict__ rstd,
                                     const float* __restrict__ resid, float* __restrict__ dx, int rows, int cols) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= rows) return;
  const size_t off = static_cast<size_t>(row) * cols;
  const float mu = mean[row], r = rstd[row];
  float s1 = 0.f, s2 = 0.f;
  for (int c = lane; c < cols; c += 32) {
    const float dxh = dy[off + c] * g[c];
    s1 += dxh;
    s2 += dxh * (x[off + c] - mu) * r;
  }
  s1 = warp_sum(s1) / cols;
  s2 = warp_sum(s2) / cols;
  for (int c = lane; c < cols; c += 32) {
    const float xh = (x[off + c] - mu) * r;
    dx[off + c] = (resid ? resid[off + c] : 0.f) + r * (dy[off + c] * g[c] - s1 - xh * s2);
  }
}

// dgamma[c] += sum_r dy * xhat, dbeta[c] += sum_r dy: one thread per column, rows in order.
__global__ void f32_ln_bwd_dgb_kernel(const float* __restrict__ dy, const float* __restrict__ x,
                                      const float* __restrict__ mean, const float* __restrict__ rstd, float* dgamma,
                                      float* dbeta, int rows, int cols) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float sg = 0.f, sb = 0.f;
  for (int r = 0; r < rows; ++r) {
    const float d = dy[static_cast<size_t>(r) * cols + c];
    sg += d * (x[static_cast<size_t>(r) * cols + c] - mean[r]) * rstd[r];
    sb += d;
  }
  dgamma[c] += sg;
  dbeta[c] += sb;
}

// ---------------------------------------------------------------- attention (warp per row)
// qkv row t = [q (H*D) | k (H*D) | v (H*D)], head-major; o / do [T][H*D]; lse natural log.
// Each warp owns one query (forward, dQ) or one key (dK / dV) of one (sequence, head); lanes
// split head_dim (D <= 128: 4 elements per lane).
constexpr int FA_MAXV = 4;
struct Heads {
  const float* qkv;
  int S, H, D, causal;
  float scale;
  const int32_t* key_len;  // per sequence valid key count (key padding), or null
  __device__ int kend(int b, int qi) const { return causal ? qi + 1 : (key_len ? key_len[b] : S); }
  __device__ const float* q(int b, int s, int h) const { return qkv + (static_cast<size_t>(b) * S + s) * 3 * H * D + h * D; }
  __device__ const float* k(int b, int s, int h) const { return q(b, s, h) + H * D; }
  __device__ const float* v(int b, int s, int h) const { return q(b, s, h) + 2 * H * D; }
};
__device__ __forceinline__ float dot_lanes(const float* a, const float* b, int D, int lane) {
  float s = 0.f;
  for (int d = lane; d < D; d += 32) s += a[d] * b[d];
  return warp_sum(s);
}

__global__ void f32_attn_fwd_kernel(Heads hd, float* __restrict__ o, float* __restrict__ lse, int B) {
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int S = hd.S, H = hd.H, D = hd.D;
  if (gw >= B * H * S) return;
  const int qi = gw % S, h = (gw / S) % H, b = gw / (S * H);
  const float* q = hd.q(b, qi, h);
  const int kend = hd.kend(b, qi);
  float m = -INFINITY;
  for (int k = 0; k < kend; ++k) m = fmaxf(m, hd.scale * dot_lanes(q, hd.k(b, k, h), D, lane));
  float l = 0.f, acc[FA_MAXV] = {0, 0, 0, 0};
  for (int k = 0; k < kend; ++k) {
    const float p = expf(hd.scale * dot_lanes(q, hd.k(b, k, h), D, lane) - m);
    l += p;
    const float* vv = hd.v(b, k, h);
#pragma unroll
    for (int e = 0; e < FA_MAXV; ++e)
      if (lane + 32 * e < D) acc[e] += p * vv[lane + 32 * e];
  }
  float* orow = o + (static_cast<size_t>(b) * S + qi) * H * D + h * D;
#pragma unroll
  for (int e = 0; e < FA_MAXV; ++e)
    if (lane + 32 * e < D) orow[lane + 32 * e] = acc[e] / l;
  if (lane == 0) lse[(static_cast<size_t>(b) * H + h) * S + qi] = m + logf(l);
}

__device__ __forceinline__ float attn_p(const Heads& hd, const float* lse, int b, int h, int qi, int k, int lane) {
  return expf(hd.scale * dot_lanes(hd.q(b, qi, h), hd.k(b, k, h), hd.D, lane) -
              lse[(static_cast<size_t>(b) * hd.H + h) * hd.S + qi]);
}

// delta[q] = sum_d dO * O  (per (b, h, q))
__global__ void f32_attn_delta_kernel(const float* __restrict__ o, const float* __restrict__ dout, float* __restrict__ delta,
                                      int B, int S, int H, int D) {
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (gw >= B * H * S) return;
  const int qi = gw % S, h = (gw / S) % H, b = gw / (S * H);
  const size_t off = (static_cast<size_t>(b) * S + qi) * H * D + h * D;
  const float s = dot_lanes(o + off, dout + off, D, lane);
  if (lane == 0) delta[(static_cast<size_t>(b) * H + h) * S + qi] = s;
}

__global__ void f32_attn_dq_kernel(Heads hd, const float* __restrict__ dout, const float* __restrict__ lse,
                                   const float* __restrict__ delta, float* __restrict__ dqkv, int B) {
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int S = hd.S, H = hd.H, D = hd.D;
  if (gw >= B * H * S) return;
  const int qi = gw % S, h = (gw / S) % H, b = gw / (S * H);
  const float* dO = dout + (static_cast<size_t>(b) * S + qi) * H * D + h * D;
  const float dl = delta[(static_cast<size_t>(b) * H + h) * S + qi];
  const int kend = hd.kend(b, qi);
  float acc[FA_MAXV] = {0, 0, 0, 0};
  for (int k = 0; k < kend; ++k) {
    const float p = attn_p(hd, lse, b, h, qi, k, lane);
    const float ds = p * (dot_lanes(dO, hd.v(b, k, h), D, lane) - dl) * hd.scale;
    const float* kk = hd.k(b, k, h);
#pragma unroll
    for (int e = 0; e < FA_MAXV; ++e)
      if (lane + 32 * e < D) acc[e] += ds * kk[lane + 32 * e];
  }
  float* dq = dqkv + (static_cast<size_t>(b) * S + qi) * 3 * H * D + h * D;
#pragma unroll
  for (int e = 0; e < FA_MAXV; ++e)
    if (lane + 32 * e < D) dq[lane + 32 * e] = acc[e];
}

__global__ void f32_attn_dkdv_kernel(Heads hd, const float* __restrict__ dout, const float* __restrict__ lse,
                                     const float* __restrict__ delta, float* __restrict__ dqkv, int B) {
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int S = hd.S, H = hd.H, D = hd.D;
  if (gw >= B * H * S) return;
  const int ki = gw % S, h = (gw / S) % H, b = gw / (S * H);
  float dk[FA_MAXV] = {0, 0, 0, 0}, dv[FA_MAXV] = {0, 0, 0, 0};
  const bool pad = !hd.causal && hd.key_len && ki >= hd.key_len[b];  // a padding key: no gradient
  for (int qi = hd.causal ? ki : 0; qi < S && !pad; ++qi) {
    const float p = attn_p(hd, lse, b, h, qi, ki, lane);
    const float* dO = dout + (static_cast<size_t>(b) * S + qi) * H * D + h * D;
    const float dl = delta[(static_cast<size_t>(b) * H + h) * S + qi];
    const float ds = p * (dot_lanes(dO, hd.v(b, ki, h), D, lane) - dl) * hd.scale;
    const float* q = hd.q(b, qi, h);
#pragma unroll
    for (int e = 0; e < FA_MAXV; ++e)
      if (lane + 32 * e < D) {
        dv[e] += p * dO[lane + 32 * e];
        dk[e] += ds * q[lane + 32 * e];
      }
  }
  float* row = dqkv + (static_cast<size_t>(b) * S + ki) * 3 * H * D + h * D;
#pragma unroll
  for (int e = 0; e < FA_MAXV; ++e)
    if (lane + 32 * e < D) {
      row[H * D + lane + 32 * e] = dk[e];
      row[2 * H * D + lane + 32 * e] = dv[e];
    }
}

// ---------------------------------------------------------------- embedding / cross-entropy
__global__ void f32_embed_fwd_kernel(const int32_t* __restrict__ tok, const float* __restrict__ wte,
                                     const float* __restrict__ wpe, float* __restrict__ x, int ntok, int seq, int h) {
  const int64_t n = static_cast<int64_t>(ntok) * h;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(i / h), c = static_cast<int>(i % h);
    x[i] = wte[static_cast<size_t>(tok[t]) * h + c] + wpe[static_cast<size_t>(t % seq) * h + c];
  }
}

// dwte over the sorted (token, position) keys: each run summed in position order.
__global__ void f32_embed_bwd_tok_kernel(const uint32_t* __restrict__ sorted, const float* __restrict__ dx,
                                         float* __restrict__ dwte, int ntok, int h) {
  const int64_t n = static_cast<int64_t>(ntok) * h;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i / h), c = static_cast<int>(i % h);
    const uint32_t t = sorted[k] >> kEmbPosBits;
    if (k > 0 && (sorted[k - 1] >> kEmbPosBits) == t) continue;
    float acc = 0.f;
    for (int r = k; r < ntok && (sorted[r] >> kEmbPosBits) == t; ++r)
      acc += dx[static_cast<size_t>(sorted[r] & ((1u << kEmbPosBits) - 1)) * h + c];
    dwte[static_cast<size_t>(t) * h + c] += acc;
  }
}

__global__ void f32_embed_bwd_pos_kernel(const float* __restrict__ dx, float* __restrict__ dwpe, int ntok, int seq, int h) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= seq * h) return;
  const int p = i / h, c = i % h;
  float acc = 0.f;
  for (int b = 0; b < ntok / seq; ++b) acc += dx[(static_cast<size_t>(b) * seq + p) * h + c];
  dwpe[i] += acc;
}

__global__ void f32_xent_kernel(float* logits, const int32_t* __restrict__ labels, float* __restrict__ row_loss,
                                int vocab, int ld, float scale) {
  __shared__ float red[32];
  __shared__ float bcast;
  const int row = blockIdx.x;
  float* lr = logits + static_cast<size_t>(row) * ld;
  const int label = labels[row];
  auto block_reduce = [&](float v, bool is_max) {
    v = is_max ? warp_max(v) : warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = red[0];
      for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) t = is_max ? fmaxf(t, red[w]) : t + red[w];
      bcast = t;
    }
    __syncthreads();
    const float r = bcast;
    __syncthreads();
    return r;
  };
  float m = -INFINITY;
  for (int v = threadIdx.x; v < vocab; v += blockDim.x) m = fmaxf(m, lr[v]);
  m = block_reduce(m, true);
  float s = 0.f;
  for (int v = threadIdx.x; v < vocab; v += blockDim.x) s += expf(lr[v] - m);
  s = block_reduce(s, false);
  const float lse = m + logf(s);
  if (threadIdx.x == 0) row_loss[row] = label >= 0 ? lse - lr[label] : 0.f;
  __syncthreads();
  for (int v = threadIdx.x; v < vocab; v += blockDim.x)
    lr[v] = label >= 0 ? scale * (expf(lr[v] - lse) - (v == label ? 1.f : 0.f)) : 0.f;
}

__global__ void f32_sum_rows_kernel(const float* __restrict__ row_loss, int n, float* loss_sum) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    float s = 0.f;
    for (int i = 0; i < n; ++i) s += row_loss[i];
    loss_sum[0] += s;
  }
}

int warps_grid(int64_t warps, int per_block = 8) { return static_cast<int>((warps + per_block - 1) / per_block); }

}  // namespace
}  // namespace amdp

using namespace amdp;

extern "C" int amdp_f32_gemm(const amdp_gemm_args* a, amdp_stream_t stream) {
  if (!a || a->M <= 0 || a->N <= 0 || a->K <= 0) return AMDP_ERR_INVALID;
  if ((a->epilogue == AMDP_EPI_RESIDUAL || a->epilogue == AMDP_EPI_GELU_BWD) && !a->aux) return AMDP_ERR_INVALID;
  if (a->epilogue == AMDP_EPI_GELU && !a->C2) return AMDP_ERR_INVALID;
  if (a->epilogue == AMDP_EPI_ROWDOT) return AMDP_ERR_INVALID;
  const dim3 grid((a->N + FT - 1) / FT, (a->M + FT - 1) / FT);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  auto A = static_cast<const float*>(a->A);
  auto B = static_cast<const float*>(a->B);
  auto C = static_cast<float*>(a->C);
  auto X = static_cast<const float*>(a->aux);
  auto C2 = static_cast<float*>(a->C2);
#define F32_GEMM(AM, BM) \
  f32_gemm_kernel<AM, BM><<<grid, 256, 0, s>>>(a->M, a->N, a->K, A, a->lda, B, a->ldb, C, a->ldc, X, a->ld_aux, C2, a->ldc2, a->epilogue, a->alpha)
  if (a->a_mn_major && a->b_mn_major) F32_GEMM(true, true);
  else if (a->a_mn_major) F32_GEMM(true, false);
  else if (a->b_mn_major) F32_GEMM(false, true);
  else F32_GEMM(false, false);
#undef F32_GEMM
  return cudaGetLastError();
}

extern "C" int amdp_f32_layernorm_fwd(const float* x, const float* gamma, const float* beta, float* y, float* mean,
                                      float* rstd, int rows, int cols, float eps, amdp_stream_t stream) {
  if (rows <= 0 || cols <= 0) return AMDP_ERR_INVALID;
  f32_ln_fwd_kernel<<<warps_grid(rows), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(x, gamma, beta, y, mean, rstd,
                                                                                          rows, cols, eps);
  return cudaGetLastError();
}

extern "C" int amdp_f32_layernorm_bwd(const float* dy, const float* x, const float* gamma, const float* mean,
                                      const float* rstd, const float* resid_grad, float* dx, float* dgamma,
                                      float* dbeta, int rows, int cols, amdp_stream_t stream) {
  if (rows <= 0 || cols <= 0) return AMDP_ERR_INVALID;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  f32_ln_bwd_dgb_kernel<<<(cols + 255) / 256, 256, 0, s>>>(dy, x, mean, rstd, dgamma, dbeta, rows, cols);
  f32_ln_bwd_dx_kernel<<<warps_grid(rows), 256, 0, s>>>(dy, x, gamma, mean, rstd, resid_grad, dx, rows, cols);
  return cudaGetLastError();
}

extern "C" int amdp_f32_attention_fwd(const float* qkv, float* out, float* lse, int batch, int seq, int heads,
                                      int head_dim, int causal, const int32_t* key_len, amdp_stream_t stream) {
  if (batch <= 0 || seq <= 0 || heads <= 0 || head_dim <= 0 || head_dim > 32 * FA_MAXV) return AMDP_ERR_INVALID;
  if (causal && key_len) return AMDP_ERR_UNSUPPORTED;
  Heads hd{qkv, seq, heads, head_dim, causal, 1.f / sqrtf(static_cast<float>(head_dim)), key_len};
  f32_attn_fwd_kernel<<<warps_grid(static_cast<int64_t>(batch) * heads * seq), 256, 0,
                        reinterpret_cast<cudaStream_t>(stream)>>>(hd, out, lse, batch);
  return cudaGetLastError();
}

extern "C" size_t amdp_f32_attention_bwd_workspace(int batch, int seq, int heads) {
  return static_cast<size_t>(batch) * heads * seq * sizeof(float);
}

extern "C" int amdp_f32_attention_bwd(const float* qkv, const float* out, const float* dout, const float* lse,
                                      float* dqkv, float* workspace, int batch, int seq, int heads, int head_dim,
                                      int causal, const int32_t* key_len, amdp_stream_t stream) {
  if (batch <= 0 || seq <= 0 || heads <= 0 || head_dim <= 0 || head_dim > 32 * FA_MAXV || !workspace)
    return AMDP_ERR_INVALID;
  if (causal && key_len) return AMDP_ERR_UNSUPPORTED;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Heads hd{qkv, seq, heads, head_dim, causal, 1.f / sqrtf(static_cast<float>(head_dim)), key_len};
  const int g = warps_grid(static_cast<int64_t>(batch) * heads * seq);
  f32_attn_delta_kernel<<<g, 256, 0, s>>>(out, dout, workspace, batch, seq, heads, head_dim);
  f32_attn_dq_kernel<<<g, 256, 0, s>>>(hd, dout, lse, workspace, dqkv, batch);
  f32_attn_dkdv_kernel<<<g, 256, 0, s>>>(hd, dout, lse, workspace, dqkv, batch);
  return cudaGetLastError();
}

extern "C" int amdp_f32_embedding_fwd(const int32_t* tokens, const float* wte, const float* wpe, float* x, int ntok,
                                      int seq, int hidden, amdp_stream_t stream) {
  if (ntok <= 0 || seq <= 0 || hidden <= 0) return AMDP_ERR_INVALID;
  const int64_t n = static_cast<int64_t>(ntok) * hidden;
  f32_embed_fwd_kernel<<<static_cast<int>(std::min<int64_t>((n + 255) / 256, 16 * 148)), 256, 0,
                         reinterpret_cast<cudaStream_t>(stream)>>>(tokens, wte, wpe, x, ntok, seq, hidden);
  return cudaGetLastError();
}

extern "C" int amdp_f32_embedding_bwd(const int32_t* tokens, const float* dx, float* dwte, float* dwpe, void* workspace,
                                      int ntok, int seq, int hidden, amdp_stream_t stream) {
  if (ntok <= 0 || seq <= 0 || hidden <= 0 || ntok % seq != 0 || !workspace || ntok > (1 << kEmbPosBits))
    return AMDP_ERR_INVALID;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int n2 = 1;
  while (n2 < ntok) n2 <<= 1;
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    cudaError_t e = cudaFuncSetAttribute(embedding_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sizeof(uint32_t) << kEmbPosBits));
    if (e != cudaSuccess) {
      attr.store(0);
      return e;
    }
  }
  uint32_t* sorted = static_cast<uint32_t*>(workspace);
  embedding_sort_kernel<<<1, 1024, static_cast<size_t>(n2) * sizeof(uint32_t), s>>>(tokens, ntok, sorted);
  const int64_t n = static_cast<int64_t>(ntok) * hidden;
  f32_embed_bwd_tok_kernel<<<static_cast<int>(std::min<int64_t>((n + 255) / 256, 16 * 148)), 256, 0, s>>>(
      sorted, dx, dwte, ntok, hidden);
  f32_embed_bwd_pos_kernel<<<(seq * hidden + 255) / 256, 256, 0, s>>>(dx, dwpe, ntok, seq, hidden);
  return cudaGetLastError();
}

extern "C" int amdp_f32_xent_fwd_bwd(float* logits, const int32_t* labels, float* loss_sum, float* row_loss, int ntok,
                                     int vocab, int ld, float scale, amdp_stream_t stream) {
  if (ntok <= 0 || vocab <= 0 || ld < vocab || !row_loss) return AMDP_ERR_INVALID;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  f32_xent_kernel<<<ntok, 512, 0, s>>>(logits, labels, row_loss, vocab, ld, scale);
  f32_sum_rows_kernel<<<1, 32, 0, s>>>(row_loss, ntok, loss_sum);
  return cudaGetLastError();
}
