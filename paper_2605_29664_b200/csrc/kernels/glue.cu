// Memory-bound stage glue: LayerNorm fwd/bwd, token+position embedding fwd/bwd,
// fused softmax cross-entropy (loss + dlogits in one pass pair).
// All are HBM-bound: 16-byte vector accesses, one warp per row (LayerNorm) or one
// CTA per row (cross-entropy over the vocabulary), warp-shuffle reductions, grids
// sized in multiples of the SM count.
#include "common.cuh"

namespace amdp {
namespace {

constexpr int LN_MAX_VEC = 12;  // up to 12 x 256 = 3072 columns per row

__device__ __forceinline__ void unpack8(const uint4& q, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 t = __bfloat1622float2(h[e]);
    f[2 * e] = t.x;
    f[2 * e + 1] = t.y;
  }
}

// ---------------------------------------------------------------- LayerNorm forward
// One warp per row; the row is held in registers as raw bf16 (4 registers per 8 columns,
// NV = ceil(cols / 256) chunks per lane), so HBM is read once and written once.
template <int NV>
__global__ void __launch_bounds__(256) layernorm_fwd_kernel(
    const bf16* __restrict__ x, const float* __restrict__ gamma, const float* __restrict__ beta,
    bf16* __restrict__ y, float* __restrict__ mean_out, float* __restrict__ rstd_out, int rows,
    int cols, float eps) {
  grid_dep_wait();  // PDL: predecessor's outputs visible from here
  grid_dep_trigger();
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  for (int row = blockIdx.x * warps + (threadIdx.x >> 5); row < rows; row += gridDim.x * warps) {
    const bf16* xr = x + static_cast<size_t>(row) * cols;
    uint4 raw[NV];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 8;
      if (c < cols) raw[i] = *reinterpret_cast<const uint4*>(xr + c);
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 8;
      if (c < cols) {
        float v[8];
        unpack8(raw[i], v);
#pragma unroll
        for (int e = 0; e < 8; ++e) s += v[e];
      }
    }
    const float mean = warp_sum(s) / cols;
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 8;
      if (c < cols) {
        float v[8];
        unpack8(raw[i], v);
#pragma unroll
        for (int e = 0; e < 8; ++e) ss += (v[e] - mean) * (v[e] - mean);
      }
    }
    const float rstd = rsqrtf(warp_sum(ss) / cols + eps);
    bf16* yr = y + static_cast<size_t>(row) * cols;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 8;
      if (c < cols) {
        float v[8], o[8];
        unpack8(raw[i], v);
        const float4 g0 = *reinterpret_cast<const float4*>(gamma + c);
        const float4 g1 = *reinterpret_cast<const float4*>(gamma + c + 4);
        const float4 b0 = *reinterpret_cast<const float4*>(beta + c);
        const float4 b1 = *reinterpret_cast<const float4*>(beta + c + 4);
        const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = (v[e] - mean) * rstd * g[e] + b[e];
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
// Two fully parallel kernels (no serial fold):
//  dx  : one warp per row: s1 = mean(dy*g), s2 = mean(dy*g*xhat), then
//        dx = resid + rstd * (dy*g - s1 - xhat*s2)   (second pass re-reads the row from L1)
//  dg/db: a CTA owns 256 columns x 64 rows; each lane accumulates 8 columns over its
//        warp's rows, the 8 warps combine in smem and add into the fp32 gradient buffer.
template <int NV>
__global__ void __launch_bounds__(256) layernorm_bwd_dx_kernel(
    const bf16* __restrict__ dy, const bf16* __restrict__ x, const float* __restrict__ gamma,
    const float* __restrict__ mean_in, const float* __restrict__ rstd_in, const bf16* resid_grad,
    bf16* dx, int rows, int cols) {
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  for (int row = blockIdx.x * warps + (threadIdx.x >> 5); row < rows; row += gridDim.x * warps) {
    const size_t off = static_cast<size_t>(row) * cols;
    const float mean = mean_in[row], rstd = rstd_in[row];
    uint4 xr[NV], dr[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 8;
      if (c < cols) {
        xr[i] = *reinterpret_cast<const uint4*>(x + off + c);
        dr[i] = *reinterpret_cast<const uint4*>(dy + off + c);
      }
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 8;
      if (c < cols) {
        float xv[8], dv[8];
        unpack8(xr[i], xv);
        unpack8(dr[i], dv);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float dxh = dv[e] * gamma[c + e];
          s1 += dxh;
          s2 += dxh * (xv[e] - mean) * rstd;
        }
      }
    }
    s1 = warp_sum(s1) / cols;
    s2 = warp_sum(s2) / cols;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 8;
      if (c < cols) {
        float xv[8], dv[8], o[8];
        float r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        unpack8(xr[i], xv);
        unpack8(dr[i], dv);
        if (resid_grad) load8(resid_grad + off + c, r);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          o[e] = r[e] + rstd * (dv[e] * gamma[c + e] - s1 - (xv[e] - mean) * rstd * s2);
        store8(dx + off + c, o);
      }
    }
  }
}

constexpr int LN_DG_ROWS = 64;
__global__ void __launch_bounds__(256) layernorm_bwd_dgb_kernel(
    const bf16* __restrict__ dy, const bf16* __restrict__ x, const float* __restrict__ mean_in,
    const float* __restrict__ rstd_in, float* __restrict__ part, int rows, int cols) {
  // per-(row block) partials [gridDim.y][2][cols], summed in a fixed order by
  // layernorm_dgb_reduce_kernel: deterministic (no atomics)
  __shared__ float red[8][2][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * 256 + lane * 8;
  const int r0 = blockIdx.y * LN_DG_ROWS;
  float g[8] = {0, 0, 0, 0, 0, 0, 0, 0}, bb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (c < cols) {
    for (int row = r0 + warp; row < min(rows, r0 + LN_DG_ROWS); row += 8) {
      const size_t off = static_cast<size_t>(row) * cols + c;
      const float mean = mean_in[row], rstd = rstd_in[row];
      float xv[8], dv[8];
      load8(x + off, xv);
      load8(dy + off, dv);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        g[e] += dv[e] * (xv[e] - mean) * rstd;
        bb[e] += dv[e];
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    red[warp][0][lane * 8 + e] = g[e];
    red[warp][1][lane * 8 + e] = bb[e];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 512; i += 256) {
    const int which = i >> 8, col = i & 255;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[w][which][col];
    const int gc = blockIdx.x * 256 + col;
    if (gc < cols) part[(static_cast<size_t>(blockIdx.y) * 2 + which) * cols + gc] = s;
  }
}

// ---------------------------------------------------------------- LayerNorm, row-group form
// Backward for the model widths (cols a multiple of 256, <= 4096): one thread per 8 columns, so a
// CTA of cols/8 threads spans a whole row and handles RG rows per iteration (RG 16-byte
// loads in flight per thread and per tensor).  Row statistics: warp shuffle, then the
// cols/256 warp partials through shared memory (double-buffered by iteration parity, so
// one __syncthreads per reduction).  The backward accumulates dgamma/dbeta for its 8
// columns in registers across all its rows and adds them once per CTA, so x and dy are
// read exactly once (dx, dgamma, dbeta fused: 4 bf16 tensors of traffic per row).
template <int RG>
__device__ __forceinline__ void block_sums(float (&v)[RG], float* red, int nw) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < RG; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < RG; ++i) red[i * 32 + w] = v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < RG; ++i) {
    float t = 0.f;
    for (int k = 0; k < nw; ++k) t += red[i * 32 + k];
    v[i] = t;
  }
}

template <int RG>
struct LnBwdRows {
  uint4 x[RG], d[RG], r[RG];
  float mu[RG], rs[RG];
  __device__ __forceinline__ void load(const bf16* __restrict__ x_, const bf16* __restrict__ dy,
                                       const bf16* resid, const float* __restrict__ mean_in,
                                       const float* __restrict__ rstd_in, int r0, int rows, int cols, int c) {
#pragma unroll
    for (int i = 0; i < RG; ++i) {
      const bool ok = r0 + i < rows;
      const size_t off = static_cast<size_t>(r0 + i) * cols + c;
      x[i] = ok ? *reinterpret_cast<const uint4*>(x_ + off) : make_uint4(0, 0, 0, 0);
      d[i] = ok ? *reinterpret_cast<const uint4*>(dy + off) : make_uint4(0, 0, 0, 0);
      r[i] = (ok && resid) ? *reinterpret_cast<const uint4*>(resid + off) : make_uint4(0, 0, 0, 0);
      mu[i] = ok ? mean_in[r0 + i] : 0.f;
      rs[i] = ok ? rstd_in[r0 + i] : 0.f;
    }
  }
};

// Software-pipelined over row groups: group k+1's loads are in flight while group k is
// reduced and written, so each CTA keeps 2 x RG rows x 3 tensors of loads outstanding.
template <int RG>
__global__ void __launch_bounds__(512) layernorm_bwd_rows_kernel(
    const bf16* __restrict__ dy, const bf16* __restrict__ x, const float* __restrict__ gamma,
    const float* __restrict__ mean_in, const float* __restrict__ rstd_in, const bf16* resid_grad, bf16* dx,
    float* __restrict__ part, int rows, int cols, int accumulate) {
  grid_dep_wait();  // PDL: predecessor's outputs visible from here
  grid_dep_trigger();
  __shared__ float red[2][2 * RG * 32];
  const int nw = blockDim.x >> 5;
  const int c = threadIdx.x * 8;
  float g[8], ag[8], ab[8];
  {
    const float4 g0 = *reinterpret_cast<const float4*>(gamma + c), g1 = *reinterpret_cast<const float4*>(gamma + c + 4);
    g[0] = g0.x; g[1] = g0.y; g[2] = g0.z; g[3] = g0.w; g[4] = g1.x; g[5] = g1.y; g[6] = g1.z; g[7] = g1.w;
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) ag[e] = ab[e] = 0.f;
  const float inv = 1.f / static_cast<float>(cols);
  const int stride = gridDim.x * RG;
  LnBwdRows<RG> cur, nxt;
  int r0 = blockIdx.x * RG;
  if (r0 < rows) cur.load(x, dy, resid_grad, mean_in, rstd_in, r0, rows, cols, c);
  for (int it = 0; r0 < rows; r0 += stride, it ^= 1) {
    if (r0 + stride < rows) nxt.load(x, dy, resid_grad, mean_in, rstd_in, r0 + stride, rows, cols, c);
    float sv[2 * RG];
#pragma unroll
    for (int i = 0; i < RG; ++i) {
      float xv[8], dv[8];
      unpack8(cur.x[i], xv);
      unpack8(cur.d[i], dv);
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float xh = (xv[e] - cur.mu[i]) * cur.rs[i];
        const float dxh = dv[e] * g[e];
        s1 += dxh;
        s2 += dxh * xh;
        ag[e] += dv[e] * xh;
        ab[e] += dv[e];
      }
      sv[2 * i] = s1;
      sv[2 * i + 1] = s2;
    }
    block_sums<2 * RG>(sv, red[it], nw);
#pragma unroll
    for (int i = 0; i < RG; ++i) {
      if (r0 + i >= rows) break;
      const float s1 = sv[2 * i] * inv, s2 = sv[2 * i + 1] * inv;
      float xv[8], dv[8], r[8], o[8];
      unpack8(cur.x[i], xv);
      unpack8(cur.d[i], dv);
      unpack8(cur.r[i], r);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        o[e] = r[e] + cur.rs[i] * (dv[e] * g[e] - s1 - (xv[e] - cur.mu[i]) * cur.rs[i] * s2);
      store8(dx + static_cast<size_t>(r0 + i) * cols + c, o);
    }
    cur = nxt;
  }
  // per-CTA column partials -> workspace row blockIdx.x: [dgamma cols | dbeta cols]; with
  // `accumulate` added to the row (the deferred form: one CTA index always owns one row, and
  // the launches on a stream are ordered, so the sums are deterministic)
  float* wrow = part + static_cast<size_t>(blockIdx.x) * 2 * cols;
  if (accumulate) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      ag[e] += wrow[c + e];
      ab[e] += wrow[cols + c + e];
    }
  }
  *reinterpret_cast<float4*>(wrow + c) = make_float4(ag[0], ag[1], ag[2], ag[3]);
  *reinterpret_cast<float4*>(wrow + c + 4) = make_float4(ag[4], ag[5], ag[6], ag[7]);
  *reinterpret_cast<float4*>(wrow + cols + c) = make_float4(ab[0], ab[1], ab[2], ab[3]);
  *reinterpret_cast<float4*>(wrow + cols + c + 4) = make_float4(ab[4], ab[5], ab[6], ab[7]);
}

// dgamma, dbeta += column sums of the [nparts][2*cols] partials ([dgamma | dbeta] per row).
// CTA = 32 columns x 32 row-lanes (each lane sums ~nparts/32 rows, all loads independent), a
// fixed-order tree over the 32 lanes: deterministic, and short enough that the kernel is not
// latency-bound (the 8-lane version spent ~9 us on 4.8 MB).
__global__ void __launch_bounds__(1024) layernorm_dgb_reduce_kernel(float* __restrict__ part, int nparts,
                                                                    int cols, float* dgamma, float* dbeta,
                                                                    int clear) {
  grid_dep_wait();  // PDL: predecessor's outputs visible from here
  grid_dep_trigger();
  __shared__ float red[32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int col = blockIdx.x * 32 + lane;  // in [0, 2*cols)
  float s = 0.f;
  if (col < 2 * cols) {
#pragma unroll 4
    for (int r = w; r < nparts; r += 32) s += part[static_cast<size_t>(r) * 2 * cols + col];
    if (clear)  // deferred form: the partial rows start the next window at zero
      for (int r = w; r < nparts; r += 32) part[static_cast<size_t>(r) * 2 * cols + col] = 0.f;
  }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 32; ++k) t += red[k][lane];
    if (col < 2 * cols) {
      if (col < cols) dgamma[col] += t;
      else dbeta[col - cols] += t;
    }
  }
}

// ---------------------------------------------------------------- embedding
__global__ void embedding_fwd_kernel(const int32_t* __restrict__ tok, const bf16* __restrict__ wte,
                                     const bf16* __restrict__ wpe, bf16* __restrict__ x, int ntok,
                                     int seq, int hidden) {
  grid_dep_wait();  // PDL: predecessor's outputs visible from here
  grid_dep_trigger();
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

// Deterministic token-table gradient: the minibatch's (token, position) keys are sorted in
// one CTA (bitonic, shared memory), then each run of equal tokens is summed in position order
// by the single thread owning that (token, 8-column) slice and added to dwte without atomics.
// The window gradient is therefore bitwise reproducible (and independent of how the stages are
// spread over GPUs).  Key = token << 14 | position: ntok <= 16384, vocab < 2^18.
__global__ void embedding_bwd_tok_kernel(const uint32_t* __restrict__ sorted, const bf16* __restrict__ dx,
                                         float* __restrict__ dwte, int ntok, int hidden) {
  grid_dep_wait();  // PDL: predecessor's outputs visible from here
  grid_dep_trigger();
  const int vecs = hidden / 8;
  const int64_t total = static_cast<int64_t>(ntok) * vecs;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i / vecs);
    const int c = static_cast<int>(i % vecs) * 8;
    const uint32_t t = sorted[k] >> kEmbPosBits;
    if (k > 0 && (sorted[k - 1] >> kEmbPosBits) == t) continue;  // not the run's first key
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // the run's end first (its keys share cache lines), then the rows in groups of 8 whose loads
    // are all in flight before the in-order adds: the same summation order as one row at a
    // time (bit-identical), without one dependent load per row (BERT's padding-token run of a
    // few hundred rows made this kernel 130 us)
    int end = k + 1;
    while (end < ntok && (sorted[end] >> kEmbPosBits) == t) ++end;
    constexpr uint32_t kPosMask = (1u << kEmbPosBits) - 1;
    int r = k;
    for (; r + 8 <= end; r += 8) {
      float g[8][8];
#pragma unroll
      for (int j = 0; j < 8; ++j) load8(dx + static_cast<size_t>(sorted[r + j] & kPosMask) * hidden + c, g[j]);
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += g[j][e];
    }
    for (; r < end; ++r) {
      float g[8];
      load8(dx + static_cast<size_t>(sorted[r] & kPosMask) * hidden + c, g);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += g[e];
    }
    float4* dst = reinterpret_cast<float4*>(dwte + static_cast<size_t>(t) * hidden + c);
    float4 a = dst[0], b = dst[1];
    a.x += acc[0]; a.y += acc[1]; a.z += acc[2]; a.w += acc[3];
    b.x += acc[4]; b.y += acc[5]; b.z += acc[6]; b.w += acc[7];
    dst[0] = a;
    dst[1] = b;
  }
}

__global__ void embedding_bwd_pos_kernel(const bf16* __restrict__ dx, float* dwpe, int ntok,
                                         int seq, int hidden) {
  grid_dep_wait();  // PDL: predecessor's outputs visible from here
  grid_dep_trigger();
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
                                                   float* __restrict__ row_loss, int vocab, int ld,
                                                   float scale) {
  grid_dep_wait();  // PDL: predecessor's outputs visible from here
  grid_dep_trigger();
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
    row_loss[row] = label >= 0 ? lse - __bfloat162float(lr[label]) : 0.f;
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

// loss_sum[0] += sum of the rows' losses in a fixed order (one CTA): deterministic.
__global__ void __launch_bounds__(1024) sum_rows_kernel(const float* __restrict__ row_loss, int n,
                                                        float* loss_sum) {
  grid_dep_wait();
  grid_dep_trigger();
  __shared__ float part[32];
  float s = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += row_loss[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) loss_sum[0] += t;
  }
}

}  // namespace
}  // namespace amdp

using namespace amdp;

// The row-group LayerNorm kernels cover widths that are whole warps of 8-column threads.
static bool ln_row_group_form(int cols) {
  static const int off = getenv("AMDP_LN_WARP_ROWS") ? atoi(getenv("AMDP_LN_WARP_ROWS")) : 0;
  return !off && cols % 256 == 0 && cols >= 256 && cols / 8 <= 512;
}

namespace amdp {
namespace {
__global__ void gelu_fwd_kernel(const bf16* __restrict__ u, bf16* __restrict__ f, int64_t n8) {
  grid_dep_wait();
  grid_dep_trigger();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float v[8];
    load8(u + i * 8, v);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = gelu_tanh_bf16in(v[e]);  // same bits as the fc1 epilogue
    store8(f + i * 8, v);
  }
}
}  // namespace
}  // namespace amdp

extern "C" int amdp_gelu_fwd(const uint16_t* u, uint16_t* f, int64_t n, amdp_stream_t stream) {
  using namespace amdp;
  if (n <= 0 || n % 8 != 0) return AMDP_ERR_INVALID;
  const int64_t n8 = n / 8;
  const int blocks = static_cast<int>(std::min<int64_t>((n8 + 255) / 256, 8 * num_sms()));
  launch_pdl(gelu_fwd_kernel, dim3(blocks), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream),
             reinterpret_cast<const bf16*>(u), reinterpret_cast<bf16*>(f), n8);
  return cudaGetLastError();
}

extern "C" int amdp_layernorm_fwd(const uint16_t* x, const float* gamma, const float* beta,
                                  uint16_t* y, float* mean, float* rstd, int rows, int cols,
                                  float eps, amdp_stream_t stream) {
  if (rows <= 0 || cols <= 0 || cols % 8 != 0 || cols > LN_MAX_VEC * 256) return AMDP_ERR_INVALID;
  const int warps_needed = rows;
  int blocks = (warps_needed + 7) / 8;
  const int cap = 8 * num_sms();
  if (blocks > cap) blocks = cap;
  auto xs = reinterpret_cast<const bf16*>(x);
  auto ys = reinterpret_cast<bf16*>(y);
  auto st = reinterpret_cast<cudaStream_t>(stream);
  const int nv = (cols + 255) / 256;
  if (nv <= 1) launch_pdl(layernorm_fwd_kernel<1>, dim3(blocks), dim3(256), 0, st, xs, gamma, beta, ys, mean, rstd, rows, cols, eps);
  else if (nv <= 4) launch_pdl(layernorm_fwd_kernel<4>, dim3(blocks), dim3(256), 0, st, xs, gamma, beta, ys, mean, rstd, rows, cols, eps);
  else if (nv <= 8) launch_pdl(layernorm_fwd_kernel<8>, dim3(blocks), dim3(256), 0, st, xs, gamma, beta, ys, mean, rstd, rows, cols, eps);
  else launch_pdl(layernorm_fwd_kernel<LN_MAX_VEC>, dim3(blocks), dim3(256), 0, st, xs, gamma, beta, ys, mean, rstd, rows, cols, eps);
  return cudaGetLastError();
}

// Row-group backward: per-CTA dgamma/dbeta partials, [ln_bwd_ctas][2][cols] fp32.
static int ln_bwd_ctas(int rows) {
  constexpr int RG = 2;
  static const int per_sm = getenv("AMDP_LN_BWD_CTAS") ? atoi(getenv("AMDP_LN_BWD_CTAS")) : 2;
  const int grid = (rows + RG - 1) / RG;
  const int cap = per_sm * num_sms();  // one resident wave (128 registers x cols/8 threads)
  return grid < cap ? grid : cap;
}

extern "C" size_t amdp_layernorm_bwd_workspace(int rows, int cols) {
  if (rows <= 0 || cols <= 0) return 16;
  const int parts = std::max(ln_bwd_ctas(rows), (rows + LN_DG_ROWS - 1) / LN_DG_ROWS);
  return static_cast<size_t>(parts) * 2 * cols * sizeof(float) + 16;
}

extern "C" int amdp_layernorm_bwd(const uint16_t* dy, const uint16_t* x, const float* gamma,
                                  const float* mean, const float* rstd,
                                  const uint16_t* resid_grad, uint16_t* dx, float* dgamma,
                                  float* dbeta, void* workspace, int rows, int cols,
                                  amdp_stream_t stream) {
  if (rows <= 0 || cols <= 0 || cols % 8 != 0 || cols > LN_MAX_VEC * 256) return AMDP_ERR_INVALID;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!workspace) return AMDP_ERR_INVALID;
  if (ln_row_group_form(cols)) {
    const int grid = ln_bwd_ctas(rows);
    float* part = static_cast<float*>(workspace);
    launch_pdl(layernorm_bwd_rows_kernel<2>, dim3(grid), dim3(cols / 8), 0, s, 
        reinterpret_cast<const bf16*>(dy), reinterpret_cast<const bf16*>(x), gamma, mean, rstd,
        reinterpret_cast<const bf16*>(resid_grad), reinterpret_cast<bf16*>(dx), part, rows, cols, 0);
    launch_pdl(layernorm_dgb_reduce_kernel, dim3((2 * cols + 31) / 32), dim3(1024), 0, s, part, grid, cols, dgamma, dbeta, 0);
    return cudaGetLastError();
  }
  int blocks = (rows + 7) / 8;
  if (blocks > 8 * num_sms()) blocks = 8 * num_sms();
  {
    auto dys = reinterpret_cast<const bf16*>(dy);
    auto xs = reinterpret_cast<const bf16*>(x);
    auto rs = reinterpret_cast<const bf16*>(resid_grad);
    auto dxs = reinterpret_cast<bf16*>(dx);
    const int nv = (cols + 255) / 256;
    if (nv <= 1) layernorm_bwd_dx_kernel<1><<<blocks, 256, 0, s>>>(dys, xs, gamma, mean, rstd, rs, dxs, rows, cols);
    else if (nv <= 4) layernorm_bwd_dx_kernel<4><<<blocks, 256, 0, s>>>(dys, xs, gamma, mean, rstd, rs, dxs, rows, cols);
    else if (nv <= 8) layernorm_bwd_dx_kernel<8><<<blocks, 256, 0, s>>>(dys, xs, gamma, mean, rstd, rs, dxs, rows, cols);
    else layernorm_bwd_dx_kernel<LN_MAX_VEC><<<blocks, 256, 0, s>>>(dys, xs, gamma, mean, rstd, rs, dxs, rows, cols);
  }
  dim3 g((cols + 255) / 256, (rows + LN_DG_ROWS - 1) / LN_DG_ROWS);
  float* part = static_cast<float*>(workspace);
  layernorm_bwd_dgb_kernel<<<g, 256, 0, s>>>(reinterpret_cast<const bf16*>(dy),
                                             reinterpret_cast<const bf16*>(x), mean, rstd, part, rows, cols);
  launch_pdl(layernorm_dgb_reduce_kernel, dim3((2 * cols + 31) / 32), dim3(1024), 0, s, part,
             static_cast<int>(g.y), cols, dgamma, dbeta, 0);
  return cudaGetLastError();
}

// Deferred parameter gradients: the window's LayerNorm backwards accumulate per-CTA partial
// rows (amdp_layernorm_bwd_rows) and one flush per window folds them into dgamma / dbeta —
// one column-reduction launch per window instead of one per minibatch.
extern "C" int amdp_layernorm_bwd_parts(int rows, int cols) {
  if (rows <= 0 || !ln_row_group_form(cols)) return 0;
  return ln_bwd_ctas(rows);
}

extern "C" int amdp_layernorm_bwd_rows(const uint16_t* dy, const uint16_t* x, const float* gamma, const float* mean,
                                       const float* rstd, const uint16_t* resid_grad, uint16_t* dx, float* part,
                                       int rows, int cols, amdp_stream_t stream) {
  if (rows <= 0 || cols <= 0 || !part) return AMDP_ERR_INVALID;
  if (!ln_row_group_form(cols)) return AMDP_ERR_UNSUPPORTED;
  launch_pdl(layernorm_bwd_rows_kernel<2>, dim3(ln_bwd_ctas(rows)), dim3(cols / 8), 0,
             reinterpret_cast<cudaStream_t>(stream), reinterpret_cast<const bf16*>(dy),
             reinterpret_cast<const bf16*>(x), gamma, mean, rstd, reinterpret_cast<const bf16*>(resid_grad),
             reinterpret_cast<bf16*>(dx), part, rows, cols, 1);
  return cudaGetLastError();
}

extern "C" int amdp_layernorm_dgb_flush(float* part, int nparts, int cols, float* dgamma, float* dbeta,
                                        amdp_stream_t stream) {
  if (!part || nparts <= 0 || cols <= 0) return AMDP_ERR_INVALID;
  launch_pdl(layernorm_dgb_reduce_kernel, dim3((2 * cols + 31) / 32), dim3(1024), 0,
             reinterpret_cast<cudaStream_t>(stream), part, nparts, cols, dgamma, dbeta, 1);
  return cudaGetLastError();
}

extern "C" int amdp_embedding_fwd(const int32_t* tokens, const uint16_t* wte, const uint16_t* wpe,
                                  uint16_t* x, int ntok, int seq, int hidden,
                                  amdp_stream_t stream) {
  if (ntok <= 0 || seq <= 0 || hidden % 8 != 0) return AMDP_ERR_INVALID;
  const int64_t work = static_cast<int64_t>(ntok) * (hidden / 8);
  int blocks = static_cast<int>((work + 255) / 256);
  if (blocks > 16 * num_sms()) blocks = 16 * num_sms();
  launch_pdl(embedding_fwd_kernel, dim3(blocks), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), 
      tokens, reinterpret_cast<const bf16*>(wte), reinterpret_cast<const bf16*>(wpe),
      reinterpret_cast<bf16*>(x), ntok, seq, hidden);
  return cudaGetLastError();
}

extern "C" int amdp_embedding_bwd(const int32_t* tokens, const uint16_t* dx, float* dwte,
                                  float* dwpe, void* workspace, int ntok, int seq, int hidden,
                                  amdp_stream_t stream) {
  if (ntok <= 0 || seq <= 0 || hidden % 8 != 0 || ntok % seq != 0 || !workspace) return AMDP_ERR_INVALID;
  if (ntok > (1 << kEmbPosBits)) return AMDP_ERR_INVALID;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int n2 = 1;
  while (n2 < ntok) n2 <<= 1;
  const size_t smem = static_cast<size_t>(n2) * sizeof(uint32_t);
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
  launch_pdl(embedding_sort_kernel, dim3(1), dim3(1024), smem, s, tokens, ntok, sorted);
  const int64_t work = static_cast<int64_t>(ntok) * (hidden / 8);
  int blocks = static_cast<int>((work + 255) / 256);
  if (blocks > 16 * num_sms()) blocks = 16 * num_sms();
  launch_pdl(embedding_bwd_tok_kernel, dim3(blocks), dim3(256), 0, s, static_cast<const uint32_t*>(sorted),
             reinterpret_cast<const bf16*>(dx), dwte, ntok, hidden);
  const int pwork = seq * (hidden / 8);
  launch_pdl(embedding_bwd_pos_kernel, dim3((pwork + 255) / 256), dim3(256), 0, s, reinterpret_cast<const bf16*>(dx),
                                                               dwpe, ntok, seq, hidden);
  return cudaGetLastError();
}

extern "C" int amdp_xent_fwd_bwd(uint16_t* logits, const int32_t* labels, float* loss_sum,
                                 float* row_loss, int ntok, int vocab, int ld, float scale,
                                 amdp_stream_t stream) {
  if (ntok <= 0 || vocab % 8 != 0 || ld % 8 != 0 || ld < vocab || !row_loss) return AMDP_ERR_INVALID;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  launch_pdl(xent_kernel, dim3(ntok), dim3(512), 0, s, reinterpret_cast<bf16*>(logits), labels, row_loss, vocab, ld,
             scale);
  launch_pdl(sum_rows_kernel, dim3(1), dim3(1024), 0, s, static_cast<const float*>(row_loss), ntok, loss_sum);
  return cudaGetLastError();
}
