// Fused causal attention for the stage executor (flash-style, never materialises S).
//
// Round-1 implementation on the warp-level tensor path (mma.sync m16n8k16 bf16,
// ldmatrix from padded shared memory, cp.async double buffering).  Forward keeps the
// online-softmax statistics as a log2-domain LSE for the backward.  The backward is
// split into two deterministic kernels, each with accumulator rows owned by one
// warp (no atomics): dQ (rows = queries) and dK/dV (rows = keys).
//
// Layout: qkv rows are tokens [batch*seq][3*H*D] = q | k | v, head-major inside each;
// out / dout rows [batch*seq][H*D]; lse/delta [batch][H][seq] fp32.
#include "common.cuh"

namespace amdp {
namespace {

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Copies `rows` x D bf16 from global (row stride ld elements) to smem (row stride D+8).
template <int D>
__device__ __forceinline__ void load_tile(bf16* s, const bf16* g, int ld, int rows) {
  constexpr int CH = D / 8;
  for (int i = threadIdx.x; i < rows * CH; i += blockDim.x) {
    const int r = i / CH, c = (i % CH) * 8;
    cp_async16(s + r * (D + 8) + c, g + static_cast<size_t>(r) * ld + c);
  }
}

// A-operand fragment (16 rows x 16 cols starting at (row0, col0)) from a padded tile.
template <int D>
__device__ __forceinline__ void lda_frag(uint32_t (&a)[4], const bf16* s, int row0, int col0) {
  const int l = threadIdx.x & 31, mat = l >> 3;
  ldsm_x4(a, s + (row0 + ((mat & 1) << 3) + (l & 7)) * (D + 8) + col0 + ((mat >> 1) << 3));
}
// B fragments for two n-tiles (rows n0..n0+15 of a [n][k] tile) at k-step col0:
// r[0],r[1] -> n-tile n0, r[2],r[3] -> n-tile n0+8.
template <int D>
__device__ __forceinline__ void ldb_frag_nk(uint32_t (&r)[4], const bf16* s, int n0, int col0) {
  const int l = threadIdx.x & 31, mat = l >> 3;
  ldsm_x4(r, s + (n0 + ((mat >> 1) << 3) + (l & 7)) * (D + 8) + col0 + ((mat & 1) << 3));
}
// B fragments from a [k][n] tile (n contiguous) via transpose: k-step rows k0..k0+15,
// n-tiles n0 and n0+8.  r[0],r[1] -> n0; r[2],r[3] -> n0+8.
template <int D>
__device__ __forceinline__ void ldb_frag_kn(uint32_t (&r)[4], const bf16* s, int k0, int n0) {
  const int l = threadIdx.x & 31, mat = l >> 3;
  ldsm_x4_t(r, s + (k0 + ((mat & 1) << 3) + (l & 7)) * (D + 8) + n0 + ((mat >> 1) << 3));
}

// ================================================================== forward
template <int D>
__global__ void __launch_bounds__(128) attn_fwd_kernel(const bf16* __restrict__ qkv,
                                                       bf16* __restrict__ out,
                                                       float* __restrict__ lse, int seq, int H,
                                                       float scale_log2, int causal,
                                                       const int32_t* __restrict__ key_len) {
  constexpr int BQ = 64, BKV = 64, LDS = D + 8;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  bf16* sQ = reinterpret_cast<bf16*>(smem_raw);
  bf16* sK = sQ + BQ * LDS;        // 2 buffers
  bf16* sV = sK + 2 * BKV * LDS;   // 2 buffers
  const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int ld = 3 * H * D;
  const bf16* base = qkv + static_cast<size_t>(b) * seq * ld;
  const bf16* gQ = base + static_cast<size_t>(qb) * BQ * ld + h * D;
  const bf16* gK = base + H * D + h * D;
  const bf16* gV = base + 2 * H * D + h * D;
  const int nkb = causal ? qb + 1 : seq / BKV;
  const int klen = key_len ? key_len[b] : seq;  // key padding (bidirectional models)

  load_tile<D>(sQ, gQ, ld, BQ);
  load_tile<D>(sK, gK, ld, BKV);
  load_tile<D>(sV, gV, ld, BKV);
  cp_async_commit();

  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  uint32_t qf[D / 16][4];
  const int q_row0 = qb * BQ + warp * 16 + g;  // this thread's rows: q_row0, q_row0 + 8

  for (int kb = 0; kb < nkb; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nkb) {
      load_tile<D>(sK + (buf ^ 1) * BKV * LDS, gK + static_cast<size_t>(kb + 1) * BKV * ld, ld, BKV);
      load_tile<D>(sV + (buf ^ 1) * BKV * LDS, gV + static_cast<size_t>(kb + 1) * BKV * ld, ld, BKV);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (kb == 0) {
#pragma unroll
      for (int d = 0; d < D / 16; ++d) lda_frag<D>(qf[d], sQ, warp * 16, d * 16);
    }
    const bf16* k_s = sK + buf * BKV * LDS;
    const bf16* v_s = sV + buf * BKV * LDS;
    float s[BKV / 8][4];
#pragma unroll
    for (int j = 0; j < BKV / 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int j = 0; j < BKV / 8; j += 2)
#pragma unroll
      for (int d = 0; d < D / 16; ++d) {
        uint32_t r[4];
        ldb_frag_nk<D>(r, k_s, j * 8, d * 16);
        mma16816(s[j], qf[d], r[0], r[1]);
        mma16816(s[j + 1], qf[d], r[2], r[3]);
      }
    // scale (log2 domain) + causal mask on the diagonal block, key-padding mask
    const bool diag = causal && kb == qb;
    const bool lim = (kb + 1) * BKV > klen;
#pragma unroll
    for (int j = 0; j < BKV / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = s[j][e] * scale_log2;
        const int key = kb * BKV + j * 8 + 2 * t + (e & 1);
        if (diag) {
          const int qrow = q_row0 + ((e >> 1) << 3);
          if (key > qrow) v = -INFINITY;
        }
        if (lim && key >= klen) v = -INFINITY;
        s[j][e] = v;
      }
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int j = 0; j < BKV / 8; ++j) {
      mx0 = fmaxf(mx0, fmaxf(s[j][0], s[j][1]));
      mx1 = fmaxf(mx1, fmaxf(s[j][2], s[j][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float a0 = exp2f(m0 - mx0), a1 = exp2f(m1 - mx1);  // m = -inf first time -> 0
    m0 = mx0;
    m1 = mx1;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int j = 0; j < BKV / 8; ++j) {
      s[j][0] = exp2f(s[j][0] - m0);
      s[j][1] = exp2f(s[j][1] - m0);
      s[j][2] = exp2f(s[j][2] - m1);
      s[j][3] = exp2f(s[j][3] - m1);
      rs0 += s[j][0] + s[j][1];
      rs1 += s[j][2] + s[j][3];
    }
    l0 = l0 * a0 + rs0;
    l1 = l1 * a1 + rs1;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      o[i][0] *= a0;
      o[i][1] *= a0;
      o[i][2] *= a1;
      o[i][3] *= a1;
    }
    // O += P V
#pragma unroll
    for (int ks = 0; ks < BKV / 16; ++ks) {
      uint32_t pa[4];
      pa[0] = pack_bf16(s[2 * ks][0], s[2 * ks][1]);
      pa[1] = pack_bf16(s[2 * ks][2], s[2 * ks][3]);
      pa[2] = pack_bf16(s[2 * ks + 1][0], s[2 * ks + 1][1]);
      pa[3] = pack_bf16(s[2 * ks + 1][2], s[2 * ks + 1][3]);
#pragma unroll
      for (int n = 0; n < D / 8; n += 2) {
        uint32_t r[4];
        ldb_frag_kn<D>(r, v_s, ks * 16, n * 8);
        mma16816(o[n], pa, r[0], r[1]);
        mma16816(o[n + 1], pa, r[2], r[3]);
      }
    }
    __syncthreads();  // buffer `buf` is refilled two iterations later
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float inv0 = 1.f / l0, inv1 = 1.f / l1;
  bf16* orow0 = out + (static_cast<size_t>(b) * seq + q_row0) * (H * D) + h * D;
  bf16* orow1 = orow0 + static_cast<size_t>(8) * H * D;
#pragma unroll
  for (int n = 0; n < D / 8; ++n) {
    *reinterpret_cast<uint32_t*>(orow0 + n * 8 + 2 * t) = pack_bf16(o[n][0] * inv0, o[n][1] * inv0);
    *reinterpret_cast<uint32_t*>(orow1 + n * 8 + 2 * t) = pack_bf16(o[n][2] * inv1, o[n][3] * inv1);
  }
  if (t == 0) {
    float* L = lse + (static_cast<size_t>(b) * H + h) * seq;
    L[q_row0] = m0 + log2f(l0);
    L[q_row0 + 8] = m1 + log2f(l1);
  }
}

// ================================================================== backward prep
// delta[b,h,s] = sum_d dout * out   (one warp per (token, head))
__global__ void attn_bwd_delta_kernel(const bf16* __restrict__ out, const bf16* __restrict__ dout,
                                      float* __restrict__ delta, int ntok, int seq, int H, int D) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= ntok * H) return;
  const int tok = w / H, h = w % H;
  const bf16* o = out + static_cast<size_t>(tok) * H * D + h * D;
  const bf16* d = dout + static_cast<size_t>(tok) * H * D + h * D;
  float s = 0.f;
  for (int c = lane; c < D; c += 32) s += __bfloat162float(o[c]) * __bfloat162float(d[c]);
  s = warp_sum(s);
  if (lane == 0) {
    const int b = tok / seq, p = tok % seq;
    delta[(static_cast<size_t>(b) * H + h) * seq + p] = s;
  }
}

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

// ================================================================== backward dQ
template <int D>
__global__ void __launch_bounds__(128) attn_bwd_dq_kernel(
    const bf16* __restrict__ qkv, const bf16* __restrict__ dout, const float* __restrict__ lse,
    const float* __restrict__ delta, bf16* __restrict__ dqkv, int seq, int H, float scale_log2,
    float scale, int causal, const int32_t* __restrict__ key_len) {
  constexpr int BQ = 64, BKV = 64, LDS = D + 8;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  bf16* sQ = reinterpret_cast<bf16*>(smem_raw);
  bf16* sdO = sQ + BQ * LDS;
  bf16* sK = sdO + BQ * LDS;      // 2 buffers
  bf16* sV = sK + 2 * BKV * LDS;  // 2 buffers
  const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int ld = 3 * H * D, ldo = H * D;
  const bf16* base = qkv + static_cast<size_t>(b) * seq * ld;
  const bf16* gK = base + H * D + h * D;
  const bf16* gV = base + 2 * H * D + h * D;
  const int nkb = causal ? qb + 1 : seq / BKV;
  const int q_row0 = qb * BQ + warp * 16 + g;
  const float* L = lse + (static_cast<size_t>(b) * H + h) * seq;
  const float* Dl = delta + (static_cast<size_t>(b) * H + h) * seq;
  const float lse0 = L[q_row0], lse1 = L[q_row0 + 8];
  const float dl0 = Dl[q_row0], dl1 = Dl[q_row0 + 8];

  load_tile<D>(sQ, base + static_cast<size_t>(qb) * BQ * ld + h * D, ld, BQ);
  load_tile<D>(sdO, dout + (static_cast<size_t>(b) * seq + qb * BQ) * ldo + h * D, ldo, BQ);
  load_tile<D>(sK, gK, ld, BKV);
  load_tile<D>(sV, gV, ld, BKV);
  cp_async_commit();

  float dq[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;

  for (int kb = 0; kb < nkb; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nkb) {
      load_tile<D>(sK + (buf ^ 1) * BKV * LDS, gK + static_cast<size_t>(kb + 1) * BKV * ld, ld, BKV);
      load_tile<D>(sV + (buf ^ 1) * BKV * LDS, gV + static_cast<size_t>(kb + 1) * BKV * ld, ld, BKV);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const bf16* k_s = sK + buf * BKV * LDS;
    const bf16* v_s = sV + buf * BKV * LDS;
    float s[BKV / 8][4], dp[BKV / 8][4];
#pragma unroll
    for (int j = 0; j < BKV / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[j][e] = dp[j][e] = 0.f;
#pragma unroll
    for (int d = 0; d < D / 16; ++d) {
      uint32_t qa[4], da[4];
      lda_frag<D>(qa, sQ, warp * 16, d * 16);
      lda_frag<D>(da, sdO, warp * 16, d * 16);
#pragma unroll
      for (int j = 0; j < BKV / 8; j += 2) {
        uint32_t r[4];
        ldb_frag_nk<D>(r, k_s, j * 8, d * 16);
        mma16816(s[j], qa, r[0], r[1]);
        mma16816(s[j + 1], qa, r[2], r[3]);
        ldb_frag_nk<D>(r, v_s, j * 8, d * 16);
        mma16816(dp[j], da, r[0], r[1]);
        mma16816(dp[j + 1], da, r[2], r[3]);
      }
    }
    const bool diag = causal && kb == qb;
    const int klen = key_len ? key_len[b] : seq;
#pragma unroll
    for (int j = 0; j < BKV / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const bool hi = e >> 1;
        float p = exp2f(s[j][e] * scale_log2 - (hi ? lse1 : lse0));
        const int key = kb * BKV + j * 8 + 2 * t + (e & 1);
        if (diag && key > q_row0 + (hi ? 8 : 0)) p = 0.f;
        if (key >= klen) p = 0.f;
        s[j][e] = p * (dp[j][e] - (hi ? dl1 : dl0));  // dS
      }
#pragma unroll
    for (int ks = 0; ks < BKV / 16; ++ks) {
      uint32_t pa[4];
      pa[0] = pack_bf16(s[2 * ks][0], s[2 * ks][1]);
      pa[1] = pack_bf16(s[2 * ks][2], s[2 * ks][3]);
      pa[2] = pack_bf16(s[2 * ks + 1][0], s[2 * ks + 1][1]);
      pa[3] = pack_bf16(s[2 * ks + 1][2], s[2 * ks + 1][3]);
#pragma unroll
      for (int n = 0; n < D / 8; n += 2) {
        uint32_t r[4];
        ldb_frag_kn<D>(r, k_s, ks * 16, n * 8);
        mma16816(dq[n], pa, r[0], r[1]);
        mma16816(dq[n + 1], pa, r[2], r[3]);
      }
    }
    __syncthreads();
  }
  bf16* r0 = dqkv + (static_cast<size_t>(b) * seq + q_row0) * ld + h * D;
  bf16* r1 = r0 + static_cast<size_t>(8) * ld;
#pragma unroll
  for (int n = 0; n < D / 8; ++n) {
    *reinterpret_cast<uint32_t*>(r0 + n * 8 + 2 * t) = pack_bf16(dq[n][0] * scale, dq[n][1] * scale);
    *reinterpret_cast<uint32_t*>(r1 + n * 8 + 2 * t) = pack_bf16(dq[n][2] * scale, dq[n][3] * scale);
  }
}

// ================================================================== backward dK, dV
template <int D, int BQ>
__global__ void __launch_bounds__(128) attn_bwd_dkdv_kernel(
    const bf16* __restrict__ qkv, const bf16* __restrict__ dout, const float* __restrict__ lse,
    const float* __restrict__ delta, bf16* __restrict__ dqkv, int seq, int H, float scale_log2,
    float scale, int causal, const int32_t* __restrict__ key_len) {
  constexpr int BKV = 64, LDS = D + 8;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  bf16* sK = reinterpret_cast<bf16*>(smem_raw);
  bf16* sV = sK + BKV * LDS;
  bf16* sQ = sV + BKV * LDS;        // 2 buffers
  bf16* sdO = sQ + 2 * BQ * LDS;    // 2 buffers
  float* sL = reinterpret_cast<float*>(sdO + 2 * BQ * LDS);  // 2 x BQ
  float* sD = sL + 2 * BQ;                                   // 2 x BQ
  const int kb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int ld = 3 * H * D, ldo = H * D;
  const bf16* base = qkv + static_cast<size_t>(b) * seq * ld;
  const bf16* gQ = base + h * D;
  const bf16* gdO = dout + static_cast<size_t>(b) * seq * ldo + h * D;
  const float* L = lse + (static_cast<size_t>(b) * H + h) * seq;
  const float* Dl = delta + (static_cast<size_t>(b) * H + h) * seq;
  const int qb0 = causal ? (kb * BKV) / BQ : 0;
  const int nqb = seq / BQ;
  const int key0 = kb * BKV + warp * 16 + g;  // this thread's key rows: key0, key0 + 8

  auto load_q = [&](int qb, int bufi) {
    load_tile<D>(sQ + bufi * BQ * LDS, gQ + static_cast<size_t>(qb) * BQ * ld, ld, BQ);
    load_tile<D>(sdO + bufi * BQ * LDS, gdO + static_cast<size_t>(qb) * BQ * ldo, ldo, BQ);
    for (int i = threadIdx.x; i < BQ; i += blockDim.x) {
      sL[bufi * BQ + i] = L[qb * BQ + i];
      sD[bufi * BQ + i] = Dl[qb * BQ + i];
    }
  };
  load_tile<D>(sK, base + H * D + static_cast<size_t>(kb) * BKV * ld + h * D, ld, BKV);
  load_tile<D>(sV, base + 2 * H * D + static_cast<size_t>(kb) * BKV * ld + h * D, ld, BKV);
  load_q(qb0, 0);
  cp_async_commit();

  float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;

  for (int qb = qb0; qb < nqb; ++qb) {
    const int buf = (qb - qb0) & 1;
    if (qb + 1 < nqb) {
      load_q(qb + 1, buf ^ 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const bf16* q_s = sQ + buf * BQ * LDS;
    const bf16* do_s = sdO + buf * BQ * LDS;
    const float* l_s = sL + buf * BQ;
    const float* d_s = sD + buf * BQ;
    float s[BQ / 8][4], dp[BQ / 8][4];
#pragma unroll
    for (int j = 0; j < BQ / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[j][e] = dp[j][e] = 0.f;
    // S^T = K Q^T and dP^T = V dO^T (rows = keys)
#pragma unroll
    for (int d = 0; d < D / 16; ++d) {
      uint32_t ka[4], va[4];
      lda_frag<D>(ka, sK, warp * 16, d * 16);
      lda_frag<D>(va, sV, warp * 16, d * 16);
#pragma unroll
      for (int j = 0; j < BQ / 8; j += 2) {
        uint32_t r[4];
        ldb_frag_nk<D>(r, q_s, j * 8, d * 16);
        mma16816(s[j], ka, r[0], r[1]);
        mma16816(s[j + 1], ka, r[2], r[3]);
        ldb_frag_nk<D>(r, do_s, j * 8, d * 16);
        mma16816(dp[j], va, r[0], r[1]);
        mma16816(dp[j + 1], va, r[2], r[3]);
      }
    }
    // P^T and dS^T
#pragma unroll
    for (int j = 0; j < BQ / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qc = j * 8 + 2 * t + (e & 1);  // query column within the block
        const int key = key0 + ((e >> 1) << 3);
        float p = exp2f(s[j][e] * scale_log2 - l_s[qc]);
        if (causal && qb * BQ + qc < key) p = 0.f;
        if (key_len && key >= key_len[b]) p = 0.f;  // a padding key
        s[j][e] = p;
        dp[j][e] = p * (dp[j][e] - d_s[qc]);
      }
    // dV += P^T dO ; dK += dS^T Q   (k = queries)
#pragma unroll
    for (int ks = 0; ks < BQ / 16; ++ks) {
      uint32_t pa[4], sa[4];
      pa[0] = pack_bf16(s[2 * ks][0], s[2 * ks][1]);
      pa[1] = pack_bf16(s[2 * ks][2], s[2 * ks][3]);
      pa[2] = pack_bf16(s[2 * ks + 1][0], s[2 * ks + 1][1]);
      pa[3] = pack_bf16(s[2 * ks + 1][2], s[2 * ks + 1][3]);
      sa[0] = pack_bf16(dp[2 * ks][0], dp[2 * ks][1]);
      sa[1] = pack_bf16(dp[2 * ks][2], dp[2 * ks][3]);
      sa[2] = pack_bf16(dp[2 * ks + 1][0], dp[2 * ks + 1][1]);
      sa[3] = pack_bf16(dp[2 * ks + 1][2], dp[2 * ks + 1][3]);
#pragma unroll
      for (int n = 0; n < D / 8; n += 2) {
        uint32_t r[4];
        ldb_frag_kn<D>(r, do_s, ks * 16, n * 8);
        mma16816(dv[n], pa, r[0], r[1]);
        mma16816(dv[n + 1], pa, r[2], r[3]);
        ldb_frag_kn<D>(r, q_s, ks * 16, n * 8);
        mma16816(dk[n], sa, r[0], r[1]);
        mma16816(dk[n + 1], sa, r[2], r[3]);
      }
    }
    __syncthreads();
  }
  bf16* k0 = dqkv + (static_cast<size_t>(b) * seq + key0) * ld + H * D + h * D;
  bf16* k1 = k0 + static_cast<size_t>(8) * ld;
  bf16* v0 = k0 + H * D;
  bf16* v1 = k1 + H * D;
#pragma unroll
  for (int n = 0; n < D / 8; ++n) {
    *reinterpret_cast<uint32_t*>(k0 + n * 8 + 2 * t) = pack_bf16(dk[n][0] * scale, dk[n][1] * scale);
    *reinterpret_cast<uint32_t*>(k1 + n * 8 + 2 * t) = pack_bf16(dk[n][2] * scale, dk[n][3] * scale);
    *reinterpret_cast<uint32_t*>(v0 + n * 8 + 2 * t) = pack_bf16(dv[n][0], dv[n][1]);
    *reinterpret_cast<uint32_t*>(v1 + n * 8 + 2 * t) = pack_bf16(dv[n][2], dv[n][3]);
  }
}

template <int D>
int launch_fwd(const bf16* qkv, bf16* out, float* lse, int B, int S, int H, int causal,
               const int32_t* key_len, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(5) * 64 * (D + 8) * sizeof(bf16);
  auto k = attn_fwd_kernel<D>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  const float scale_log2 = kLog2e / sqrtf(static_cast<float>(D));
  k<<<dim3(S / 64, H, B), 128, smem, st>>>(qkv, out, lse, S, H, scale_log2, causal, key_len);
  return cudaGetLastError();
}

template <int D>
int launch_bwd(const bf16* qkv, const bf16* out, const bf16* dout, const float* lse,
               bf16* dqkv, float* delta, int B, int S, int H, int causal, const int32_t* key_len, cudaStream_t st) {
  const int ntok = B * S;
  attn_bwd_delta_kernel<<<(ntok * H + 7) / 8, 256, 0, st>>>(out, dout, delta, ntok, S, H, D);
  const float scale = 1.f / sqrtf(static_cast<float>(D));
  const float scale_log2 = kLog2e * scale;
  {
    const size_t smem = static_cast<size_t>(6) * 64 * (D + 8) * sizeof(bf16);
    auto k = attn_bwd_dq_kernel<D>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k<<<dim3(S / 64, H, B), 128, smem, st>>>(qkv, dout, lse, delta, dqkv, S, H, scale_log2, scale,
                                             causal, key_len);
  }
  {
    constexpr int BQ = D > 64 ? 32 : 64;
    const size_t smem = static_cast<size_t>(2 * 64 + 4 * BQ) * (D + 8) * sizeof(bf16) +
                        4 * BQ * sizeof(float);
    auto k = attn_bwd_dkdv_kernel<D, BQ>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k<<<dim3(S / 64, H, B), 128, smem, st>>>(qkv, dout, lse, delta, dqkv, S, H, scale_log2,
                                             scale, causal, key_len);
  }
  return cudaGetLastError();
}

}  // namespace
}  // namespace amdp

namespace amdp {
int attention_fwd_tc(const bf16* qkv, bf16* out, float* lse, int B, int S, int H, int D, int causal,
                     const int32_t* key_len, cudaStream_t st);
int attention_bwd_tc(const bf16* qkv, const bf16* dout, const float* lse, const float* delta, bf16* dqkv, int B,
                     int S, int H, int D, int causal, const int32_t* key_len, cudaStream_t st);
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
  switch (head_dim) {
    case 32: return launch_fwd<32>(q, o, lse, batch, seq, heads, causal, key_len, s);
    case 64: return launch_fwd<64>(q, o, lse, batch, seq, heads, causal, key_len, s);
    case 80: return launch_fwd<80>(q, o, lse, batch, seq, heads, causal, key_len, s);
    case 128: return launch_fwd<128>(q, o, lse, batch, seq, heads, causal, key_len, s);
  }
  return AMDP_ERR_UNSUPPORTED;
}

extern "C" int amdp_attention_bwd_delta(const uint16_t* qkv, const uint16_t* dout, const float* lse,
                                        const float* delta, uint16_t* dqkv, int batch, int seq, int heads,
                                        int head_dim, int causal, const int32_t* key_len, amdp_stream_t stream) {
  if (batch <= 0 || seq <= 0 || heads <= 0 || !delta) return AMDP_ERR_INVALID;
  if (causal && key_len) return AMDP_ERR_UNSUPPORTED;
  if (!amdp_attention_bwd_delta_supported(seq, head_dim)) return AMDP_ERR_UNSUPPORTED;
  return attention_bwd_tc(reinterpret_cast<const bf16*>(qkv), reinterpret_cast<const bf16*>(dout), lse,
                          const_cast<float*>(delta), reinterpret_cast<bf16*>(dqkv), batch, seq, heads, head_dim,
                          causal, key_len, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int amdp_attention_impl(int seq, int head_dim, int backward) {
  const bool tc_dim = head_dim == 64 || head_dim == 80 || head_dim == 128;
  if (seq <= 0 || seq % 64 != 0) return -1;
  if (tc_dim && seq % (backward ? 128 : 256) == 0) return AMDP_ATTN_IMPL_TCGEN05;
  if (head_dim == 32 || tc_dim) return AMDP_ATTN_IMPL_MMA_SYNC;
  return -1;
}

extern "C" int amdp_attention_bwd_delta_supported(int seq, int head_dim) {
  return (head_dim == 64 || head_dim == 80 || head_dim == 128) && seq > 0 && seq % 128 == 0;
}

extern "C" size_t amdp_attention_bwd_workspace(int batch, int seq, int heads, int head_dim) {
  (void)head_dim;
  return static_cast<size_t>(batch) * seq * heads * sizeof(float);
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
  if ((head_dim == 64 || head_dim == 80 || head_dim == 128) && seq % 128 == 0) {  // tcgen05 path
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
    return attention_bwd_tc(q, d, lse, w, dq, batch, seq, heads, head_dim, causal, key_len, s);
  }
  switch (head_dim) {
    case 32: return launch_bwd<32>(q, o, d, lse, dq, w, batch, seq, heads, causal, key_len, s);
    case 64: return launch_bwd<64>(q, o, d, lse, dq, w, batch, seq, heads, causal, key_len, s);
    case 80: return launch_bwd<80>(q, o, d, lse, dq, w, batch, seq, heads, causal, key_len, s);
    case 128: return launch_bwd<128>(q, o, d, lse, dq, w, batch, seq, heads, causal, key_len, s);
  }
  return AMDP_ERR_UNSUPPORTED;
}
