// Short-sequence attention on the 5th-generation tensor cores (sm_100a): seq <= 128,
// head_dim 32 or 64 — the sequences the tiled kernels (attention_tc.cu, attention_bwd_tc.cu:
// 256-query / 128-key tiles) do not cover, e.g. the reference's tiny configuration (seq 64,
// head_dim 32).  One CTA of 4 warps per (sequence, head): the whole sequence is a single
// 128 x 128 score tile, so there is no online rescaling and no cross-CTA reduction.
//
// Forward : S = Q K^T (SS) -> row softmax in registers (thread = query = TMEM lane) -> P as
//           bf16 pairs over S's first 64 TMEM columns -> O = P V (TS, V MN-major in smem).
// Backward: transposed orientation (thread = key = TMEM lane):
//           S^T = K Q^T, dP^T = V dO^T                         (SS)
//           P^T = 2^(S^T c - lse), dS^T = P^T (dP^T - delta)   (lse / delta per column, smem)
//           dV = P^T dO, dK = dS^T Q                           (TS: P^T / dS^T from TMEM)
//           dQ = dS K                                          (SS: dS^T stored in smem rows
//                                                               indexed by key, i.e. the
//                                                               MN-major form of dS)
// Rows of the 128-row tiles past the sequence (the next sequence's rows, or TMA zero fill) are
// masked: keys >= min(seq, key_len) and queries >= seq get P = 0, and only rows < seq are
// stored.  Conventions as the tiled kernels: lse in the log2 domain with the softmax scale
// folded in; delta = rowsum(dO * O); dK, dQ carry the softmax scale.
#include "common.cuh"
#include "sm100_ptx.cuh"
#include "tma_host.hpp"

namespace amdp {
namespace {

constexpr uint32_t ST = 16384;  // one [128 rows][64 bf16] SW128 tile

__device__ __forceinline__ float ex2s(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&t);
}
__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~static_cast<uintptr_t>(1023));
}

// This thread's TMEM row (D fp32 columns at `src`) times `mul` -> bf16 at dst.
template <int D>
__device__ __forceinline__ void row_out(uint32_t src, bf16* dst, float mul) {
#pragma unroll
  for (int c = 0; c < D / 32; ++c) {
    uint32_t o[32];
    ptx::tmem_ld_32x32b_x32(src + c * 32, o);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float f[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(o[8 * u + e]) * mul;
      store8(dst + c * 32 + 8 * u, f);
    }
  }
}

template <int D>
__global__ void __launch_bounds__(128, 1)
    fa_short_fwd_kernel(const __grid_constant__ CUtensorMap qkv_map, bf16* __restrict__ out, float* __restrict__ lse,
                        int seq, int H, float scale_log2, int causal, const int32_t* __restrict__ key_len) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = align1024(smem_raw);
  uint64_t* ld_full = reinterpret_cast<uint64_t*>(sm + 3 * ST);
  uint64_t* mma_done = ld_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ld_full + 2);
  const int warp = threadIdx.x >> 5, r = threadIdx.x;
  const int b = blockIdx.x / H, h = blockIdx.x % H, row0 = b * seq;
  if (threadIdx.x == 0) {
    ptx::tma_prefetch(&qkv_map);
    ptx::mbar_init(ld_full, 1);
    ptx::mbar_init(mma_done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc<256>(tmem_slot);  // S: 0-127, O: 128-(128+D)
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  ptx::pdl_wait();
  ptx::pdl_trigger();
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(ld_full, 3 * ST);
    for (int t = 0; t < 3; ++t) ptx::tma_load_2d(sm + t * ST, &qkv_map, ld_full, t * H * D + h * D, row0);
  }
  ptx::mbar_wait(ld_full, 0);
  if (warp == 0) {  // S = Q K^T
    ptx::tc_fence_after();
    constexpr uint32_t id_s = ptx::idesc_bf16_f32(128, 128, false, false);
    const uint64_t dq = ptx::umma_desc_sw128(ptx::smem_u32(sm), 16, 1024);
    const uint64_t dk = ptx::umma_desc_sw128(ptx::smem_u32(sm + ST), 16, 1024);
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) ptx::mma_bf16_ss_w(tmem, dq + kk * 2, dk + kk * 2, id_s, kk > 0 ? 1u : 0u);
    ptx::mma_commit_w(mma_done);
  }
  ptx::mbar_wait(mma_done, 0);
  ptx::tc_fence_after();
  const uint32_t lanes = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  const int klen = key_len ? min(seq, key_len[b]) : seq;
  const int kend = causal ? min(klen, r + 1) : klen;  // keys [0, kend) of this query row
  uint32_t v[128];
#pragma unroll
  for (int c = 0; c < 4; ++c) ptx::tmem_ld_32x32b_x32(lanes + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&v[c * 32]));
  ptx::tmem_ld_wait();
  float mx = -INFINITY;
#pragma unroll
  for (int e = 0; e < 128; ++e)
    if (e < kend) mx = fmaxf(mx, __uint_as_float(v[e]));
  const float m = mx * scale_log2;
  float l = 0.f;
#pragma unroll
  for (int c = 0; c < 4; ++c) {  // 32 keys -> 16 bf16 pairs -> TMEM columns [16 c, 16 c + 16)
    uint32_t p[16];
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      const int k = 32 * c + e;
      const float p0 = k < kend ? ex2s(fmaf(__uint_as_float(v[k]), scale_log2, -m)) : 0.f;
      const float p1 = k + 1 < kend ? ex2s(fmaf(__uint_as_float(v[k + 1]), scale_log2, -m)) : 0.f;
      l += p0 + p1;
      p[e >> 1] = pack_bf16(p0, p1);
    }
    ptx::tmem_st_32x32b_x16(lanes + c * 16, p);
  }
  ptx::tmem_st_wait();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {  // O = P V (P from TMEM, V MN-major)
    ptx::tc_fence_after();
    constexpr uint32_t id_o = ptx::idesc_bf16_f32(128, D, false, true);
    const uint64_t dv = ptx::umma_desc_sw128(ptx::smem_u32(sm + 2 * ST), ST, 1024);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) ptx::mma_bf16_ts_w(tmem + 128, tmem + kk * 8, dv + kk * 128, id_o, kk > 0 ? 1u : 0u);
    ptx::mma_commit_w(mma_done);
  }
  ptx::mbar_wait(mma_done, 1);
  ptx::tc_fence_after();
  if (r < seq) {
    row_out<D>(lanes + 128, out + (static_cast<size_t>(row0) + r) * (static_cast<size_t>(H) * D) + h * D, 1.f / l);
    lse[(static_cast<size_t>(b) * H + h) * seq + r] = m + log2f(l);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<256>(tmem);
  }
}

template <int D>
__global__ void __launch_bounds__(128, 1)
    fa_short_bwd_kernel(const __grid_constant__ CUtensorMap qkv_map, const __grid_constant__ CUtensorMap do_map,
                        const float* __restrict__ lse, const float* __restrict__ delta, bf16* __restrict__ dqkv,
                        int seq, int H, float scale_log2, float scale, int causal,
                        const int32_t* __restrict__ key_len) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = align1024(smem_raw);
  // Q | K | V | dO | dS^T (2 chunks of [128 keys][64 queries]) | lse | delta | barriers
  uint8_t* s_q = sm;
  uint8_t* s_k = sm + ST;
  uint8_t* s_v = sm + 2 * ST;
  uint8_t* s_do = sm + 3 * ST;
  uint8_t* s_ds = sm + 4 * ST;
  float* lse_s = reinterpret_cast<float*>(sm + 6 * ST);
  float* del_s = lse_s + 128;
  uint64_t* ld_full = reinterpret_cast<uint64_t*>(del_s + 128);
  uint64_t* mma_done = ld_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ld_full + 2);
  const int warp = threadIdx.x >> 5, r = threadIdx.x;
  const int b = blockIdx.x / H, h = blockIdx.x % H, row0 = b * seq;
  const size_t bh = (static_cast<size_t>(b) * H + h) * seq;
  if (threadIdx.x == 0) {
    ptx::tma_prefetch(&qkv_map);
    ptx::tma_prefetch(&do_map);
    ptx::mbar_init(ld_full, 1);
    ptx::mbar_init(mma_done, 1);
    ptx::fence_mbar_init();
  }
  // S^T 0-127 | dP^T 128-255 | dV 256 | dK 320 | dQ 384 (D <= 64 columns each)
  if (warp == 0) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  ptx::pdl_wait();
  ptx::pdl_trigger();
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(ld_full, 4 * ST);
    for (int t = 0; t < 3; ++t) ptx::tma_load_2d(sm + t * ST, &qkv_map, ld_full, t * H * D + h * D, row0);
    ptx::tma_load_2d(s_do, &do_map, ld_full, h * D, row0);
  }
  lse_s[r] = r < seq ? lse[bh + r] : 0.f;
  del_s[r] = r < seq ? delta[bh + r] : 0.f;
  ptx::mbar_wait(ld_full, 0);
  if (warp == 0) {  // S^T = K Q^T, dP^T = V dO^T
    ptx::tc_fence_after();
    constexpr uint32_t id_s = ptx::idesc_bf16_f32(128, 128, false, false);
    const uint64_t dq = ptx::umma_desc_sw128(ptx::smem_u32(s_q), 16, 1024);
    const uint64_t dk = ptx::umma_desc_sw128(ptx::smem_u32(s_k), 16, 1024);
    const uint64_t dv = ptx::umma_desc_sw128(ptx::smem_u32(s_v), 16, 1024);
    const uint64_t ddo = ptx::umma_desc_sw128(ptx::smem_u32(s_do), 16, 1024);
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) ptx::mma_bf16_ss_w(tmem, dk + kk * 2, dq + kk * 2, id_s, kk > 0 ? 1u : 0u);
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk)
      ptx::mma_bf16_ss_w(tmem + 128, dv + kk * 2, ddo + kk * 2, id_s, kk > 0 ? 1u : 0u);
    ptx::mma_commit_w(mma_done);
  }
  __syncthreads();  // lse_s / del_s written
  ptx::mbar_wait(mma_done, 0);
  ptx::tc_fence_after();
  const uint32_t lanes = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  const int klen = key_len ? min(seq, key_len[b]) : seq;
  const bool key_ok = r < klen;  // this thread's key
  const int qbeg = causal ? r : 0;  // queries [qbeg, seq) see this key
  // 32 queries per chunk: P^T / dS^T as bf16 pairs over TMEM columns [16 c, 16 c + 16) of S^T /
  // dP^T (already read: chunk c reads columns [32 c, 32 c + 32)) — the TS operands of dV, dK —
  // and dS^T into smem: chunk k2 = c / 2 of the MN-major dS tile holds queries [64 k2, +64) of
  // this key's row as 8 swizzled 16-byte units (unit u at u ^ (key & 7)), as a TMA box would
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t s[32], d[32], pp[16], dd[16];
    ptx::tmem_ld_32x32b_x32(lanes + c * 32, s);
    ptx::tmem_ld_32x32b_x32(lanes + 128 + c * 32, d);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      const int q = c * 32 + e;
      const bool ok0 = key_ok && q >= qbeg && q < seq, ok1 = key_ok && q + 1 >= qbeg && q + 1 < seq;
      const float p0 = ok0 ? ex2s(fmaf(__uint_as_float(s[e]), scale_log2, -lse_s[q])) : 0.f;
      const float p1 = ok1 ? ex2s(fmaf(__uint_as_float(s[e + 1]), scale_log2, -lse_s[q + 1])) : 0.f;
      pp[e >> 1] = pack_bf16(p0, p1);
      dd[e >> 1] = pack_bf16(p0 * (__uint_as_float(d[e]) - del_s[q]), p1 * (__uint_as_float(d[e + 1]) - del_s[q + 1]));
    }
    ptx::tmem_st_32x32b_x16(lanes + c * 16, pp);
    ptx::tmem_st_32x32b_x16(lanes + 128 + c * 16, dd);
#pragma unroll
    for (int u4 = 0; u4 < 4; ++u4) {
      const int u = (c & 1) * 4 + u4;
      *reinterpret_cast<uint4*>(s_ds + (c >> 1) * ST + r * 128 + ((u ^ (r & 7)) << 4)) =
          make_uint4(dd[4 * u4], dd[4 * u4 + 1], dd[4 * u4 + 2], dd[4 * u4 + 3]);
    }
  }
  ptx::fence_proxy_async_smem();
  ptx::tmem_st_wait();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    constexpr uint32_t id_kv = ptx::idesc_bf16_f32(128, D, false, true);  // A from TMEM, B MN-major
    constexpr uint32_t id_q = ptx::idesc_bf16_f32(128, D, true, true);    // A, B MN-major (smem)
    const uint64_t bq = ptx::umma_desc_sw128(ptx::smem_u32(s_q), ST, 1024);
    const uint64_t bk = ptx::umma_desc_sw128(ptx::smem_u32(s_k), ST, 1024);
    const uint64_t bdo = ptx::umma_desc_sw128(ptx::smem_u32(s_do), ST, 1024);
    const uint64_t ads = ptx::umma_desc_sw128(ptx::smem_u32(s_ds), ST, 1024);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {  // 16 queries (dV, dK) / 16 keys (dQ) per step
      ptx::mma_bf16_ts_w(tmem + 256, tmem + kk * 8, bdo + kk * 128, id_kv, kk > 0 ? 1u : 0u);
      ptx::mma_bf16_ts_w(tmem + 320, tmem + 128 + kk * 8, bq + kk * 128, id_kv, kk > 0 ? 1u : 0u);
      ptx::mma_bf16_ss_w(tmem + 384, ads + kk * 128, bk + kk * 128, id_q, kk > 0 ? 1u : 0u);
    }
    ptx::mma_commit_w(mma_done);
  }
  ptx::mbar_wait(mma_done, 1);
  ptx::tc_fence_after();
  if (r < seq) {
    const size_t ld = static_cast<size_t>(3) * H * D;
    bf16* row = dqkv + (static_cast<size_t>(row0) + r) * ld + h * D;
    row_out<D>(lanes + 384, row, scale);              // dQ (row = query r)
    row_out<D>(lanes + 320, row + H * D, scale);      // dK (row = key r)
    row_out<D>(lanes + 256, row + 2 * H * D, 1.f);    // dV
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

template <class K>
int smem_attr(K k, size_t bytes, std::atomic<uint64_t>& flag) {
  if (!first_on_device(flag)) return 0;
  const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e != cudaSuccess) flag.store(0);
  return e;
}

template <int D>
int launch_short_fwd(const bf16* qkv, bf16* out, float* lse, int B, int S, int H, int causal, const int32_t* key_len,
                     cudaStream_t st) {
  CUtensorMap map;
  if (!tma_map_bf16_2d(&map, qkv, static_cast<uint64_t>(3) * H * D, static_cast<uint64_t>(B) * S,
                       static_cast<uint64_t>(3) * H * D, 64, 128))
    return AMDP_ERR_TMA;
  const size_t smem = 1024 + 3 * ST + 64;
  static std::atomic<uint64_t> attr{0};
  if (int e = smem_attr(fa_short_fwd_kernel<D>, smem, attr)) return e;
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(D));
  cudaError_t e = launch_pdl(fa_short_fwd_kernel<D>, dim3(B * H), dim3(128), smem, st, map, out, lse, S, H, scale_log2,
                             causal, key_len);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int D>
int launch_short_bwd(const bf16* qkv, const bf16* dout, const float* lse, const float* delta, bf16* dqkv, int B,
                     int S, int H, int causal, const int32_t* key_len, cudaStream_t st) {
  CUtensorMap qmap, omap;
  if (!tma_map_bf16_2d(&qmap, qkv, static_cast<uint64_t>(3) * H * D, static_cast<uint64_t>(B) * S,
                       static_cast<uint64_t>(3) * H * D, 64, 128) ||
      !tma_map_bf16_2d(&omap, dout, static_cast<uint64_t>(H) * D, static_cast<uint64_t>(B) * S,
                       static_cast<uint64_t>(H) * D, 64, 128))
    return AMDP_ERR_TMA;
  const size_t smem = 1024 + 6 * ST + 2 * 128 * sizeof(float) + 64;
  static std::atomic<uint64_t> attr{0};
  if (int e = smem_attr(fa_short_bwd_kernel<D>, smem, attr)) return e;
  const float scale = 1.f / sqrtf(static_cast<float>(D));
  const float scale_log2 = 1.4426950408889634f * scale;
  cudaError_t e = launch_pdl(fa_short_bwd_kernel<D>, dim3(B * H), dim3(128), smem, st, qmap, omap, lse, delta, dqkv, S,
                             H, scale_log2, scale, causal, key_len);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

bool attention_short_supported(int S, int D) { return S > 0 && S <= 128 && S % 8 == 0 && (D == 32 || D == 64); }

int attention_fwd_short(const bf16* qkv, bf16* out, float* lse, int B, int S, int H, int D, int causal,
                        const int32_t* key_len, cudaStream_t st) {
  if (D == 32) return launch_short_fwd<32>(qkv, out, lse, B, S, H, causal, key_len, st);
  if (D == 64) return launch_short_fwd<64>(qkv, out, lse, B, S, H, causal, key_len, st);
  return AMDP_ERR_UNSUPPORTED;
}

int attention_bwd_short(const bf16* qkv, const bf16* dout, const float* lse, const float* delta, bf16* dqkv, int B,
                        int S, int H, int D, int causal, const int32_t* key_len, cudaStream_t st) {
  if (D == 32) return launch_short_bwd<32>(qkv, dout, lse, delta, dqkv, B, S, H, causal, key_len, st);
  if (D == 64) return launch_short_bwd<64>(qkv, dout, lse, delta, dqkv, B, S, H, causal, key_len, st);
  return AMDP_ERR_UNSUPPORTED;
}

}  // namespace amdp
