// Flash-attention backward on the 5th-generation tensor cores (sm_100a).
//
// Two deterministic kernels (no atomics), each with its accumulators in TMEM:
//   dK/dV : one CTA per (128-key tile, head, sequence), looping over 64-query blocks:
//           S^T = K Q_i^T, dP^T = V dO_i^T            (M=128 keys, N=64, K=D)
//           P^T = 2^(S^T c - lse), dS^T = P^T (dP^T - delta)  (warps 4-7, thread = key)
//           dV += P^T dO_i, dK += dS^T Q_i              (M=128, N=D, K=64)
//   dQ    : one CTA per (128-query tile, head, sequence), looping over 64-key blocks:
//           S = Q K_j^T, dP = dO V_j^T; dS = P (dP - delta); dQ += dS K_j
// Every operand is in its natural layout: the same SWIZZLE_128B tile of Q, dO or K is
// read K-major by one MMA and MN-major by another, P^T / dS^T / dS are written by the
// softmax threads straight into the K-major swizzled layout the tensor core reads.
// lse / delta use the forward's log2-domain convention (softmax scale folded in);
// delta = rowsum(dO * O) comes from attn_bwd_delta_kernel (attention.cu).
#include "common.cuh"
#include "sm100_ptx.cuh"
#include "tma_host.hpp"

namespace amdp {
namespace {

constexpr uint32_t T128 = 16384;  // [128 rows][64 bf16] SW128 tile

// Diagnostics (amdp_debug_attention_bwd_trace): CTA 0 of the dQ kernel records clock64().
__device__ long long* g_bw_dbg = nullptr;
#define BW_T(slot, j)                                                                       \
  do {                                                                                      \
    if (dbg_ != nullptr && (j) < 64) dbg_[(slot)*64 + (j)] = clock64(); \
  } while (0)
constexpr uint32_t T64 = 8192;    // [64 rows][64 bf16]

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&t);
}

// ==================================================================== dK / dV
template <int D>
struct KvSmem {
  static constexpr int NB = D / 64;
  static constexpr uint32_t K = 0;
  static constexpr uint32_t V = K + NB * T128;
  static constexpr int NS = 3;                   // Q / dO / lse / delta ring depth
  static constexpr uint32_t Q = V + NB * T128;   // NS stages of NB x T64
  static constexpr uint32_t DO = Q + NS * NB * T64;
  static constexpr uint32_t PT = DO + NS * NB * T64;  // 2 warpgroups x [128 keys][64 q]
  static constexpr uint32_t DST = PT + 2 * T128;
  static constexpr uint32_t LD = DST + 2 * T128;  // NS stages x (64 lse + 64 delta) fp32
  static constexpr uint32_t BAR = LD + NS * 512;
  static constexpr uint32_t BYTES = BAR + 256;
  static constexpr uint32_t TMEM_COLS = 512;
};

template <int D>
__global__ void __launch_bounds__(384, 1)
    fa_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap qkv128, const __grid_constant__ CUtensorMap qkv64,
                       const __grid_constant__ CUtensorMap do64, const float* __restrict__ lse,
                       const float* __restrict__ delta, bf16* __restrict__ dqkv, int seq, int H, int n_kt,
                       float scale_log2, float scale, int causal) {
  using L = KvSmem<D>;
  extern __shared__ uint8_t smem_raw[];
  long long* const dbg_ = blockIdx.x == 0 ? g_bw_dbg : nullptr;  // trace hook, read once
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~static_cast<uintptr_t>(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  constexpr int NS = L::NS;
  uint64_t* kv_full = bar + 0;
  uint64_t* q_full = bar + 1;   // [NS]
  uint64_t* q_empty = bar + 5;  // [NS]
  uint64_t* s_full = bar + 9;   // [2] per warpgroup
  uint64_t* s_empty = bar + 11; // [2]
  uint64_t* p_full = bar + 13;  // [2]
  uint64_t* pd_done = bar + 15; // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 17);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kt = static_cast<int>(blockIdx.x % n_kt);  // causal: small kt = most work, first
  const int hb = static_cast<int>(blockIdx.x / n_kt);
  const int h = hb % H, b = hb / H;
  const int row0 = b * seq;
  const int nqb = seq / 64;
  const int i0 = causal ? 2 * kt : 0;
  const int N = nqb - i0;
  const float* lse_bh = lse + (static_cast<size_t>(b) * H + h) * seq;
  const float* del_bh = delta + (static_cast<size_t>(b) * H + h) * seq;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&qkv128);
    ptx::tma_prefetch(&qkv64);
    ptx::tma_prefetch(&do64);
    ptx::mbar_init(kv_full, 1);
    for (int s = 0; s < NS; ++s) {
      ptx::mbar_init(&q_full[s], 1);
      ptx::mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&s_full[s], 1);
      ptx::mbar_init(&s_empty[s], 128);
      ptx::mbar_init(&p_full[s], 128);
      ptx::mbar_init(&pd_done[s], 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<L::TMEM_COLS>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM: S^T_w at 128w, dP^T_w at 128w + 64 (w = warpgroup), dV at 256, dK at 256 + D
  const uint32_t t_dv = tmem + 256, t_dk = tmem + 256 + D;

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(kv_full, 2 * L::NB * T128);
      for (int c = 0; c < L::NB; ++c) {
        ptx::tma_load_2d(sm + L::K + c * T128, &qkv128, kv_full, H * D + h * D + 64 * c, row0 + kt * 128);
        ptx::tma_load_2d(sm + L::V + c * T128, &qkv128, kv_full, 2 * H * D + h * D + 64 * c, row0 + kt * 128);
      }
      for (int n = 0; n < N; ++n) {
        const int st = n % NS, i = i0 + n;
        ptx::mbar_wait(&q_empty[st], ((n / NS) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&q_full[st], 2 * L::NB * T64 + 512);
        for (int c = 0; c < L::NB; ++c) {
          ptx::tma_load_2d(sm + L::Q + (st * L::NB + c) * T64, &qkv64, &q_full[st], h * D + 64 * c, row0 + i * 64);
          ptx::tma_load_2d(sm + L::DO + (st * L::NB + c) * T64, &do64, &q_full[st], h * D + 64 * c, row0 + i * 64);
        }
        ptx::bulk_load(sm + L::LD + st * 512, lse_bh + i * 64, 256, &q_full[st]);
        ptx::bulk_load(sm + L::LD + st * 512 + 256, del_bh + i * 64, 256, &q_full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = ptx::idesc_bf16_f32(128, 64, false, false);
      constexpr uint32_t id_g = ptx::idesc_bf16_f32(128, D, false, true);
      const uint32_t sk = ptx::smem_u32(sm + L::K), sv = ptx::smem_u32(sm + L::V);
      ptx::mbar_wait(kv_full, 0);
      for (int n = 0; n <= N; ++n) {
        if (n < N) {
          const int st = n % NS, w = n & 1;
          const uint32_t t_st = tmem + 128 * w, t_dpt = t_st + 64;
          ptx::mbar_wait(&q_full[st], (n / NS) & 1);
          ptx::mbar_wait(&s_empty[w], ((n >> 1) & 1) ^ 1);
          ptx::tc_fence_after();
          const uint32_t sq = ptx::smem_u32(sm + L::Q + st * L::NB * T64);
          const uint32_t sdo = ptx::smem_u32(sm + L::DO + st * L::NB * T64);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t oa = (kk >> 2) * T128 + (kk & 3) * 32, ob = (kk >> 2) * T64 + (kk & 3) * 32;
            ptx::mma_bf16_ss(t_st, ptx::umma_desc_sw128(sk + oa, 16, 1024), ptx::umma_desc_sw128(sq + ob, 16, 1024),
                             id_s, kk > 0);
            ptx::mma_bf16_ss(t_dpt, ptx::umma_desc_sw128(sv + oa, 16, 1024),
                             ptx::umma_desc_sw128(sdo + ob, 16, 1024), id_s, kk > 0);
          }
          ptx::mma_commit(&s_full[w]);
        }
        if (n > 0) {
          const int m = n - 1, st = m % NS, w = m & 1;
          ptx::mbar_wait(&p_full[w], (m >> 1) & 1);
          ptx::tc_fence_after();
          const uint32_t sq = ptx::smem_u32(sm + L::Q + st * L::NB * T64);
          const uint32_t sdo = ptx::smem_u32(sm + L::DO + st * L::NB * T64);
          const uint32_t spt = ptx::smem_u32(sm + L::PT + w * T128), sdst = ptx::smem_u32(sm + L::DST + w * T128);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // K = 64 queries
            ptx::mma_bf16_ss(t_dv, ptx::umma_desc_sw128(spt + kk * 32, 16, 1024),
                             ptx::umma_desc_sw128(sdo + kk * 2048, T64, 1024), id_g, (m > 0 || kk > 0));
            ptx::mma_bf16_ss(t_dk, ptx::umma_desc_sw128(sdst + kk * 32, 16, 1024),
                             ptx::umma_desc_sw128(sq + kk * 2048, T64, 1024), id_g, (m > 0 || kk > 0));
          }
          ptx::mma_commit(&pd_done[w]);
          ptx::mma_commit(&q_empty[st]);
        }
      }
    }
  } else if (warp >= 4) {
    const int wg = (warp - 4) >> 2;  // blocks n = wg, wg + 2, ...
    const int q = warp & 3;
    const int r = q * 32 + lane;  // key row within the tile
    const int key = kt * 128 + r;
    const uint32_t lanes = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t t_st = tmem + 128 * wg, t_dpt = t_st + 64;
    int it = 0;
    for (int n = wg; n < N; n += 2, ++it) {
      const int st = n % NS, i = i0 + n;
      const bool diag = causal && i < i0 + 2;
      ptx::mbar_wait(&q_full[st], (n / NS) & 1);  // lse / delta of this block visible
      ptx::mbar_wait(&s_full[wg], it & 1);
      ptx::tc_fence_after();
      uint32_t s0[32], s1[32], d0[32], d1[32];
      ptx::tmem_ld_32x32b_x32(t_st + lanes, s0);
      ptx::tmem_ld_32x32b_x32(t_st + lanes + 32, s1);
      ptx::tmem_ld_32x32b_x32(t_dpt + lanes, d0);
      ptx::tmem_ld_32x32b_x32(t_dpt + lanes + 32, d1);
      ptx::tmem_ld_wait();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&s_empty[wg]);
      const float4* ls4 = reinterpret_cast<const float4*>(sm + L::LD + st * 512);
      uint32_t pp[32], dd[32];
#pragma unroll
      for (int c4 = 0; c4 < 16; ++c4) {
        const float4 lq = ls4[c4], dq = ls4[16 + c4];
        const float lv[4] = {lq.x, lq.y, lq.z, lq.w}, dv[4] = {dq.x, dq.y, dq.z, dq.w};
        float p[4], g[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int cc = 4 * c4 + u;
          const float s = __uint_as_float(cc < 32 ? s0[cc] : s1[cc - 32]);
          const float dp = __uint_as_float(cc < 32 ? d0[cc] : d1[cc - 32]);
          p[u] = ex2(fmaf(s, scale_log2, -lv[u]));
          g[u] = dp - dv[u];
        }
        if (diag) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (i * 64 + 4 * c4 + u < key) p[u] = 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) g[u] *= p[u];
        pp[2 * c4] = pack2(p[0], p[1]);
        pp[2 * c4 + 1] = pack2(p[2], p[3]);
        dd[2 * c4] = pack2(g[0], g[1]);
        dd[2 * c4 + 1] = pack2(g[2], g[3]);
      }
      if (it > 0) ptx::mbar_wait(&pd_done[wg], (it - 1) & 1);  // previous P^T / dS^T consumed
      uint8_t* spt = sm + L::PT + wg * T128;
      uint8_t* sdst = sm + L::DST + wg * T128;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t off = ptx::sw128_offset(r, u);
        *reinterpret_cast<uint4*>(spt + off) = make_uint4(pp[4 * u], pp[4 * u + 1], pp[4 * u + 2], pp[4 * u + 3]);
        *reinterpret_cast<uint4*>(sdst + off) = make_uint4(dd[4 * u], dd[4 * u + 1], dd[4 * u + 2], dd[4 * u + 3]);
      }
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive(&p_full[wg]);
    }
    if (it > 0) ptx::mbar_wait(&pd_done[wg], (it - 1) & 1);
    asm volatile("bar.sync 1, 256;" ::: "memory");  // both warpgroups drained: dK, dV final
    ptx::tc_fence_after();
    // warpgroup 0 writes dK, warpgroup 1 writes dV
    const size_t ld = static_cast<size_t>(3) * H * D;
    bf16* dst = dqkv + (static_cast<size_t>(row0) + key) * ld + (wg == 0 ? H * D : 2 * H * D) + h * D;
    const uint32_t src = (wg == 0 ? t_dk : t_dv) + lanes;
    const float mul = wg == 0 ? scale : 1.f;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t a[32];
      ptx::tmem_ld_32x32b_x32(src + c * 32, a);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float f[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(a[8 * u + e]) * mul;
        store8(dst + c * 32 + 8 * u, f);
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<L::TMEM_COLS>(tmem);
  }
}

// ==================================================================== dQ
// dS never touches shared memory: the softmax threads write it (bf16) over the TMEM
// columns of the S tile they just read, and dQ += dS K_j reads it as the TMEM A operand
// (tcgen05 "TS" form).  Three S/dP TMEM buffers let S_{n+1} issue while dQ_{n-1} is still
// reading buffer n-1; the freed smem goes into a 5-deep K/V TMA ring (TMA latency on this
// path is ~3-5k cycles, profiles/r01_attn_fwd_trace.txt).
template <int D>
struct QSmem {
  static constexpr int NB = D / 64;
  static constexpr int NS = D == 128 ? 5 : 8;     // K / V ring depth
  static constexpr uint32_t Q = 0;
  static constexpr uint32_t DO = Q + NB * T128;
  static constexpr uint32_t K = DO + NB * T128;   // NS stages of NB x T64
  static constexpr uint32_t V = K + NS * NB * T64;
  static constexpr uint32_t BAR = V + NS * NB * T64;
  static constexpr uint32_t BYTES = BAR + 256;
  static constexpr uint32_t TMEM_COLS = 512;
};

template <int D>
__global__ void __launch_bounds__(384, 1)
    fa_bwd_dq_kernel(const __grid_constant__ CUtensorMap qkv128, const __grid_constant__ CUtensorMap qkv64,
                     const __grid_constant__ CUtensorMap do128, const float* __restrict__ lse,
                     const float* __restrict__ delta, bf16* __restrict__ dqkv, int seq, int H, int n_qt,
                     float scale_log2, float scale, int causal) {
  using L = QSmem<D>;
  constexpr int NS = L::NS;
  extern __shared__ uint8_t smem_raw[];
  long long* const dbg_ = blockIdx.x == 0 ? g_bw_dbg : nullptr;  // trace hook, read once
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~static_cast<uintptr_t>(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* kv_full = bar + 1;        // [NS]
  uint64_t* kv_empty = kv_full + 8;   // [NS]
  uint64_t* s_full = kv_empty + 8;    // [3] TMEM S/dP buffers
  uint64_t* s_empty = s_full + 3;     // [3]
  uint64_t* p_full = s_empty + 3;     // [2] per warpgroup: dS written
  uint64_t* dq_done = p_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = n_qt - 1 - static_cast<int>(blockIdx.x % n_qt);  // heavy first
  const int hb = static_cast<int>(blockIdx.x / n_qt);
  const int h = hb % H, b = hb / H;
  const int row0 = b * seq;
  const int N = causal ? 2 * qt + 2 : seq / 64;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&qkv128);
    ptx::tma_prefetch(&qkv64);
    ptx::tma_prefetch(&do128);
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < NS; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    for (int s = 0; s < 3; ++s) {
      ptx::mbar_init(&s_full[s], 1);
      ptx::mbar_init(&s_empty[s], 1);
    }
    ptx::mbar_init(&p_full[0], 128);
    ptx::mbar_init(&p_full[1], 128);
    ptx::mbar_init(dq_done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<L::TMEM_COLS>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM: buffer b: S at 128b (dS bf16 overwrites its first 32 columns), dP at 128b + 64;
  // dQ at 384.
  const uint32_t t_dq = tmem + 384;
  if (threadIdx.x == 0) BW_T(7, 0);

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(q_full, 2 * L::NB * T128);
      for (int c = 0; c < L::NB; ++c) {
        ptx::tma_load_2d(sm + L::Q + c * T128, &qkv128, q_full, h * D + 64 * c, row0 + qt * 128);
        ptx::tma_load_2d(sm + L::DO + c * T128, &do128, q_full, h * D + 64 * c, row0 + qt * 128);
      }
      for (int n = 0; n < N; ++n) {
        const int st = n % NS;
        ptx::mbar_wait(&kv_empty[st], ((n / NS) & 1) ^ 1);
        BW_T(6, n);
        ptx::mbar_arrive_expect_tx(&kv_full[st], 2 * L::NB * T64);
        for (int c = 0; c < L::NB; ++c) {
          ptx::tma_load_2d(sm + L::K + (st * L::NB + c) * T64, &qkv64, &kv_full[st], H * D + h * D + 64 * c,
                           row0 + n * 64);
          ptx::tma_load_2d(sm + L::V + (st * L::NB + c) * T64, &qkv64, &kv_full[st], 2 * H * D + h * D + 64 * c,
                           row0 + n * 64);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = ptx::idesc_bf16_f32(128, 64, false, false);
      constexpr uint32_t id_g = ptx::idesc_bf16_f32(128, D, false, true);
      const uint32_t sq = ptx::smem_u32(sm + L::Q), sdo = ptx::smem_u32(sm + L::DO);
      ptx::mbar_wait(q_full, 0);
      for (int n = 0; n <= N; ++n) {
        if (n < N) {
          const int st = n % NS, bf = n % 3;
          const uint32_t t_s = tmem + 128 * bf, t_dp = t_s + 64;
          ptx::mbar_wait(&kv_full[st], (n / NS) & 1);
          BW_T(0, n);
          ptx::mbar_wait(&s_empty[bf], ((n / 3) & 1) ^ 1);
          BW_T(1, n);
          ptx::tc_fence_after();
          const uint32_t sk = ptx::smem_u32(sm + L::K + st * L::NB * T64);
          const uint32_t sv = ptx::smem_u32(sm + L::V + st * L::NB * T64);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t oa = (kk >> 2) * T128 + (kk & 3) * 32, ob = (kk >> 2) * T64 + (kk & 3) * 32;
            ptx::mma_bf16_ss(t_s, ptx::umma_desc_sw128(sq + oa, 16, 1024), ptx::umma_desc_sw128(sk + ob, 16, 1024),
                             id_s, kk > 0);
            ptx::mma_bf16_ss(t_dp, ptx::umma_desc_sw128(sdo + oa, 16, 1024),
                             ptx::umma_desc_sw128(sv + ob, 16, 1024), id_s, kk > 0);
          }
          ptx::mma_commit(&s_full[bf]);
        }
        if (n > 0) {
          const int m = n - 1, st = m % NS, bf = m % 3;
          ptx::mbar_wait(&p_full[m & 1], (m >> 1) & 1);
          BW_T(2, m);
          ptx::tc_fence_after();
          const uint32_t sk = ptx::smem_u32(sm + L::K + st * L::NB * T64);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // K = 64 keys, 16 per instruction (8 TMEM columns)
            ptx::mma_bf16_ts(t_dq, tmem + 128 * bf + kk * 8, ptx::umma_desc_sw128(sk + kk * 2048, T64, 1024), id_g,
                             (m > 0 || kk > 0));
          ptx::mma_commit(&s_empty[bf]);
          ptx::mma_commit(&kv_empty[st]);
        }
      }
      ptx::mma_commit(dq_done);
    }
  } else if (warp >= 4) {
    const int wg = (warp - 4) >> 2;
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int qrow = qt * 128 + r;
    const uint32_t lanes = static_cast<uint32_t>(q * 32) << 16;
    const size_t bh = (static_cast<size_t>(b) * H + h) * seq;
    const float nl = -lse[bh + qrow], dl = delta[bh + qrow];
    int it = 0;
    for (int n = wg; n < N; n += 2, ++it) {
      const int bf = n % 3;
      const uint32_t t_s = tmem + 128 * bf + lanes, t_dp = t_s + 64;
      const bool diag = causal && n >= 2 * qt;
      ptx::mbar_wait(&s_full[bf], (n / 3) & 1);
      if (lane == 0 && q == 0) BW_T(3, n);
      ptx::tc_fence_after();
      uint32_t s0[32], s1[32], d0[32], d1[32];
      ptx::tmem_ld_32x32b_x32(t_s, s0);
      ptx::tmem_ld_32x32b_x32(t_s + 32, s1);
      ptx::tmem_ld_32x32b_x32(t_dp, d0);
      ptx::tmem_ld_32x32b_x32(t_dp + 32, d1);
      ptx::tmem_ld_wait();
      float g[64];
#pragma unroll
      for (int cc = 0; cc < 64; ++cc) {
        const float sv = __uint_as_float(cc < 32 ? s0[cc] : s1[cc - 32]);
        const float dp = __uint_as_float(cc < 32 ? d0[cc] : d1[cc - 32]);
        g[cc] = ex2(fmaf(sv, scale_log2, nl)) * (dp - dl);
      }
      if (diag) {
#pragma unroll
        for (int cc = 0; cc < 64; ++cc)
          if (n * 64 + cc > qrow) g[cc] = 0.f;
      }
      uint32_t gg[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) gg[c] = pack2(g[2 * c], g[2 * c + 1]);
      if (lane == 0 && q == 0) BW_T(4, n);
      ptx::tmem_st_32x32b_x32(t_s, gg);  // dS (bf16 pairs) over the S columns just read
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&p_full[wg]);
      if (lane == 0 && q == 0) BW_T(5, n);
    }
    ptx::mbar_wait(dq_done, 0);
    ptx::tc_fence_after();
    // each warpgroup writes half of the D columns
    bf16* rowq = dqkv + (static_cast<size_t>(row0) + qrow) * (static_cast<size_t>(3) * H * D) + h * D;
#pragma unroll 1
    for (int c = wg * (D / 64); c < (wg + 1) * (D / 64); ++c) {
      uint32_t a[32];
      ptx::tmem_ld_32x32b_x32(t_dq + lanes + c * 32, a);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float f[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(a[8 * u + e]) * scale;
        store8(rowq + c * 32 + 8 * u, f);
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<L::TMEM_COLS>(tmem);
  }
}

template <class K>
int set_smem(K k, size_t bytes) {
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}

template <int D>
int launch_bwd_tc(const bf16* qkv, const bf16* dout, const float* lse, const float* delta, bf16* dqkv, int B,
                  int S, int H, int causal, cudaStream_t st) {
  CUtensorMap q128, q64, o128, o64;
  const uint64_t ldq = static_cast<uint64_t>(3) * H * D, ldo = static_cast<uint64_t>(H) * D;
  const uint64_t rows = static_cast<uint64_t>(B) * S;
  if (!tma_map_bf16_2d(&q128, qkv, ldq, rows, ldq, 64, 128) || !tma_map_bf16_2d(&q64, qkv, ldq, rows, ldq, 64, 64) ||
      !tma_map_bf16_2d(&o128, dout, ldo, rows, ldo, 64, 128) || !tma_map_bf16_2d(&o64, dout, ldo, rows, ldo, 64, 64))
    return AMDP_ERR_TMA;
  const float scale = 1.f / sqrtf(static_cast<float>(D));
  const float scale_log2 = 1.4426950408889634f * scale;
  static bool attr = false;
  const size_t smem_kv = KvSmem<D>::BYTES + 1024, smem_q = QSmem<D>::BYTES + 1024;
  if (!attr) {
    int e = set_smem(fa_bwd_dkdv_kernel<D>, smem_kv);
    if (e) return e;
    e = set_smem(fa_bwd_dq_kernel<D>, smem_q);
    if (e) return e;
    attr = true;
  }
  const int nt = S / 128;
  fa_bwd_dkdv_kernel<D><<<nt * H * B, 384, smem_kv, st>>>(q128, q64, o64, lse, delta, dqkv, S, H, nt, scale_log2,
                                                          scale, causal);
  fa_bwd_dq_kernel<D><<<nt * H * B, 384, smem_q, st>>>(q128, q64, o128, lse, delta, dqkv, S, H, nt, scale_log2,
                                                       scale, causal);
  return cudaGetLastError();
}

}  // namespace

// Used by amdp_attention_bwd (after the delta pre-pass) when the tensor-core path applies.
int attention_bwd_tc(const bf16* qkv, const bf16* dout, const float* lse, const float* delta, bf16* dqkv, int B,
                     int S, int H, int D, int causal, cudaStream_t st) {
  if (S % 128 != 0) return AMDP_ERR_UNSUPPORTED;
  if (D == 128) return launch_bwd_tc<128>(qkv, dout, lse, delta, dqkv, B, S, H, causal, st);
  if (D == 64) return launch_bwd_tc<64>(qkv, dout, lse, delta, dqkv, B, S, H, causal, st);
  return AMDP_ERR_UNSUPPORTED;
}

}  // namespace amdp

extern "C" int amdp_debug_attention_bwd_trace(long long* device_buf) {
  return cudaMemcpyToSymbol(amdp::g_bw_dbg, &device_buf, sizeof(device_buf));
}
