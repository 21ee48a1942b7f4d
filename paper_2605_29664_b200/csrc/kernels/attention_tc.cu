// Flash-attention forward on the 5th-generation tensor cores (sm_100a).
//
// One CTA per (128-query tile, head, sequence), 12 warps:
//   warp 0     : TMA producer — Q once, K_j and V_j (128 keys) into separate 2-stage rings,
//                straight out of the packed qkv activation rows (no repacking);
//   warp 1     : tcgen05.mma issuer — S_j = Q K_j^T (M=128, N=128, K=D) into TMEM buffer
//                S[j%2]; O[j%2] += P[j%2] V_j (M=128, N=D, K=128), P from swizzled smem,
//                V consumed MN-major;
//   warp 2     : TMEM allocator (512 columns: S0 | S1 | O0 | O1);
//   warps 4-7  : softmax warpgroup 0 — even KV blocks;  warps 8-11 : warpgroup 1 — odd.
// Each warpgroup runs an independent online softmax (its own running max m, sum l and
// O accumulator) over its half of the KV blocks, so the two never synchronise per block;
// thread t of a warpgroup owns query row t (TMEM lane t).  The halves are merged once at
// the end: O = (O0 2^(m0-m) + O1 2^(m1-m)) / (l0 2^(m0-m) + l1 2^(m1-m)).
// Per score: one FFMA (scale folded into the exponent), one ex2.approx, one FADD, half a
// pack; the running max is only pushed into O (rescale in TMEM) when it grows by more
// than 2^8 — exact, since P and O then share the stale reference.
// LSE is stored in the log2 domain with the softmax scale folded in, the convention the
// backward kernels in attention.cu consume.
#include "common.cuh"
#include "sm100_ptx.cuh"
#include "tma_host.hpp"

namespace amdp {
namespace {

constexpr int FA_BQ = 128, FA_BKV = 128, FA_THREADS = 384;

// Diagnostics: when set (amdp_debug_attention_trace), CTA 0 records clock64() at each
// pipeline hand-off into this buffer (slot layout in scripts/attn_trace.py).
__device__ long long* g_fa_dbg = nullptr;
#define FA_T(slot, j)                                             \
  do {                                                            \
    if (g_fa_dbg != nullptr && blockIdx.x == 0) g_fa_dbg[(slot)*64 + (j)] = clock64(); \
  } while (0)
constexpr uint32_t TILE = 16384;  // one [128 rows][64 bf16] SW128 tile

template <int D>
struct FaSmem {
  static constexpr int NB = D / 64;  // 64-wide column blocks per row tile
  static constexpr uint32_t Q = 0;
  static constexpr uint32_t K = Q + NB * TILE;      // 2 stages
  static constexpr uint32_t V = K + 2 * NB * TILE;  // 2 stages
  static constexpr uint32_t P = V + 2 * NB * TILE;  // 2 buffers of [128 q][128 keys]
  static constexpr uint32_t XCH = P + 4 * TILE;     // warpgroup-1 (m, l) hand-off
  static constexpr uint32_t BAR = XCH + 2 * 128 * 4;
  static constexpr uint32_t BYTES = BAR + 256;
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int D>
__global__ void __launch_bounds__(FA_THREADS, 1)
    fa_fwd_tc_kernel(const __grid_constant__ CUtensorMap qkv_map, bf16* __restrict__ out,
                     float* __restrict__ lse, int seq, int H, int n_qt, float scale_log2,
                     int causal) {
  using L = FaSmem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~static_cast<uintptr_t>(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;   // [2]
  uint64_t* k_empty = bar + 3;  // [2]
  uint64_t* v_full = bar + 5;   // [2]
  uint64_t* v_empty = bar + 7;  // [2]
  uint64_t* s_full = bar + 9;   // [2] per warpgroup
  uint64_t* s_empty = bar + 11; // [2]
  uint64_t* p_full = bar + 13;  // [2]
  uint64_t* pv_done = bar + 15; // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 17);
  float* xch = reinterpret_cast<float*>(sm + L::XCH);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = n_qt - 1 - static_cast<int>(blockIdx.x % n_qt);  // heavy (late) tiles first
  const int hb = static_cast<int>(blockIdx.x / n_qt);
  const int h = hb % H, b = hb / H;
  const int nkv = causal ? qt + 1 : seq / FA_BKV;
  const int row0 = b * seq;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&qkv_map);
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&k_full[s], 1);
      ptx::mbar_init(&k_empty[s], 1);
      ptx::mbar_init(&v_full[s], 1);
      ptx::mbar_init(&v_empty[s], 1);
      ptx::mbar_init(&s_full[s], 1);
      ptx::mbar_init(&s_empty[s], 128);
      ptx::mbar_init(&p_full[s], 128);
      ptx::mbar_init(&pv_done[s], 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) FA_T(10, 0);

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(q_full, L::NB * TILE);
      for (int c = 0; c < L::NB; ++c)
        ptx::tma_load_2d(sm + L::Q + c * TILE, &qkv_map, q_full, h * D + 64 * c, row0 + qt * FA_BQ);
      // K_j runs one block ahead of V_j: S_j needs K_j before PV_{j-1} needs V_{j-1}
      for (int j = 0; j <= nkv; ++j) {
        if (j < nkv) {
          const int st = j & 1;
          ptx::mbar_wait(&k_empty[st], ((j >> 1) & 1) ^ 1);
          FA_T(8, j);
          ptx::mbar_arrive_expect_tx(&k_full[st], L::NB * TILE);
          for (int c = 0; c < L::NB; ++c)
            ptx::tma_load_2d(sm + L::K + (st * L::NB + c) * TILE, &qkv_map, &k_full[st],
                             H * D + h * D + 64 * c, row0 + j * FA_BKV);
        }
        if (j > 0) {
          const int jj = j - 1, st = jj & 1;
          ptx::mbar_wait(&v_empty[st], ((jj >> 1) & 1) ^ 1);
          FA_T(9, jj);
          ptx::mbar_arrive_expect_tx(&v_full[st], L::NB * TILE);
          for (int c = 0; c < L::NB; ++c)
            ptx::tma_load_2d(sm + L::V + (st * L::NB + c) * TILE, &qkv_map, &v_full[st],
                             2 * H * D + h * D + 64 * c, row0 + jj * FA_BKV);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = ptx::idesc_bf16_f32(FA_BQ, FA_BKV, false, false);
      constexpr uint32_t id_o = ptx::idesc_bf16_f32(FA_BQ, D, false, true);
      const uint32_t sq = ptx::smem_u32(sm + L::Q);
      ptx::mbar_wait(q_full, 0);
      for (int j = 0; j <= nkv; ++j) {
        if (j < nkv) {
          const int st = j & 1;  // K stage == S buffer == warpgroup
          ptx::mbar_wait(&k_full[st], (j >> 1) & 1);
          FA_T(0, j);
          ptx::mbar_wait(&s_empty[st], ((j >> 1) & 1) ^ 1);
          FA_T(1, j);
          ptx::tc_fence_after();
          const uint32_t sk = ptx::smem_u32(sm + L::K + st * L::NB * TILE);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * TILE + (kk & 3) * 32;
            ptx::mma_bf16_ss(tmem + st * FA_BKV, ptx::umma_desc_sw128(sq + off, 16, 1024),
                             ptx::umma_desc_sw128(sk + off, 16, 1024), id_s, kk > 0 ? 1u : 0u);
          }
          ptx::mma_commit(&s_full[st]);
          ptx::mma_commit(&k_empty[st]);
        }
        if (j > 0) {
          const int jj = j - 1, w = jj & 1;
          ptx::mbar_wait(&v_full[w], (jj >> 1) & 1);
          FA_T(2, jj);
          ptx::mbar_wait(&p_full[w], (jj >> 1) & 1);
          FA_T(3, jj);
          ptx::tc_fence_after();
          const uint32_t sv = ptx::smem_u32(sm + L::V + w * L::NB * TILE);
          const uint32_t sp = ptx::smem_u32(sm + L::P + w * 2 * TILE);
#pragma unroll
          for (int kk = 0; kk < FA_BKV / 16; ++kk) {
            ptx::mma_bf16_ss(tmem + 256 + w * 128,
                             ptx::umma_desc_sw128(sp + (kk >> 2) * TILE + (kk & 3) * 32, 16, 1024),
                             ptx::umma_desc_sw128(sv + kk * 2048, TILE, 1024), id_o,
                             (jj >= 2 || kk > 0) ? 1u : 0u);
          }
          ptx::mma_commit(&pv_done[w]);
          ptx::mma_commit(&v_empty[w]);
        }
      }
    }
  } else if (warp >= 4) {
    const int wg = (warp - 4) >> 2;      // softmax warpgroup: KV blocks j = wg, wg + 2, ...
    const int q = warp & 3;              // TMEM lane quadrant
    const int r = q * 32 + lane;         // query row within the tile
    const int qrow = qt * FA_BQ + r;
    const uint32_t lanes = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t ts = lanes + wg * FA_BKV;
    const uint32_t to = lanes + 256 + wg * 128;
    uint8_t* sp = sm + L::P + wg * 2 * TILE;
    float m_ref = -INFINITY, l = 0.f;
    int it = 0;
    for (int j = wg; j < nkv; j += 2, ++it) {
      const bool diag = causal && j == qt;
      ptx::mbar_wait(&s_full[wg], it & 1);
      if (lane == 0 && (warp & 3) == 0) FA_T(4, j);
      ptx::tc_fence_after();
      // pass 1: row max of the raw scores (scale > 0 commutes with max)
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < FA_BKV / 32; ++c) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(ts + c * 32, v);
        ptx::tmem_ld_wait();
        if (diag) {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (j * FA_BKV + c * 32 + e <= qrow) mx = fmaxf(mx, __uint_as_float(v[e]));
        } else {
#pragma unroll
          for (int e = 0; e < 32; e += 2) mx = fmaxf(mx, fmaxf(__uint_as_float(v[e]), __uint_as_float(v[e + 1])));
        }
      }
      const float m_new = fmaxf(m_ref, mx * scale_log2);
      if (lane == 0 && (warp & 3) == 0) FA_T(5, j);
      if (it > 0) ptx::mbar_wait(&pv_done[wg], (it - 1) & 1);  // P[wg] free, O[wg] settled
      if (lane == 0 && (warp & 3) == 0) FA_T(6, j);
      if (it == 0) {
        m_ref = m_new;
      } else if (__any_sync(0xffffffffu, m_new > m_ref + 8.f)) {  // warp-collective TMEM ops
        const float alpha = ex2(m_ref - m_new);
        ptx::tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          uint32_t o[32];
          ptx::tmem_ld_32x32b_x32(to + c * 32, o);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
          ptx::tmem_st_32x32b_x32(to + c * 32, o);
        }
        ptx::tmem_st_wait();
        l *= alpha;
        m_ref = m_new;
      }
      const float nm = -m_ref;
      // pass 2: P = 2^(s*scale - m) -> bf16 -> swizzled smem
#pragma unroll
      for (int c = 0; c < FA_BKV / 32; ++c) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(ts + c * 32, v);
        ptx::tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float p0 = ex2(fmaf(__uint_as_float(v[e]), scale_log2, nm));
          float p1 = ex2(fmaf(__uint_as_float(v[e + 1]), scale_log2, nm));
          if (diag) {
            const int k0 = j * FA_BKV + c * 32 + e;
            if (k0 > qrow) p0 = 0.f;
            if (k0 + 1 > qrow) p1 = 0.f;
          }
          l += p0 + p1;
          __nv_bfloat162 t2 = __floats2bfloat162_rn(p0, p1);
          pk[e >> 1] = *reinterpret_cast<uint32_t*>(&t2);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          *reinterpret_cast<uint4*>(sp + (c >> 1) * TILE + ptx::sw128_offset(r, (c & 1) * 4 + u)) =
              make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&s_empty[wg]);
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive(&p_full[wg]);
      if (lane == 0 && (warp & 3) == 0) FA_T(7, j);
    }
    // drain this warpgroup's last PV
    if (it > 0) ptx::mbar_wait(&pv_done[wg], (it - 1) & 1);
    ptx::tc_fence_after();
    // merge the two halves: warpgroup 1 hands (m, l) to warpgroup 0 through smem
    if (wg == 1) {
      xch[r] = m_ref;
      xch[128 + r] = l;
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (wg == 0) {
      const bool has1 = nkv > 1;
      const float m1 = has1 ? xch[r] : -INFINITY, l1 = has1 ? xch[128 + r] : 0.f;
      const float m = fmaxf(m_ref, m1);
      const float a0 = ex2(m_ref - m), a1 = has1 ? ex2(m1 - m) : 0.f;
      const float inv = 1.f / (l * a0 + l1 * a1);
      const float c0 = a0 * inv, c1 = a1 * inv;
      bf16* orow = out + (static_cast<size_t>(row0) + qrow) * (static_cast<size_t>(H) * D) + h * D;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o0[32], o1[32];
        ptx::tmem_ld_32x32b_x32(lanes + 256 + c * 32, o0);
        ptx::tmem_ld_32x32b_x32(lanes + 384 + c * 32, o1);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float f[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            f[e] = __uint_as_float(o0[8 * u + e]) * c0 + (has1 ? __uint_as_float(o1[8 * u + e]) * c1 : 0.f);
          store8(orow + c * 32 + 8 * u, f);
        }
      }
      lse[(static_cast<size_t>(b) * H + h) * seq + qrow] = m + log2f(l * a0 + l1 * a1);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

template <int D>
int launch_fa_fwd(const bf16* qkv, bf16* out, float* lse, int B, int S, int H, int causal, cudaStream_t st) {
  CUtensorMap map;
  if (!tma_map_bf16_2d(&map, qkv, static_cast<uint64_t>(3) * H * D, static_cast<uint64_t>(B) * S,
                       static_cast<uint64_t>(3) * H * D, 64, 128))
    return AMDP_ERR_TMA;
  const size_t smem = FaSmem<D>::BYTES + 1024;
  auto k = fa_fwd_tc_kernel<D>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int n_qt = S / FA_BQ;
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(D));
  k<<<n_qt * H * B, FA_THREADS, smem, st>>>(map, out, lse, S, H, n_qt, scale_log2, causal);
  return cudaGetLastError();
}

}  // namespace

// Used by amdp_attention_fwd when the tensor-core path applies.
int attention_fwd_tc(const bf16* qkv, bf16* out, float* lse, int B, int S, int H, int D, int causal,
                     cudaStream_t st) {
  if (S % FA_BQ != 0) return AMDP_ERR_UNSUPPORTED;
  if (D == 128) return launch_fa_fwd<128>(qkv, out, lse, B, S, H, causal, st);
  if (D == 64) return launch_fa_fwd<64>(qkv, out, lse, B, S, H, causal, st);
  return AMDP_ERR_UNSUPPORTED;
}

}  // namespace amdp

// Diagnostics hook (see g_fa_dbg): device buffer of >= 11 * 64 int64, or NULL to disable.
extern "C" int amdp_debug_attention_trace(long long* device_buf) {
  return cudaMemcpyToSymbol(amdp::g_fa_dbg, &device_buf, sizeof(device_buf));
}
