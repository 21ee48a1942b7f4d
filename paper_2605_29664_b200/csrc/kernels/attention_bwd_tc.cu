// Flash-attention backward on the 5th-generation tensor cores (sm_100a).
//
// Default (head_dim 64 / 128): the dK/dV kernel below also stores dS^T (DS_CHUNK layout) and
// fa_bwd_dq_gemm_kernel computes dQ = scale * dS K from it — five GEMM units and one softmax
// pass.  The dQ kernel described second recomputes S, dP and the softmax instead; it serves
// head_dim 80 and AMDP_ATTN_DQ=recompute (A/B).
// Deterministic kernels (no atomics), each with its accumulators in TMEM:
//   dK/dV : one CTA per (128-key tile, head, sequence), looping over 64-query halves:
//           S^T = K Q_i^T, dP^T = V dO_i^T                    (SS, M=128 keys, N=64 queries)
//           P^T = 2^(S^T c - lse), dS^T = P^T (dP^T - delta)  (thread = key, one warpgroup
//                                                              per half, overlapping the
//                                                              other half's MMAs)
//           dV += P^T dO_i, dK += dS^T Q_i                    (TS: P^T / dS^T from TMEM)
//   dQ    : one CTA per (128-query tile, head, sequence), looping over 128-key blocks:
//           S = Q K_j^T (TS, Q in TMEM), dP = dO V_j^T; dS = P (dP - delta); dQ += dS K_j (TS)
//           dS goes to its own TMEM columns, so S/dP's TMEM frees as soon as the softmax
//           threads have loaded it, letting S_{j+1} overlap the dS math of block j.
// The backward softmax is elementwise given lse and delta, so the two softmax warpgroups
// split each block by columns and no cross-thread reduction is needed.
// tcgen05.mma issue blocks once ~5 MMAs are queued (the issuing thread runs at the pipe's
// pace), so each kernel issues its MMA groups in the order their inputs become ready.  The
// issuing warp runs converged and elect.sync picks the lane inside each MMA's asm: with a
// single-lane branch the compiler wrapped every UTCHMMA in an ELECT / R2UR.BROADCAST /
// BRA.U.ANY loop (~15 instructions), which made issue, not the tensor pipe, the limit for
// the N=64 / N=128 MMAs here (dQ kernel 166 -> 146 us).
// lse / delta use the forward's log2-domain convention (softmax scale folded in);
// delta = rowsum(dO * O) comes from attn_bwd_delta_vec_kernel (attention.cu).
#include <cstring>

#include "common.cuh"
#include "sm100_ptx.cuh"
#include "tma_host.hpp"

namespace amdp {
namespace {

constexpr uint32_t T128 = 16384;  // [128 rows][64 bf16] SW128 tile
#ifndef FA_BWD_POLY_PAIRS
#define FA_BWD_POLY_PAIRS 0  // dQ softmax: exponent pairs (of 4) on the FMA pipe; 0 measured best (MUFU is not the limit)
#endif

// Diagnostics (amdp_debug_attention_bwd_trace): CTA 0 of the dQ kernel records clock64().
__device__ long long* g_bw_dbg = nullptr;
#define BW_T(slot, j)                                                   \
  do {                                                                  \
    if (dbg_ != nullptr && (j) < 64) dbg_[(slot)*64 + (j)] = clock64(); \
  } while (0)

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 16-byte global store that does not allocate in L1 (the dS^T stream would evict lse / delta)
__device__ __forceinline__ void st_na_v4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&t);
}
__device__ __forceinline__ void tmem_st_x16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
// Writes NCOLS fp32 TMEM columns of this thread's lane, times mul, as bf16 to dst.
template <int NCOLS>
__device__ __forceinline__ void tmem_row_to_global(uint32_t src, bf16* dst, float mul) {
#pragma unroll 1
  for (int c = 0; c < NCOLS / 32; ++c) {
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
  constexpr int T0 = (NCOLS / 32) * 32;  // head_dim 80: 16- / 8-column tails
  if constexpr (NCOLS % 32 >= 16) {
    uint32_t a[16];
    ptx::tmem_ld_32x32b_x16(src + T0, a);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      float f[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(a[8 * u + e]) * mul;
      store8(dst + T0 + 8 * u, f);
    }
  }
  if constexpr (NCOLS % 16 == 8) {
    constexpr int T1 = T0 + (NCOLS % 32 >= 16 ? 16 : 0);
    uint32_t a[8];
    ptx::tmem_ld_32x32b_x8(src + T1, a);
    ptx::tmem_ld_wait();
    float f[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(a[e]) * mul;
    store8(dst + T1, f);
  }
}

// ==================================================================== dK / dV
// The 128-query block is processed as two 64-query halves a / b, one per softmax
// warpgroup, with the MMAs interleaved so each half's softmax overlaps the other half's
// tensor work:   dVdK_a(i) | S_a(i+1) | dVdK_b(i) | S_b(i+1) | ...   (S_x = S^T_x + dP^T_x)
// Q / dO stream in half-block units through a 5-deep ring, so a unit's load starts ~3
// half-block MMA groups ahead of its first use; lse / delta are read from L2 (broadcast).
constexpr uint32_t T64 = 8192;  // [64 rows][64 bf16] SW128 tile

// dS^T scratch for the dQ GEMM: per (sequence, head), one 16 KB chunk per (128-key tile kt,
// 64-query half-block) the dK/dV kernel visits, holding dS [64 queries][128 keys] bf16 as two
// 8 KB key halves, each [8 query groups][64 keys][8 queries] (16-byte unit of key r, queries
// 8v..8v+7 at (r / 64) 8192 + v 1024 + (r % 64) 16).  That is the no-swizzle MN-major core-
// matrix layout of the MMA operand (8 keys x 16 bytes contiguous), so the dQ kernel moves a key
// half with one bulk copy and hands it to the MMA as is, and the dK/dV threads (thread = key)
// store it coalesced: a warp's 16-byte stores of one query group cover 512 contiguous bytes.
// Key tile kt's chunks are consecutive (causal: query blocks kt..nqb-1, else all), two per
// 128-query block.
constexpr uint32_t DS_CHUNK = 16384;
__host__ __device__ inline int ds_chunks_per_head(int nqb, int causal) { return causal ? nqb * (nqb + 1) : 2 * nqb * nqb; }
__host__ __device__ inline int ds_chunk_offset(int nqb, int kt, int causal) {
  return causal ? kt * (2 * nqb - kt + 1) : 2 * kt * nqb;
}

// head_dim 80 uses the 128-wide layout (two SW128 boxes per row tile; see attention_tc.cu):
// K-dim loops run D/16 steps, the D-wide outputs are N = D MMAs, TMEM keeps 128-column slots.
template <int D>
struct KvSmem {
  static constexpr int NB = (D + 63) / 64;
  static constexpr int NU = NB == 2 ? 5 : 10;         // half-block units in flight
  static constexpr uint32_t UNIT = 2 * NB * T64;      // Q half, dO half
  static constexpr uint32_t K = 0;
  static constexpr uint32_t V = K + NB * T128;
  static constexpr uint32_t U = V + NB * T128;        // NU units
  static constexpr uint32_t BAR = U + NU * UNIT;
  static constexpr uint32_t BYTES = BAR + 256;
};

template <int D, bool KPAD>
__global__ void __launch_bounds__(384, 1)
    fa_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap kv_map, const __grid_constant__ CUtensorMap qkv_map,
                       const __grid_constant__ CUtensorMap do_map, const float* __restrict__ lse, const float* __restrict__ delta, bf16* __restrict__ dqkv,
                       int seq, int H, int n_kt, int BH, float scale_log2, float scale, int causal,
                       const int32_t* __restrict__ key_len, uint8_t* __restrict__ ds_ws) {
  using L = KvSmem<D>;
  constexpr int NU = L::NU;
  extern __shared__ uint8_t smem_raw[];
  long long* const dbg_ = blockIdx.x == 0 && g_bw_dbg != nullptr ? g_bw_dbg + 16 * 64 : nullptr;  // trace hook
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~static_cast<uintptr_t>(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* kv_full = bar + 0;
  uint64_t* u_full = bar + 1;        // [NU]
  uint64_t* u_empty = u_full + 10;   // [NU]
  uint64_t* s_full = u_empty + 10;   // [2] per half
  uint64_t* p_full = s_full + 2;     // [2] 128 arrivals: P^T / dS^T of the half in TMEM
  uint64_t* kv_done = p_full + 2;    // the tile's last dK/dV MMA retired
  uint64_t* kv_empty = kv_done + 1;  // the tile's last S/dP MMA has read K / V
  uint64_t* acc_empty = kv_empty + 1;  // 256 arrivals: dK / dV drained from TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Persistent: one CTA per SM walks (128-key tile, head, sequence) tiles heavy first (causal:
  // key tile kt carries n_kt - kt query blocks) in a snake order.  The Q/dO ring and the S/P
  // hand-offs run on across tiles (global unit counter g = 2 * blocks done + u), so the next
  // tile's K/V and first Q/dO units load, and its first S/dP MMAs run, while this tile's dK/dV
  // drain from TMEM.
  const int ntiles = n_kt * BH;
  const int G = static_cast<int>(gridDim.x), cta = static_cast<int>(blockIdx.x);
  const int nqb = seq / 128;
  struct Tile { int kt, h, b, i0, N; };
  auto tile_of = [&](int it, Tile& t) -> bool {
    const int idx = it * G + ((it & 1) ? (G - 1 - cta) : cta);
    if (idx >= ntiles) return false;
    t.kt = idx / BH;
    const int hb = idx % BH;
    t.h = hb % H;
    t.b = hb / H;
    t.i0 = causal ? t.kt : 0;
    t.N = nqb - t.i0;  // 128-query blocks; 2N half-block units
    return true;
  };

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&kv_map);
    ptx::tma_prefetch(&qkv_map);
    ptx::tma_prefetch(&do_map);
    ptx::mbar_init(kv_full, 1);
    for (int s = 0; s < NU; ++s) {
      ptx::mbar_init(&u_full[s], 1);
      ptx::mbar_init(&u_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&s_full[s], 1);
      ptx::mbar_init(&p_full[s], 128);
    }
    ptx::mbar_init(kv_done, 1);
    ptx::mbar_init(kv_empty, 1);
    ptx::mbar_init(acc_empty, 256);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  ptx::pdl_wait();
  ptx::pdl_trigger();
  // TMEM: S^T_a at 0, S^T_b at 64 (P^T_x bf16 pairs over their first 32 columns),
  // dP^T_a at 128, dP^T_b at 192 (dS^T_x likewise), dV at 256, dK at 256 + 64 NB
  const uint32_t t_dv = tmem + 256, t_dk = tmem + 256 + 64 * L::NB;

  if (warp == 0) {
    ptx::regs_dec<56>();
    if (lane == 0) {
      Tile t;
      for (int it = 0, g0 = 0; tile_of(it, t); g0 += 2 * t.N, ++it) {
        const int row0 = t.b * seq, h = t.h;
        ptx::mbar_wait(kv_empty, (it & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(kv_full, 2 * L::NB * T128);
        for (int c = 0; c < L::NB; ++c) {
          ptx::tma_load_2d(sm + L::K + c * T128, &kv_map, kv_full, H * D + h * D + 64 * c, row0 + t.kt * 128);
          ptx::tma_load_2d(sm + L::V + c * T128, &kv_map, kv_full, 2 * H * D + h * D + 64 * c, row0 + t.kt * 128);
        }
        for (int u = 0; u < 2 * t.N; ++u) {
          const int g = g0 + u, st = g % NU, q0 = t.i0 * 128 + u * 64;
          uint8_t* unit = sm + L::U + st * L::UNIT;
          ptx::mbar_wait(&u_empty[st], ((g / NU) & 1) ^ 1);
          BW_T(6, u);
#ifdef FA_ABL_NOLOAD  // ablation: keep the ring's first fill, skip every later load
          if (g >= NU) { ptx::mbar_arrive(&u_full[st]); continue; }
#endif
          ptx::mbar_arrive_expect_tx(&u_full[st], L::UNIT);
          for (int c = 0; c < L::NB; ++c) {
            ptx::tma_load_2d(unit + c * T64, &qkv_map, &u_full[st], h * D + 64 * c, row0 + q0);
            ptx::tma_load_2d(unit + (L::NB + c) * T64, &do_map, &u_full[st], h * D + 64 * c, row0 + q0);
          }
        }
      }
    }
  } else if (warp == 1) {
    ptx::regs_dec<56>();
    {  // warp-wide MMA issue (elect.sync inside the asm; see mma_bf16_*_w)
      constexpr uint32_t id_s = ptx::idesc_bf16_f32(128, 64, false, false);
      constexpr uint32_t id_g = ptx::idesc_bf16_f32(128, D, false, true);
      const uint64_t dk0 = ptx::umma_desc_sw128(ptx::smem_u32(sm + L::K), 16, 1024);
      const uint64_t dv0 = ptx::umma_desc_sw128(ptx::smem_u32(sm + L::V), 16, 1024);
      auto unit = [&](int g) { return ptx::smem_u32(sm + L::U + (g % NU) * L::UNIT); };
      // S^T_x, dP^T_x of global half-unit g (x = g & 1) into columns 64x / 128 + 64x
      auto issue_s = [&](int g) {
        const int x = g & 1;
        ptx::mbar_wait(&u_full[g % NU], (g / NU) & 1);
        BW_T(0, g);
        ptx::tc_fence_after();
        const uint64_t dq = ptx::umma_desc_sw128(unit(g), 16, 1024);
        const uint64_t ddo = dq + ((L::NB * T64) >> 4);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t oa = ((kk >> 2) * T128 + (kk & 3) * 32) >> 4, ob = ((kk >> 2) * T64 + (kk & 3) * 32) >> 4;
          ptx::mma_bf16_ss_w(tmem + 64 * x, dk0 + oa, dq + ob, id_s, kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t oa = ((kk >> 2) * T128 + (kk & 3) * 32) >> 4, ob = ((kk >> 2) * T64 + (kk & 3) * 32) >> 4;
          ptx::mma_bf16_ss_w(tmem + 128 + 64 * x, dv0 + oa, ddo + ob, id_s, kk > 0);
        }
        ptx::mma_commit_w(&s_full[x]);
        BW_T(1, g);
      };
      // dV += P^T_x dO_x, dK += dS^T_x Q_x (K = 64 queries; P^T / dS^T from TMEM); first = the
      // tile's first unit (overwrites the accumulators)
      auto issue_g = [&](int g, bool first) {
        const int x = g & 1;
        ptx::mbar_wait(&p_full[x], (g >> 1) & 1);
        BW_T(2, g);
        ptx::tc_fence_after();
        const uint64_t dq = ptx::umma_desc_sw128(unit(g), T64, 1024);
        const uint64_t ddo = dq + ((L::NB * T64) >> 4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          ptx::mma_bf16_ts_w(t_dv, tmem + 64 * x + kk * 8, ddo + ((kk * 2048) >> 4), id_g, (!first || kk > 0));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          ptx::mma_bf16_ts_w(t_dk, tmem + 128 + 64 * x + kk * 8, dq + ((kk * 2048) >> 4), id_g, (!first || kk > 0));
        ptx::mma_commit_w(&u_empty[g % NU]);
        BW_T(3, g);
      };
      // Per tile: S(0) S(1) | dVdK(u) S(u + 2) ... (S(u+2) reuses the columns dVdK(u) reads).
      // The next tile's S(0) S(1) are issued before this tile's dK/dV are drained; its first
      // dVdK waits for the drain (acc_empty).
      Tile t;
      for (int it = 0, g0 = 0; tile_of(it, t); g0 += 2 * t.N, ++it) {
        const int U = 2 * t.N;
        ptx::mbar_wait(kv_full, it & 1);
        issue_s(g0);
        if (U > 1) issue_s(g0 + 1);
        if (U <= 2) ptx::mma_commit_w(kv_empty);
        ptx::mbar_wait(acc_empty, (it & 1) ^ 1);
        for (int u = 0; u < U; ++u) {
          issue_g(g0 + u, u == 0);
          if (u + 2 < U) {
            issue_s(g0 + u + 2);
            if (u + 3 == U) ptx::mma_commit_w(kv_empty);
          }
        }
        ptx::mma_commit_w(kv_done);
      }
    }
  } else if (warp >= 4) {
    ptx::regs_inc<224>();
    const int x = (warp - 4) >> 2;  // half: queries [64 x, 64 x + 64) of every block
    const int q = warp & 3;
    const int r = q * 32 + lane;  // key row within the tile
    const uint32_t lanes = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t t_s = tmem + lanes + 64 * x, t_d = tmem + 128 + lanes + 64 * x;
    const float2 c2 = make_float2(scale_log2, scale_log2);
    Tile t;
    for (int it = 0, g0 = 0; tile_of(it, t); g0 += 2 * t.N, ++it) {
      const int key = t.kt * 128 + r;
      // a padding key (KPAD instances only: the unpadded kernel carries no mask code)
      const bool kpad = KPAD && key >= key_len[t.b];
      const float* lse_bh = lse + (static_cast<size_t>(t.b) * H + t.h) * seq;
      const float* del_bh = delta + (static_cast<size_t>(t.b) * H + t.h) * seq;
      // dS^T chunks of this tile (dQ GEMM operand, see DS_CHUNK): this thread's key in chunk
      // (block n, half x)
      uint8_t* ds_row = ds_ws == nullptr ? nullptr
                                         : ds_ws + ((static_cast<size_t>(t.b) * H + t.h) * ds_chunks_per_head(nqb, causal) +
                                                    ds_chunk_offset(nqb, t.kt, causal) + x) * DS_CHUNK +
                                               (r >> 6) * 8192 + (r & 63) * 16;
      for (int n = 0; n < t.N; ++n) {
        const int u = g0 + 2 * n + x;
        const int qbase = (t.i0 + n) * 128 + 64 * x;
        const bool diag = causal && n == 0;
        float4 lq4[16], dq4[16];  // this half's 64 lse / delta (same address across the warp)
#pragma unroll
        for (int c4 = 0; c4 < 16; ++c4) {
          lq4[c4] = __ldg(reinterpret_cast<const float4*>(lse_bh + qbase) + c4);
          dq4[c4] = __ldg(reinterpret_cast<const float4*>(del_bh + qbase) + c4);
        }
        ptx::mbar_wait(&s_full[x], (u >> 1) & 1);
        if (threadIdx.x == 128) BW_T(4, u);
        ptx::tc_fence_after();
        uint32_t s[64], d[64];
        ptx::tmem_ld_32x32b_x32(t_s, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
        ptx::tmem_ld_32x32b_x32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
        ptx::tmem_ld_32x32b_x32(t_d, *reinterpret_cast<uint32_t(*)[32]>(&d[0]));
        ptx::tmem_ld_32x32b_x32(t_d + 32, *reinterpret_cast<uint32_t(*)[32]>(&d[32]));
        ptx::tmem_ld_wait();
        uint32_t pp[32], dd[32];
#pragma unroll
        for (int c4 = 0; c4 < 16; ++c4) {
          const float4 lq = lq4[c4], dq = dq4[c4];
          const int cc = 4 * c4;
          float2 x0 = __ffma2_rn(make_float2(__uint_as_float(s[cc]), __uint_as_float(s[cc + 1])), c2,
                                 make_float2(-lq.x, -lq.y));
          float2 x1 = __ffma2_rn(make_float2(__uint_as_float(s[cc + 2]), __uint_as_float(s[cc + 3])), c2,
                                 make_float2(-lq.z, -lq.w));
#ifdef FA_ABL_NOSOFT
          float2 p0 = x0, p1 = x1;
#else
          float2 p0 = make_float2(ex2(x0.x), ex2(x0.y)), p1 = make_float2(ex2(x1.x), ex2(x1.y));
#endif
          if (diag) {  // query < key is masked
            if (qbase + cc < key) p0.x = 0.f;
            if (qbase + cc + 1 < key) p0.y = 0.f;
            if (qbase + cc + 2 < key) p1.x = 0.f;
            if (qbase + cc + 3 < key) p1.y = 0.f;
          }
          if (KPAD && kpad) p0 = p1 = make_float2(0.f, 0.f);
          const float2 g0 = __fmul2_rn(
              __fadd2_rn(make_float2(__uint_as_float(d[cc]), __uint_as_float(d[cc + 1])), make_float2(-dq.x, -dq.y)), p0);
          const float2 g1 = __fmul2_rn(
              __fadd2_rn(make_float2(__uint_as_float(d[cc + 2]), __uint_as_float(d[cc + 3])), make_float2(-dq.z, -dq.w)),
              p1);
          pp[2 * c4] = pack2(p0.x, p0.y);
          pp[2 * c4 + 1] = pack2(p1.x, p1.y);
          dd[2 * c4] = pack2(g0.x, g0.y);
          dd[2 * c4 + 1] = pack2(g1.x, g1.y);
        }
        if (threadIdx.x == 128) BW_T(5, u);
        // P^T_x / dS^T_x (bf16 pairs) over the first 32 columns of this half's S^T / dP^T
        tmem_st_x16(t_s, pp);
        tmem_st_x16(t_s + 16, pp + 16);
        tmem_st_x16(t_d, dd);
        tmem_st_x16(t_d + 16, dd + 16);
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&p_full[x]);
        // dS^T for the dQ GEMM, after the hand-off (the arrive's release would otherwise wait
        // for these global stores)
        if (ds_row != nullptr) {
          uint8_t* dst = ds_row + static_cast<size_t>(2 * n) * DS_CHUNK;
#pragma unroll
          for (int v = 0; v < 8; ++v)
            st_na_v4(dst + v * 1024, dd[4 * v], dd[4 * v + 1], dd[4 * v + 2], dd[4 * v + 3]);
        }
        if (threadIdx.x == 128) BW_T(7, u);
      }
      ptx::mbar_wait(kv_done, it & 1);
      ptx::tc_fence_after();
      // warpgroup 0 writes dK, warpgroup 1 writes dV
      const size_t ld = static_cast<size_t>(3) * H * D;
      bf16* dst = dqkv + (static_cast<size_t>(t.b) * seq + key) * ld + (x == 0 ? H * D : 2 * H * D) + t.h * D;
      tmem_row_to_global<D>((x == 0 ? t_dk : t_dv) + lanes, dst, x == 0 ? scale : 1.f);
      ptx::tc_fence_before();
      ptx::mbar_arrive(acc_empty);
    }
  } else {
    ptx::regs_dec<56>();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// ==================================================================== dQ
template <int D>
struct QSmem {
  static constexpr int NB = (D + 63) / 64;
  // K is held from S(j) until dQ(j) (one block later), V only until dP(j): separate rings.
  // Q lives in TMEM (S = Q K^T is a TS MMA), which frees the smem for a 4-deep K ring: K
  // loads start ~3 blocks ahead of use, covering the ~3k-cycle TMA latency under load.
  static constexpr int NSK = NB == 2 ? 4 : 8, NSV = NB == 2 ? 2 : 4;
  static constexpr uint32_t DO = 0;
  static constexpr uint32_t K = DO + NB * T128;   // NSK stages of NB x T128
  static constexpr uint32_t V = K + NSK * NB * T128;
  static constexpr uint32_t BAR = V + NSV * NB * T128;
  static constexpr uint32_t BYTES = BAR + 512;
};

// Persistent: one CTA per SM walks (128-query tile, head, sequence) tiles heavy-first in a
// snake order; the K/V ring, the S/dP/dS hand-off barriers and the dO buffer run on across
// tiles, so the next tile's loads land during this tile's last blocks and epilogue instead of
// behind a fresh CTA's prologue (the non-persistent version spent ~9k cycles before its
// first MMA: profiles/r01_attn_traces.md).
template <int D, bool KPAD>
__global__ void __launch_bounds__(384, 1)
    fa_bwd_dq_kernel(const __grid_constant__ CUtensorMap qkv_map, const __grid_constant__ CUtensorMap do_map,
                     const bf16* __restrict__ qkv, const float* __restrict__ lse, const float* __restrict__ delta,
                     bf16* __restrict__ dqkv, int seq, int H, int n_qt, int BH, float scale_log2, float scale,
                     int causal, int early, const int32_t* __restrict__ key_len) {
  using L = QSmem<D>;
  constexpr int NSK = L::NSK, NSV = L::NSV;
  extern __shared__ uint8_t smem_raw[];
  long long* const dbg_ = blockIdx.x == 0 ? g_bw_dbg : nullptr;  // trace hook, read once
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~static_cast<uintptr_t>(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* q_full = bar + 0;          // 256 arrivals: Q rows stored into TMEM
  uint64_t* do_full = bar + 1;
  uint64_t* k_full = bar + 2;          // [NSK]
  uint64_t* k_empty = k_full + 8;      // [NSK]
  uint64_t* v_full = k_empty + 8;      // [NSV]
  uint64_t* v_empty = v_full + 4;      // [NSV]
  uint64_t* s_full = v_empty + 4;
  uint64_t* s_empty = s_full + 1;      // 256 arrivals: S loaded into registers
  uint64_t* d_empty = s_empty + 1;     // 256 arrivals: dP loaded into registers
  uint64_t* p_full = d_empty + 1;      // 256 arrivals: dS written into TMEM
  uint64_t* ds_empty = p_full + 1;     // dQ MMA has read dS
  uint64_t* dq_done = ds_empty + 1;
  uint64_t* do_empty = dq_done + 1;    // the tile's last dP MMA has read dO
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(do_empty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = n_qt * BH;
  const int G = static_cast<int>(gridDim.x), cta = static_cast<int>(blockIdx.x);
  // tile it of this CTA: snake over the heavy-first list (query tile n_qt-1 of every head first)
  auto tile_of = [&](int it, int& qt, int& h, int& b) -> bool {
    const int idx = it * G + ((it & 1) ? (G - 1 - cta) : cta);
    if (idx >= ntiles) return false;
    qt = n_qt - 1 - idx / BH;
    const int hb = idx % BH;
    h = hb % H;
    b = hb / H;
    return true;
  };
  auto nblocks = [&](int qt) { return causal ? qt + 1 : seq / 128; };

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&qkv_map);
    ptx::tma_prefetch(&do_map);
    ptx::mbar_init(q_full, 256);
    ptx::mbar_init(do_full, 1);
    for (int s = 0; s < NSK; ++s) {
      ptx::mbar_init(&k_full[s], 1);
      ptx::mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < NSV; ++s) {
      ptx::mbar_init(&v_full[s], 1);
      ptx::mbar_init(&v_empty[s], 1);
    }
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(s_empty, 256);
    ptx::mbar_init(d_empty, 256);
    ptx::mbar_init(p_full, 256);
    ptx::mbar_init(ds_empty, 1);
    ptx::mbar_init(dq_done, 1);
    ptx::mbar_init(do_empty, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // PDL: this kernel's predecessor is the dK/dV kernel, which it does not read (dQ and dK/dV
  // are disjoint columns of dqkv); its inputs (qkv, dO, lse, delta) were complete when dK/dV
  // passed its own griddepcontrol.wait, which precedes the trigger that let this grid launch.
  // So dQ CTAs start on the SMs the dK/dV tail frees, and wait for dK/dV only before exiting
  // (the next kernel's wait on this grid then also covers dK/dV).
  if (!early) ptx::pdl_wait();
  ptx::pdl_trigger();
  // TMEM: S at 0, dP at 128, dQ at 256, dS (bf16 pairs, 64 columns) at 256 + 64 NB,
  // Q (bf16 pairs, D / 2 columns) at 320 + 64 NB
  const uint32_t t_dq = tmem + 256, t_ds = tmem + 256 + 64 * L::NB, t_q = tmem + 320 + 64 * L::NB;
  if (threadIdx.x == 0) BW_T(7, 0);

  if (warp == 0) {
    ptx::regs_dec<56>();
    if (lane == 0) {
      int g0 = 0;  // K/V blocks loaded by this CTA so far (ring position)
      int qt, h, b;
      for (int it = 0; tile_of(it, qt, h, b); ++it) {
        const int row0 = b * seq, N = nblocks(qt);
        ptx::mbar_wait(do_empty, (it & 1) ^ 1);  // previous tile's last dP MMA read dO
        ptx::mbar_arrive_expect_tx(do_full, L::NB * T128);
        for (int c = 0; c < L::NB; ++c)
          ptx::tma_load_2d(sm + L::DO + c * T128, &do_map, do_full, h * D + 64 * c, row0 + qt * 128);
        // K(j) ahead of V(j): S(j) is issued before dP(j)
        for (int n = 0; n < N; ++n) {
          const int g = g0 + n, sk = g % NSK, sv = g % NSV;
          ptx::mbar_wait(&k_empty[sk], ((g / NSK) & 1) ^ 1);
          if (it == 0) BW_T(6, n);
          ptx::mbar_arrive_expect_tx(&k_full[sk], L::NB * T128);
          for (int c = 0; c < L::NB; ++c)
            ptx::tma_load_2d(sm + L::K + (sk * L::NB + c) * T128, &qkv_map, &k_full[sk], H * D + h * D + 64 * c,
                             row0 + n * 128);
          ptx::mbar_wait(&v_empty[sv], ((g / NSV) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&v_full[sv], L::NB * T128);
          for (int c = 0; c < L::NB; ++c)
            ptx::tma_load_2d(sm + L::V + (sv * L::NB + c) * T128, &qkv_map, &v_full[sv],
                             2 * H * D + h * D + 64 * c, row0 + n * 128);
        }
        g0 += N;
      }
    }
  } else if (warp == 1) {
    ptx::regs_dec<56>();
    {  // warp-wide MMA issue (elect.sync inside the asm; see mma_bf16_*_w); descriptors built
       // once per stage and advanced by adding the 16-byte-unit offset to their address field
      constexpr uint32_t id_s = ptx::idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t id_g = ptx::idesc_bf16_f32(128, D, false, true);
      const uint64_t dsdo = ptx::umma_desc_sw128(ptx::smem_u32(sm + L::DO), 16, 1024);
      int g0 = 0;
      int qt, h, b;
      for (int it = 0; tile_of(it, qt, h, b); ++it) {
        const int N = nblocks(qt);
        ptx::mbar_wait(q_full, it & 1);   // this tile's Q in TMEM (written after the last dQ drain)
        ptx::mbar_wait(do_full, it & 1);
        for (int n = 0; n <= N; ++n) {
          if (n < N) {
            const int g = g0 + n, stk = g % NSK, stv = g % NSV;
            ptx::mbar_wait(&k_full[stk], (g / NSK) & 1);
            if (it == 0) BW_T(0, n);
            ptx::mbar_wait(s_empty, (g & 1) ^ 1);
            if (it == 0) BW_T(1, n);
            ptx::tc_fence_after();
            const uint64_t dk = ptx::umma_desc_sw128(ptx::smem_u32(sm + L::K + stk * L::NB * T128), 16, 1024);
            const uint64_t dv = ptx::umma_desc_sw128(ptx::smem_u32(sm + L::V + stv * L::NB * T128), 16, 1024);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
              ptx::mma_bf16_ts_w(tmem, t_q + kk * 8, dk + (((kk >> 2) * T128 + (kk & 3) * 32) >> 4), id_s, kk > 0);
            ptx::mbar_wait(&v_full[stv], (g / NSV) & 1);
            ptx::mbar_wait(d_empty, (g & 1) ^ 1);  // dP(g-1) loaded: S(g) above overlapped that load
            ptx::tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t o = ((kk >> 2) * T128 + (kk & 3) * 32) >> 4;
              ptx::mma_bf16_ss_w(tmem + 128, dsdo + o, dv + o, id_s, kk > 0);
            }
            ptx::mma_commit_w(s_full);
            ptx::mma_commit_w(&v_empty[stv]);
            if (n == N - 1) ptx::mma_commit_w(do_empty);  // last read of this tile's dO
            if (it == 0) BW_T(8, n);
          }
          if (n > 0) {
            const int m = n - 1, g = g0 + m, stk = g % NSK;
            ptx::mbar_wait(p_full, g & 1);
            if (it == 0) BW_T(2, m);
            ptx::tc_fence_after();
            const uint64_t dk = ptx::umma_desc_sw128(ptx::smem_u32(sm + L::K + stk * L::NB * T128), T128, 1024);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              ptx::mma_bf16_ts_w(t_dq, t_ds + kk * 8, dk + ((kk * 2048) >> 4), id_g, (m > 0 || kk > 0));
            ptx::mma_commit_w(ds_empty);
            ptx::mma_commit_w(&k_empty[stk]);
            if (it == 0) BW_T(9, m);
          }
        }
        ptx::mma_commit_w(dq_done);
        g0 += N;
      }
    }
  } else if (warp >= 4) {
    ptx::regs_inc<224>();
    const int wg = (warp - 4) >> 2;  // keys [64 wg, 64 wg + 64) of every block
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t lanes = static_cast<uint32_t>(q * 32) << 16;
    const int c0 = 64 * wg;
    constexpr int MAIN = 32 * (D / 64);  // dims per warpgroup in the 64-multiple part
    int g0 = 0;
    int qt, h, b;
    for (int it = 0; tile_of(it, qt, h, b); ++it) {
      const int row0 = b * seq, N = nblocks(qt);
      const int qrow = qt * 128 + r;
      const size_t bh = (static_cast<size_t>(b) * H + h) * seq;
      const float nl = -lse[bh + qrow], dl = delta[bh + qrow];
      {  // this thread's half of its Q row -> TMEM (bf16 pairs: column j holds dims 2j, 2j+1).
         // Warpgroup wg owns dims [32 (D/64) wg, +32 (D/64)) and, for head_dim 80, the tail dims
         // [64 + 8 wg, +8): every TMEM access stays aligned to its own width.  Written after the
         // previous tile's dQ was drained, i.e. after all its MMAs (dq_done).
        const bf16* qrow_p = qkv + (static_cast<size_t>(row0) + qrow) * (3 * H * D) + h * D;
        const uint4* src = reinterpret_cast<const uint4*>(qrow_p + wg * MAIN);
        uint32_t qv[MAIN / 2];
#pragma unroll
        for (int u = 0; u < MAIN / 8; ++u) {
          const uint4 t = src[u];
          qv[4 * u] = t.x;
          qv[4 * u + 1] = t.y;
          qv[4 * u + 2] = t.z;
          qv[4 * u + 3] = t.w;
        }
#pragma unroll
        for (int u = 0; u < MAIN / 32; ++u) tmem_st_x16(t_q + lanes + wg * (MAIN / 2) + 16 * u, qv + 16 * u);
        if constexpr (D % 64 == 16) {
          const uint4 t = *reinterpret_cast<const uint4*>(qrow_p + 2 * MAIN + 8 * wg);
          const uint32_t tv[4] = {t.x, t.y, t.z, t.w};
          ptx::tmem_st_32x32b_x4(t_q + lanes + MAIN + 4 * wg, tv);
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(q_full);
      }
      const int klen = KPAD ? key_len[b] : seq;  // key padding (bidirectional models)
      for (int n = 0; n < N; ++n) {
        const int g = g0 + n;
        const bool diag = causal && n == N - 1;
        const bool lim = KPAD && (n + 1) * 128 > klen;
        ptx::mbar_wait(s_full, g & 1);
        if (it == 0 && lane == 0 && q == 0 && wg == 0) BW_T(3, n);
        ptx::tc_fence_after();
        uint32_t s[64], d[64];
        // S first, released as soon as it is in registers so S(n+1) overlaps the dP load
        ptx::tmem_ld_32x32b_x32(tmem + lanes + c0, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
        ptx::tmem_ld_32x32b_x32(tmem + lanes + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(s_empty);
        ptx::tmem_ld_32x32b_x32(tmem + 128 + lanes + c0, *reinterpret_cast<uint32_t(*)[32]>(&d[0]));
        ptx::tmem_ld_32x32b_x32(tmem + 128 + lanes + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&d[32]));
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(d_empty);
        uint32_t gg[32];
#pragma unroll
        for (int cc = 0; cc < 64; cc += 2) {
          // packed pairs; FA_BWD_POLY_PAIRS of every 4 exponent pairs on the FMA pipe
#ifdef FA_DQ_SCALAR
          float g0f = ex2(fmaf(__uint_as_float(s[cc]), scale_log2, nl)) * (__uint_as_float(d[cc]) - dl);
          float g1f = ex2(fmaf(__uint_as_float(s[cc + 1]), scale_log2, nl)) * (__uint_as_float(d[cc + 1]) - dl);
#else
          const float2 x = __ffma2_rn(make_float2(__uint_as_float(s[cc]), __uint_as_float(s[cc + 1])),
                                      make_float2(scale_log2, scale_log2), make_float2(nl, nl));
          const float2 p = ((cc >> 1) & 3) < FA_BWD_POLY_PAIRS ? ex2_fma2(x) : make_float2(ex2(x.x), ex2(x.y));
          const float2 gv = __fmul2_rn(p, __fadd2_rn(make_float2(__uint_as_float(d[cc]), __uint_as_float(d[cc + 1])),
                                                     make_float2(-dl, -dl)));
          float g0f = gv.x, g1f = gv.y;
#endif
          if (diag) {
            const int k0 = n * 128 + c0 + cc;
            if (k0 > qrow) g0f = 0.f;
            if (k0 + 1 > qrow) g1f = 0.f;
          } else if (lim) {
            const int k0 = n * 128 + c0 + cc;
            if (k0 >= klen) g0f = 0.f;
            if (k0 + 1 >= klen) g1f = 0.f;
          }
          gg[cc >> 1] = pack2(g0f, g1f);
        }
        if (it == 0 && lane == 0 && q == 0 && wg == 0) BW_T(4, n);
        ptx::mbar_wait(ds_empty, (g & 1) ^ 1);  // dQ(g-1) has read the previous dS
        ptx::tc_fence_after();
        tmem_st_x16(t_ds + lanes + 32 * wg, gg);
        tmem_st_x16(t_ds + lanes + 32 * wg + 16, gg + 16);
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(p_full);
        if (it == 0 && lane == 0 && q == 0 && wg == 0) BW_T(5, n);
      }
      ptx::mbar_wait(dq_done, it & 1);
      ptx::tc_fence_after();
      // each warpgroup writes half of the D columns (head_dim 80: 32 + 8 each, aligned as above)
      bf16* rowq = dqkv + (static_cast<size_t>(row0) + qrow) * (static_cast<size_t>(3) * H * D) + h * D;
      tmem_row_to_global<MAIN>(t_dq + lanes + wg * MAIN, rowq + wg * MAIN, scale);
      if constexpr (D % 64 == 16)
        tmem_row_to_global<8>(t_dq + lanes + 2 * MAIN + 8 * wg, rowq + 2 * MAIN + 8 * wg, scale);
      ptx::tc_fence_before();
      g0 += N;
    }
  } else {
    ptx::regs_dec<56>();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
  if (early) ptx::pdl_wait();  // the dK/dV grid has completed before this one does
}

// ==================================================================== dQ GEMM
// dQ = scale * dS K per (128-query tile, head, sequence), from the dS^T chunks the dK/dV kernel
// stored (DS_CHUNK): no second pass over S, dP and the softmax.  A plain K-loop over the
// tile's keys, 64 per step:  A = dS [128 queries][64 keys] (MN-major, no swizzle: the matching
// 8 KB key halves of the block's two chunks, one bulk copy each), B = K [64 keys][D]
// (MN-major, D/64 TMA boxes), fp32 accumulator [128 queries][D] in TMEM.  dS streams from HBM
// once and K re-reads hit L2, so they have separate rings: a deep one for dS (bytes in flight
// against DRAM latency) and a two-deep one for K, each with its own loading thread (warp 0 /
// warp 2 lane 0); one warp issues the MMAs and four drain TMEM.  Deterministic: every dQ
// element sums its keys in one accumulator in a fixed order.
template <int D, int NA_, int NB_>
struct DqgSmem {
  static constexpr int NB = (D + 63) / 64;
  static constexpr int NA = NA_, NK = NB_;  // dS / K ring depths
  static constexpr uint32_t ASZ = 2 * T64, BSZ = NB * T64;
  static constexpr uint32_t B0 = 0;                 // K ring first: SW128 boxes need 1024-B alignment
  static constexpr uint32_t A0 = NK * BSZ;
  static constexpr uint32_t BAR = A0 + NA * ASZ;
  static constexpr uint32_t BYTES = BAR + 128;
};

template <int D, int NA_, int NB_>
__global__ void __launch_bounds__(192, 1)
    fa_bwd_dq_gemm_kernel(const __grid_constant__ CUtensorMap k64_map, const __grid_constant__ CUtensorMap dq_map,
                          const uint8_t* __restrict__ ds_ws, bf16* __restrict__ dqkv, int seq, int H, int n_qt, int BH,
                          float scale, int causal) {
  using L = DqgSmem<D, NA_, NB_>;
  static_assert(D % 64 == 0, "the TMA-store epilogue writes 64-column boxes");
  static_assert(NA_ * 2 * T64 >= 4 * (D / 64) * 4096, "dQ staging reuses the dS ring");
  constexpr int NA = L::NA, NK = L::NK;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~static_cast<uintptr_t>(1023));
  uint64_t* a_full = reinterpret_cast<uint64_t*>(sm + L::BAR);  // [NA]
  uint64_t* a_empty = a_full + NA;                                // [NA]
  uint64_t* b_full = a_empty + NA;                                // [NK]
  uint64_t* b_empty = b_full + NK;                                // [NK]
  uint64_t* acc_full = b_empty + NK;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int idx = static_cast<int>(blockIdx.x);
  const int qt = causal ? n_qt - 1 - idx / BH : idx / BH;  // causal: heavy tiles first
  const int hb = idx % BH, h = hb % H, b = hb / H;
  const int steps = 2 * (causal ? qt + 1 : n_qt);  // 64-key steps
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&k64_map);
    for (int s = 0; s < NA; ++s) {
      ptx::mbar_init(&a_full[s], 1);
      ptx::mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < NK; ++s) {
      ptx::mbar_init(&b_full[s], 1);
      ptx::mbar_init(&b_empty[s], 1);
    }
    ptx::mbar_init(acc_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<128>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  ptx::pdl_wait();  // dS^T comes from the dK/dV grid
  ptx::pdl_trigger();
  if (warp == 0) {
    if (lane == 0) {  // dS ring
      const uint8_t* ds_head = ds_ws + static_cast<size_t>(hb) * ds_chunks_per_head(n_qt, causal) * DS_CHUNK;
      for (int j = 0; j < steps; ++j) {
        const int s = j % NA, kt = j >> 1, hk = j & 1;
        uint8_t* st = sm + L::A0 + s * L::ASZ;
        ptx::mbar_wait(&a_empty[s], ((j / NA) & 1) ^ 1);
#ifdef FA_DQG_NODS  // ablation: no dS^T loads
        ptx::mbar_arrive(&a_full[s]);
        continue;
#endif
        ptx::mbar_arrive_expect_tx(&a_full[s], L::ASZ);
        const uint8_t* c0 = ds_head +
                            static_cast<size_t>(ds_chunk_offset(n_qt, kt, causal) + 2 * (qt - (causal ? kt : 0))) * DS_CHUNK +
                            hk * T64;
        ptx::bulk_load(st, c0, T64, &a_full[s]);                  // queries [0, 64), keys 64 hk + [0, 64)
        ptx::bulk_load(st + T64, c0 + DS_CHUNK, T64, &a_full[s]);  // queries [64, 128)
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, D, true, true);  // A, B MN-major
    for (int j = 0; j < steps; ++j) {
      const int sa = j % NA, sb = j % NK;
      ptx::mbar_wait(&a_full[sa], (j / NA) & 1);
      ptx::mbar_wait(&b_full[sb], (j / NK) & 1);
      ptx::tc_fence_after();
      // A: core matrices of 8 keys x 8 queries, 128 B apart along keys, 1024 B along queries
      const uint64_t ad = ptx::umma_desc_noswz(ptx::smem_u32(sm + L::A0 + sa * L::ASZ), 128, 1024);
      const uint64_t bd = ptx::umma_desc_sw128(ptx::smem_u32(sm + L::B0 + sb * L::BSZ), T64, 1024);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)  // 16 keys per MMA: A +256 B, B +2048 B (16 SW128 rows)
        ptx::mma_bf16_ss_w(tmem, ad + kk * 16, bd + kk * 128, id, (j > 0 || kk > 0) ? 1u : 0u);
      ptx::mma_commit_w(&a_empty[sa]);
      ptx::mma_commit_w(&b_empty[sb]);
    }
    ptx::mma_commit_w(acc_full);
  } else {
    if (warp == 2 && lane == 0) {  // K ring (L2-resident re-reads)
      for (int j = 0; j < steps; ++j) {
        const int s = j % NK, kt = j >> 1, hk = j & 1;
        uint8_t* st = sm + L::B0 + s * L::BSZ;
        ptx::mbar_wait(&b_empty[s], ((j / NK) & 1) ^ 1);
#ifdef FA_DQG_NOK  // ablation: no K loads
        ptx::mbar_arrive(&b_full[s]);
        continue;
#endif
        ptx::mbar_arrive_expect_tx(&b_full[s], L::BSZ);
        for (int c = 0; c < L::NB; ++c)
          ptx::tma_load_2d(st + c * T64, &k64_map, &b_full[s], H * D + h * D + 64 * c, b * seq + kt * 128 + hk * 64);
      }
    }
    __syncwarp();
    const int q = warp & 3;  // TMEM lane quarter of this warp (warps 2..5 -> 2, 3, 0, 1)
    ptx::mbar_wait(acc_full, 0);
    ptx::tc_fence_after();
    // Epilogue: bf16(scale * dQ) rows -> this warp's SW128 staging blocks (the dS ring is free
    // once every MMA retired: 32 rows x 64 columns, 16-byte unit v of row r at v ^ (r & 7),
    // conflict-free) -> one TMA store per 64-column block (the per-row 16-byte stores this
    // replaces were a quarter of the kernel: 70 -> 53 us without them at the 1.3B shape)
    uint8_t* stg = sm + L::A0 + q * (D / 64) * 4096;
#pragma unroll
    for (int c = 0; c < D / 64; ++c) {
      uint32_t lo[32], hi[32];
      const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) + 64 * c;
      ptx::tmem_ld_32x32b_x32(ta, lo);
      ptx::tmem_ld_32x32b_x32(ta + 32, hi);
      ptx::tmem_ld_wait();
      uint8_t* rowp = stg + c * 4096 + lane * 128;
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const uint32_t* src = v < 4 ? lo + 8 * v : hi + 8 * (v - 4);
        uint4 pk;
        pk.x = pack2(__uint_as_float(src[0]) * scale, __uint_as_float(src[1]) * scale);
        pk.y = pack2(__uint_as_float(src[2]) * scale, __uint_as_float(src[3]) * scale);
        pk.z = pack2(__uint_as_float(src[4]) * scale, __uint_as_float(src[5]) * scale);
        pk.w = pack2(__uint_as_float(src[6]) * scale, __uint_as_float(src[7]) * scale);
        *reinterpret_cast<uint4*>(rowp + ((v ^ (lane & 7)) << 4)) = pk;
      }
    }
    ptx::fence_proxy_async_smem();
    __syncwarp();
#ifndef FA_DQG_NOEPI  // ablation: no dQ stores
    if (lane == 0) {
      for (int c = 0; c < D / 64; ++c)
        ptx::tma_store_2d(&dq_map, stg + c * 4096, h * D + 64 * c, b * seq + qt * 128 + q * 32);
      ptx::bulk_commit();
      ptx::bulk_wait<0>();  // stores complete before the CTA exits (as the GEMM epilogue does)
    }
#endif
    ptx::tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<128>(tmem);
  }
}

template <class K>
int set_smem(K k, size_t bytes) {
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}

template <int D>
int launch_bwd_tc(const bf16* qkv, const bf16* dout, const float* lse, const float* delta, bf16* dqkv, int B,
                  int S, int H, int causal, const int32_t* key_len, uint8_t* ds_ws, cudaStream_t st) {
  CUtensorMap q128, o128, q64, o64;
  const uint64_t ldq = static_cast<uint64_t>(3) * H * D, ldo = static_cast<uint64_t>(H) * D;
  const uint64_t rows = static_cast<uint64_t>(B) * S;
  if (!tma_map_bf16_2d(&q128, qkv, ldq, rows, ldq, 64, 128) || !tma_map_bf16_2d(&o128, dout, ldo, rows, ldo, 64, 128) ||
      !tma_map_bf16_2d(&q64, qkv, ldq, rows, ldq, 64, 64) || !tma_map_bf16_2d(&o64, dout, ldo, rows, ldo, 64, 64))
    return AMDP_ERR_TMA;
  const float scale = 1.f / sqrtf(static_cast<float>(D));
  const float scale_log2 = 1.4426950408889634f * scale;
  static std::atomic<uint64_t> attr{0};
  // dQ GEMM dS ring depth (AMDP_ATTN_DQ_STAGES; the K ring is two deep).  Measured best: two
  // (head_dim 128, 64 KB: three CTAs per SM) / three (head_dim 64, 64 KB); deeper rings with
  // fewer CTAs per SM were slower (profiles/r02/dq_gemm).  head_dim 80 has no dQ GEMM.
  constexpr int DG = D % 64 == 0 ? D : 64;
  static const int dq_stages = getenv("AMDP_ATTN_DQ_STAGES") ? atoi(getenv("AMDP_ATTN_DQ_STAGES")) : (D > 64 ? 2 : 3);
  auto dq_gemm = dq_stages == 2 ? fa_bwd_dq_gemm_kernel<DG, 2, 2> : dq_stages == 3 ? fa_bwd_dq_gemm_kernel<DG, 3, 2>
               : dq_stages == 4 ? fa_bwd_dq_gemm_kernel<DG, 4, 2> : fa_bwd_dq_gemm_kernel<DG, 5, 2>;
  const size_t smem_g = 1024 + (dq_stages == 2 ? DqgSmem<DG, 2, 2>::BYTES : dq_stages == 3 ? DqgSmem<DG, 3, 2>::BYTES
                                : dq_stages == 4 ? DqgSmem<DG, 4, 2>::BYTES : DqgSmem<DG, 5, 2>::BYTES);
  if (D != DG) ds_ws = nullptr;
  const size_t smem_kv = KvSmem<D>::BYTES + 1024, smem_q = QSmem<D>::BYTES + 1024;
  if (first_on_device(attr)) {
    int e = set_smem(fa_bwd_dkdv_kernel<D, false>, smem_kv);
    if (!e) e = set_smem(fa_bwd_dkdv_kernel<D, true>, smem_kv);
    if (!e) e = set_smem(fa_bwd_dq_kernel<D, false>, smem_q);
    if (!e) e = set_smem(fa_bwd_dq_kernel<D, true>, smem_q);
    if (!e && D == DG) e = set_smem(dq_gemm, smem_g);
    if (e) {
      attr.store(0);
      return e;
    }
  }
  const int nt = S / 128;
  const int kv_grid = std::min(nt * H * B, num_sms());  // persistent
  cudaError_t e = launch_pdl(key_len ? fa_bwd_dkdv_kernel<D, true> : fa_bwd_dkdv_kernel<D, false>, dim3(kv_grid),
                             dim3(384), smem_kv, st, q128, q64, o64, lse, delta, dqkv, S, H, nt, H * B, scale_log2,
                             scale, causal, key_len, ds_ws);
  if (e != cudaSuccess) return e;
  if (ds_ws != nullptr) {  // dQ = dS K from the stored dS^T
    CUtensorMap dq_out;  // dq columns of dqkv, 64 x 32 boxes (the epilogue's TMA stores)
    if (!tma_map_bf16_2d(&dq_out, dqkv, ldq, rows, ldq, 64, 32)) return AMDP_ERR_TMA;
    e = launch_pdl(dq_gemm, dim3(nt * H * B), dim3(192), smem_g, st, q64, dq_out, ds_ws, dqkv, S, H, nt,
                   H * B, scale, causal);
    return e != cudaSuccess ? e : cudaGetLastError();
  }
  const int dq_grid = std::min(nt * H * B, num_sms());  // persistent
  static const int early = getenv("AMDP_ATTN_DQ_EARLY") ? atoi(getenv("AMDP_ATTN_DQ_EARLY")) : 1;
  e = launch_pdl(key_len ? fa_bwd_dq_kernel<D, true> : fa_bwd_dq_kernel<D, false>, dim3(dq_grid), dim3(384), smem_q,
                 st, q128, o128, qkv, lse, delta, dqkv, S, H, nt, H * B, scale_log2, scale, causal, early, key_len);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

// Used by amdp_attention_bwd (after the delta pre-pass) when the tensor-core path applies.
// ds_ws: dS^T scratch of attention_bwd_ds_bytes(); nullptr selects the dQ kernel that
// recomputes S / dP (AMDP_ATTN_DQ=recompute; A/B only).
int attention_bwd_tc(const bf16* qkv, const bf16* dout, const float* lse, const float* delta, bf16* dqkv, int B,
                     int S, int H, int D, int causal, const int32_t* key_len, uint8_t* ds_ws, cudaStream_t st) {
  if (S % 128 != 0) return AMDP_ERR_UNSUPPORTED;
  static const bool recompute = getenv("AMDP_ATTN_DQ") && strcmp(getenv("AMDP_ATTN_DQ"), "recompute") == 0;
  if (recompute || D == 80) ds_ws = nullptr;  // head_dim 80: storing dS^T costs the dK/dV kernel more than it saves
  if (D == 128) return launch_bwd_tc<128>(qkv, dout, lse, delta, dqkv, B, S, H, causal, key_len, ds_ws, st);
  if (D == 64) return launch_bwd_tc<64>(qkv, dout, lse, delta, dqkv, B, S, H, causal, key_len, ds_ws, st);
  if (D == 80) return launch_bwd_tc<80>(qkv, dout, lse, delta, dqkv, B, S, H, causal, key_len, ds_ws, st);
  return AMDP_ERR_UNSUPPORTED;
}

size_t attention_bwd_ds_bytes(int B, int S, int H, int causal) {
  return static_cast<size_t>(B) * H * ds_chunks_per_head(S / 128, causal) * DS_CHUNK;
}

}  // namespace amdp

extern "C" int amdp_debug_attention_bwd_trace(long long* device_buf) {
  return cudaMemcpyToSymbol(amdp::g_bw_dbg, &device_buf, sizeof(device_buf));
}
