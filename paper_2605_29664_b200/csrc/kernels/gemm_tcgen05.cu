// Stage GEMM for the AMDP executor: C = epi(alpha * A * B^T), bf16 in, fp32 accumulate.
//
// sm_100a design (no mma.sync / wgmma), two kernels with the same warp roles:
//   * gemm_bf16_tc_pair: a CTA pair (cta_group::2) per 256x256 tile, 6-stage TMA ring; every
//     stage GEMM with M >= 256 (the last partial wave of K-major-B GEMMs is split along N);
//     gemm_bf16_tcgen05: one CTA per 128x256 tile, 4-stage ring, for M < 256;
//   * persistent CTAs (grid = co-resident CTAs / pairs), launched with programmatic
//     dependent launch so the prologue overlaps the previous kernel's tail;
//   * warp 0: TMA producer, warp 1: tcgen05.mma issue, both warp-converged with elect.sync in
//     the asm (a single-lane branch made the compiler wrap every UTMALDG / UTCHMMA in a
//     serialisation loop, which starved the MN-major pair main loop) and descriptors advanced
//     by offset; two TMEM
//     accumulators so a tile's epilogue overlaps the next tile's main loop;
//   * warps 4..7: epilogue, each owning 32 TMEM lanes: tcgen05.ld -> fused op in registers
//     -> swizzled smem staging -> TMA store (or TMA reduce-add for the fp32 window gradient).
// Operands may be K-major or MN-major independently, so forward (X W^T), activation-gradient
// (dY W, via transposed weight copies) and weight-gradient (dY^T X) run without transposes
// of the activations.  Epilogues: plain bf16 store, GELU (stores pre-activation too),
// residual add, fp32 accumulate (weight-gradient accumulation across the minibatches of one
// AMDP window), GELU-backward, fp32 store.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>

#include "amdp_kernels.h"
#include "common.cuh"
#include "sm100_ptx.cuh"

namespace amdp {
namespace {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;
constexpr int A_STAGE_BYTES = BM * BK * 2;  // 16 KiB
constexpr int NUM_THREADS = 256;
constexpr int GROUP_M = 8;
constexpr int STG_BYTES = 4 * 2 * 4096;  // TMA-store epilogue staging (4 warps x 2 x 4 KB)

// Single-CTA tile 128 x TBN: TBN = 256 (4-stage ring, 2 x 256 TMEM columns) or TBN = 128
// (6-stage ring, 2 x 128 columns) for small products whose 128 x 256 tiles leave SMs idle.
template <int TBN>
struct SingleCfg {
  static constexpr int B_STAGE_BYTES = TBN * BK * 2;
  static constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
  static constexpr int STAGES = TBN == 256 ? 4 : 6;
  static constexpr uint32_t TMEM_COLS = 2 * TBN;
  static constexpr size_t SMEM = 1024 /*align slack*/ + STAGES * STAGE_BYTES + STG_BYTES + 256 /*barriers*/;
};

struct EpiParams {
  int M, N, K;
  void* C;
  int ldc;
  const __nv_bfloat16* aux;
  int ld_aux;
  __nv_bfloat16* C2;
  int ldc2;
  float alpha;
  float* rowdot;  // AMDP_EPI_ROWDOT: [M / seq][N / seg][seq] fp32
  int seg, seq;
};

// tanh on the SFU (tanh.approx.f32, max rel. error ~2^-11): the GELU epilogues run once per
// output element of the largest GEMMs, and their results are rounded to bf16 (2^-8).
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_tanh_grad(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float t = tanh_fast(k0 * (x + k1 * x * x * x));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x * x);
}

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int& tm, int& tn, int group_m = GROUP_M) {
  const int GROUP_M = group_m;
  const int in_group = GROUP_M * tiles_n;
  const int g = t / in_group;
  const int first_m = g * GROUP_M;
  const int gsz = min(tiles_m - first_m, GROUP_M);
  const int r = t % in_group;
  tm = first_m + r % gsz;
  tn = r / gsz;
}

constexpr int EPI_DISCARD = 99; // experiment only: drain TMEM, store nothing (AMDP_GEMM_DISCARD)

// Output tensor maps of the pair kernel's TMA epilogue: C (bf16 box {64, 32} or f32 box
// {32, 32}), C2 (GELU pre-activation), aux (residual / pre-activation input), SWIZZLE_128B.
struct EpiMaps {
  CUtensorMap c, c2, aux;
};

__device__ __forceinline__ uint32_t sw_chunk(int lane, int j) {
  return static_cast<uint32_t>(lane) * 128u + ((static_cast<uint32_t>(j) ^ (static_cast<uint32_t>(lane) & 7u)) << 4);
}

// One epilogue warp drains its 32 TMEM lanes (rows row0..row0+31) x `width` columns:
// tcgen05.ld -> fused op in registers -> swizzled row into a 4 KB staging buffer (conflict
// free: 8 consecutive lanes hit 8 distinct 16-byte bank groups) -> one TMA store (or
// reduce-add for the fp32 window gradient) per 32 x 64 bf16 / 32 x 32 fp32 block.  Two
// staging buffers per warp alternate, so a block's store overlaps the next block's math.
// Residual / GELU' inputs arrive by TMA into the same buffer before the math.
template <int EPI>
__device__ __forceinline__ void pair_epilogue(const EpiMaps& em, const EpiParams& p, uint32_t t_row, int width,
                                              int n0, int row0, uint8_t* stg, uint64_t* aux_bar,
                                              uint32_t& aux_phase, int& bsel, int lane) {
  // aux_bar[b] / bit b of aux_phase: the residual / pre-activation block landing in staging
  // buffer b.  Block c+1's load is issued before block c's math (one block of prefetch).
  constexpr bool F32 = (EPI == AMDP_EPI_ACCUM_F32 || EPI == AMDP_EPI_STORE_F32);
  constexpr bool ROWDOT = EPI == AMDP_EPI_ROWDOT;
  constexpr bool AUX = (EPI == AMDP_EPI_RESIDUAL || EPI == AMDP_EPI_GELU_BWD || ROWDOT);
  if constexpr (F32) {
#pragma unroll 1
    for (int cc = 0; cc < width; cc += 32) {
      if (n0 + cc >= p.N) break;
      uint32_t raw[32];
      ptx::tmem_ld_32x32b_x32(t_row + cc, raw);
      uint8_t* buf = stg + bsel * 4096;
      if (lane == 0) ptx::bulk_wait_read<1>();
      __syncwarp();
      ptx::tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float4 o = make_float4(__uint_as_float(raw[4 * j]) * p.alpha, __uint_as_float(raw[4 * j + 1]) * p.alpha,
                               __uint_as_float(raw[4 * j + 2]) * p.alpha, __uint_as_float(raw[4 * j + 3]) * p.alpha);
        *reinterpret_cast<float4*>(buf + sw_chunk(lane, j)) = o;
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if constexpr (EPI == AMDP_EPI_ACCUM_F32) ptx::tma_reduce_add_2d(&em.c, buf, n0 + cc, row0);
        else ptx::tma_store_2d(&em.c, buf, n0 + cc, row0);
        ptx::bulk_commit();
      }
      bsel ^= 1;
    }
  } else {
    const int n_end = min(width, p.N - n0);
    float dot = 0.f;  // ROWDOT: this row's partial sum over the current segment
    if constexpr (AUX) {  // block 0's residual / pre-activation / dot operand
      if (lane == 0) {
        ptx::bulk_wait_read<1>();
        ptx::mbar_arrive_expect_tx(&aux_bar[bsel], 4096);
        ptx::tma_load_2d(stg + bsel * 4096, &em.aux, &aux_bar[bsel], n0, row0);
      }
    }
#pragma unroll 1
    for (int cc = 0; cc < n_end; cc += 64) {
      uint32_t raw[64];
      ptx::tmem_ld_32x32b_x32(t_row + cc, *reinterpret_cast<uint32_t(*)[32]>(&raw[0]));
      ptx::tmem_ld_32x32b_x32(t_row + cc + 32, *reinterpret_cast<uint32_t(*)[32]>(&raw[32]));
      uint8_t* buf = stg + bsel * 4096;
      float v[64];
      if constexpr (AUX) {
        if (lane == 0 && cc + 64 < n_end) {  // prefetch block c+1 into the other buffer
          const int nb = bsel ^ 1;
          ptx::bulk_wait_read<0>();  // block c-1's store has finished reading it
          ptx::mbar_arrive_expect_tx(&aux_bar[nb], 4096);
          ptx::tma_load_2d(stg + nb * 4096, &em.aux, &aux_bar[nb], n0 + cc + 64, row0);
        }
        ptx::mbar_wait(&aux_bar[bsel], (aux_phase >> bsel) & 1u);
        aux_phase ^= 1u << bsel;
      } else {
        if (lane == 0) ptx::bulk_wait_read<1>();
        __syncwarp();
      }
      ptx::tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 64; ++j) v[j] = __uint_as_float(raw[j]) * p.alpha;
      if constexpr (AUX && !ROWDOT) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint4 q = *reinterpret_cast<const uint4*>(buf + sw_chunk(lane, j));
          const __nv_bfloat162* hq = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(hq[e]);
            if constexpr (EPI == AMDP_EPI_RESIDUAL) {
              v[8 * j + 2 * e] += f.x;
              v[8 * j + 2 * e + 1] += f.y;
            } else {
              v[8 * j + 2 * e] *= gelu_tanh_grad(f.x);
              v[8 * j + 2 * e + 1] *= gelu_tanh_grad(f.y);
            }
          }
        }
      }
      if constexpr (EPI == AMDP_EPI_GELU) {  // pre-activation to C2 first
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint4 q;
          __nv_bfloat162* hq = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
          for (int e = 0; e < 4; ++e) hq[e] = __floats2bfloat162_rn(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]);
          *reinterpret_cast<uint4*>(buf + sw_chunk(lane, j)) = q;
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          ptx::tma_store_2d(&em.c2, buf, n0 + cc, row0);
          ptx::bulk_commit();
        }
        bsel ^= 1;
        buf = stg + bsel * 4096;
        if (lane == 0) ptx::bulk_wait_read<1>();
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 64; ++j) v[j] = gelu_tanh_bf16in(v[j]);  // of the stored u
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        uint4 q;
        __nv_bfloat162* hq = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
        for (int e = 0; e < 4; ++e) hq[e] = __floats2bfloat162_rn(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]);
        if constexpr (ROWDOT) {  // dot of the stored (bf16) values with the aux chunk in place
          const uint4 a = *reinterpret_cast<const uint4*>(buf + sw_chunk(lane, j));
          const __nv_bfloat162* ha = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 x = __bfloat1622float2(hq[e]), y = __bfloat1622float2(ha[e]);
            dot = fmaf(x.x, y.x, dot);
            dot = fmaf(x.y, y.y, dot);
          }
        }
        *reinterpret_cast<uint4*>(buf + sw_chunk(lane, j)) = q;
      }
      if constexpr (ROWDOT) {
        const int col_end = n0 + cc + 64;  // segments end on 64-column block boundaries
        if (col_end % p.seg == 0 || cc + 64 >= n_end) {
          const int row = row0 + lane;
          const int seg_lo = ((col_end - 1) / p.seg) * p.seg;
          if (row < p.M) {
            float* dst = p.rowdot + (static_cast<size_t>(row / p.seq) * (p.N / p.seg) + seg_lo / p.seg) * p.seq +
                         row % p.seq;
            // a segment split across two tiles (64-wide tail sub-tiles): two partial sums
            // added to zero, exact in either order
            if (seg_lo >= n0 && seg_lo + p.seg <= n0 + n_end) *dst = dot;
            else atomicAdd(dst, dot);
          }
          dot = 0.f;
        }
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        ptx::tma_store_2d(&em.c, buf, n0 + cc, row0);
        ptx::bulk_commit();
      }
      bsel ^= 1;
    }
  }
}

template <bool A_MN, bool B_MN, int EPI, int TBN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap map_a,
                      const __grid_constant__ CUtensorMap map_b, const __grid_constant__ EpiMaps em,
                      const EpiParams p) {
  using Cfg = SingleCfg<TBN>;
  constexpr int STAGES = Cfg::STAGES, B_STAGE_BYTES = Cfg::B_STAGE_BYTES, STAGE_BYTES = Cfg::STAGE_BYTES;
  constexpr uint32_t TMEM_COLS = Cfg::TMEM_COLS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + STAGES * A_STAGE_BYTES;
  uint8_t* stg_all = smem + STAGES * STAGE_BYTES;  // epilogue staging, 4 warps x 2 x 4 KB
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(stg_all + STG_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* aux_bar = tempty_bar + 2;  // [4][2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aux_bar + 8);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int tiles_m = (p.M + BM - 1) / BM;
  const int tiles_n = (p.N + TBN - 1) / TBN;
  const int num_tiles = tiles_m * tiles_n;
  const int num_kb = p.K / BK;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&map_a);
    ptx::tma_prefetch(&map_b);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull_bar[b], 1);
      ptx::mbar_init(&tempty_bar[b], 128);
    }
    for (int q = 0; q < 8; ++q) ptx::mbar_init(&aux_bar[q], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 3 && lane == 0) {
    ptx::tma_prefetch(&em.c);
    if (EPI == AMDP_EPI_GELU) ptx::tma_prefetch(&em.c2);
    if (EPI == AMDP_EPI_RESIDUAL || EPI == AMDP_EPI_GELU_BWD || EPI == AMDP_EPI_ROWDOT) ptx::tma_prefetch(&em.aux);
  }
  if (warp == 2) ptx::tmem_alloc<TMEM_COLS>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  ptx::pdl_wait();  // setup above overlapped the previous kernel's tail (PDL)
  ptx::pdl_trigger();

  if (warp == 0) {
    {  // ---------------- TMA producer (warp-converged, elect.sync in the asm)
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int tm, tn;
        tile_coords(t, tiles_m, tiles_n, tm, tn);
        const int m0 = tm * BM, n0 = tn * TBN;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem_a + stage * A_STAGE_BYTES;
          uint8_t* sb = smem_b + stage * B_STAGE_BYTES;
          ptx::mbar_arrive_expect_tx_w(&full_bar[stage], STAGE_BYTES);
          const int k0 = kb * BK;
          if constexpr (A_MN) {
#pragma unroll
            for (int i = 0; i < BM / 64; ++i)
              ptx::tma_load_2d_w(sa + i * (64 * BK * 2), &map_a, &full_bar[stage], m0 + 64 * i, k0);
          } else {
            ptx::tma_load_2d_w(sa, &map_a, &full_bar[stage], k0, m0);
          }
          if constexpr (B_MN) {
#pragma unroll
            for (int i = 0; i < TBN / 64; ++i)
              ptx::tma_load_2d_w(sb + i * (64 * BK * 2), &map_b, &full_bar[stage], n0 + 64 * i, k0);
          } else {
            ptx::tma_load_2d_w(sb, &map_b, &full_bar[stage], k0, n0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    {  // ---------------- MMA issuer (warp-converged, elect.sync inside the asm)
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(BM, TBN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        ptx::mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * TBN;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const uint64_t a0 = ptx::umma_desc_sw128(ptx::smem_u32(smem_a + stage * A_STAGE_BYTES),
                                                   A_MN ? 64 * BK * 2 : 16, 1024);
          const uint64_t b0 = ptx::umma_desc_sw128(ptx::smem_u32(smem_b + stage * B_STAGE_BYTES),
                                                   B_MN ? 64 * BK * 2 : 16, 1024);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)  // MN-major: 16 K-rows of 128 B; K-major: 32 B along the row
            ptx::mma_bf16_ss_w(d_tmem, a0 + ((A_MN ? k * 2048 : k * 32) >> 4), b0 + ((B_MN ? k * 2048 : k * 32) >> 4),
                               idesc, (kb | k) != 0 ? 1u : 0u);
          ptx::mma_commit_w(&empty_bar[stage]);  // frees the smem slot when these MMAs retire
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        ptx::mma_commit_w(&tfull_bar[acc]);  // accumulator ready for the epilogue
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: warp (4+q) owns TMEM lanes [32q, 32q+32)
    const int q = warp - 4;
    int acc = 0;
    uint32_t acc_phase = 0, aux_phase = 0;
    int bsel = 0;
    uint8_t* stg = stg_all + q * 8192;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int tm, tn;
      tile_coords(t, tiles_m, tiles_n, tm, tn);
      ptx::mbar_wait(&tfull_bar[acc], acc_phase);
      ptx::tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * TBN;
      if constexpr (EPI == EPI_DISCARD) {
        uint32_t raw[32];
        for (int c = 0; c < TBN; c += 32) ptx::tmem_ld_32x32b_x32(t_row + c, raw);
        ptx::tmem_ld_wait();
      } else {
        pair_epilogue<EPI>(em, p, t_row, TBN, tn * TBN, tm * BM + q * 32, stg, &aux_bar[2 * q], aux_phase, bsel,
                           lane);
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) ptx::bulk_wait<0>();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

// ------------------------------------------------------------------ CTA-pair kernel
// cta_group::2 variant: a cluster of two CTAs computes a 256 x 256 tile with one
// tcgen05.mma (M=256) per K=16 step, issued by the even CTA.  CTA r loads A rows
// [m0 + 128 r, +128) and B rows [n0 + r W/2, +W/2) into its own smem; both CTAs' TMA
// bytes land on the even CTA's `full` barrier; each CTA's TMEM holds its 128 rows x W
// columns.
//
// Tail waves: with 74 pairs, a GEMM of T tiles runs ceil(T/74) tile-times while only
// T/74 are busy (N=2048 stage GEMMs: 256 tiles = 3.46 waves -> 4).  The last T mod 74
// tiles are therefore split along N into `tail_split` sub-tiles of width 256/s (one
// tcgen05.mma of N = 256/s per K step), so the final wave takes 1/s of a tile-time.
constexpr int PAIR_THREADS = 256;
constexpr int PBN = 256;

template <int NST>
struct PairCfg {
  static constexpr int B_HALF = PBN / 2;
  static constexpr int A_BYTES = 128 * BK * 2;
  static constexpr int B_BYTES = B_HALF * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int NSTAGE = NST;
  static constexpr int STG = 4 * 2 * 4096;  // epilogue staging: 4 warps x 2 x 4 KB
  static constexpr size_t SMEM = 1024 + NSTAGE * STAGE + STG + 256;
  static constexpr uint32_t TMEM = 512;
};

struct PairSched {
  int tiles_m, tiles_n;
  int full_tiles;   // tiles before the split tail (raster order)
  int tail_split;   // 1, 2 or 4
  int num_work;     // full_tiles + tail_split * (tiles - full_tiles)  (ksplit: + 2 * tail)
  int group_m;      // raster: tile rows per group (L2 reuse of B across consecutive tiles)
  // Weight-gradient tail (C += A B, fp32): the last partial wave's tiles split into two K
  // halves, all first halves listed before all second halves.  A second half reduce-adds into
  // C only after its first half's reduce-add has completed (flag = epoch per (tail tile,
  // CTA, epilogue warp)), so the fp32 summation order is fixed: (C + P0) + P1.
  int ksplit;       // 1 or 2
  int* flags;       // [tail tiles][2][4]
  int epoch;        // this launch's flag value
  // L2 policy of the operand loads (see raster_group): 0 none, 1 A streamed once (evict_first)
  // and B resident (evict_last), 2 the reverse
  int l2hint;
};

// Work item w -> output rows [m0, m0 + 256), columns [n0, n0 + width), K blocks [kb0, kb1);
// khalf: -1 whole K, 0 / 1 first / second half of K-split tail tile `tail` (ksplit = 2).
__device__ __forceinline__ void pair_work(const PairSched& s, int w, int num_kb, int& m0, int& n0, int& width,
                                          int& kb0, int& kb1, int& khalf, int& tail) {
  int t = w, part = 0, split = 1;
  kb0 = 0;
  kb1 = num_kb;
  khalf = -1;
  tail = 0;
  if (w >= s.full_tiles) {
    const int u = w - s.full_tiles;
    if (s.ksplit == 2) {
      const int ntail = (s.num_work - s.full_tiles) / 2;
      khalf = u >= ntail ? 1 : 0;
      tail = u - khalf * ntail;
      t = s.full_tiles + tail;
      const int mid = num_kb / 2;
      kb0 = khalf ? mid : 0;
      kb1 = khalf ? num_kb : mid;
    } else {
      split = s.tail_split;
      t = s.full_tiles + u / split;
      part = u % split;
    }
  }
  int tm, tn;
  tile_coords(t, s.tiles_m, s.tiles_n, tm, tn, s.group_m);
  width = PBN / split;
  m0 = tm * 256;
  n0 = tn * PBN + part * width;
}

template <bool A_MN, bool B_MN, int EPI, int NST>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PAIR_THREADS, 1)
    gemm_bf16_tc_pair(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                      const __grid_constant__ CUtensorMap map_b_tail, const __grid_constant__ EpiMaps em,
                      const EpiParams p, const PairSched sc) {
  using C = PairCfg<NST>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + C::NSTAGE * C::A_BYTES;
  uint8_t* stg_all = smem + C::NSTAGE * C::STAGE;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(stg_all + C::STG);
  uint64_t* empty_bar = full_bar + C::NSTAGE;
  uint64_t* tfull_bar = empty_bar + C::NSTAGE;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* aux_bar = tempty_bar + 2;  // [4][2]: per epilogue warp, per staging buffer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aux_bar + 8);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = ptx::cluster_rank();
  const int num_kb = p.K / BK;
  const int cluster = blockIdx.x / 2, nclusters = gridDim.x / 2;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&map_a);
    ptx::tma_prefetch(&map_b);
    if (sc.tail_split > 1) ptx::tma_prefetch(&map_b_tail);
    for (int s = 0; s < C::NSTAGE; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull_bar[b], 1);
      ptx::mbar_init(&tempty_bar[b], 2 * 128);
    }
    for (int q = 0; q < 8; ++q) ptx::mbar_init(&aux_bar[q], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 3 && lane == 0) {
    ptx::tma_prefetch(&em.c);
    if (EPI == AMDP_EPI_GELU) ptx::tma_prefetch(&em.c2);
    if (EPI == AMDP_EPI_RESIDUAL || EPI == AMDP_EPI_GELU_BWD || EPI == AMDP_EPI_ROWDOT) ptx::tma_prefetch(&em.aux);
  }
  if (warp == 2) ptx::tmem_alloc_pair<C::TMEM>(tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  ptx::pdl_wait();  // setup above overlapped the previous kernel's tail (PDL)
  ptx::pdl_trigger();

  if (warp == 0) {
    {  // TMA producer (warp-converged, elect.sync in the asm)
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t pol_stream = ptx::l2_policy_evict_first(), pol_keep = ptx::l2_policy_evict_last();
      const uint64_t pol_a = sc.l2hint == 1 ? pol_stream : pol_keep;
      const uint64_t pol_b = sc.l2hint == 1 ? pol_keep : pol_stream;
      for (int w = cluster; w < sc.num_work; w += nclusters) {
        int m0, n0, width, kb0, kb1, khalf, tail;
        pair_work(sc, w, num_kb, m0, n0, width, kb0, kb1, khalf, tail);
        const int ma = m0 + 128 * static_cast<int>(rank);
        const int half = width / 2;
        const int nb = n0 + half * static_cast<int>(rank);
        const uint32_t bytes = 2u * (C::A_BYTES + static_cast<uint32_t>(half) * BK * 2);
        const CUtensorMap* mb = (width == PBN || B_MN) ? &map_b : &map_b_tail;
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          const uint32_t fb = ptx::mapa(ptx::smem_u32(&full_bar[stage]), 0);
          if (rank == 0) ptx::mbar_arrive_expect_tx_w(&full_bar[stage], bytes);
          uint8_t* sa = smem_a + stage * C::A_BYTES;
          uint8_t* sb = smem_b + stage * C::B_BYTES;
          const int k0 = kb * BK;
          if (sc.l2hint == 0) {
            if constexpr (A_MN) {
              ptx::tma_load_2d_pair_w(sa, &map_a, fb, ma, k0);
              ptx::tma_load_2d_pair_w(sa + 64 * BK * 2, &map_a, fb, ma + 64, k0);
            } else {
              ptx::tma_load_2d_pair_w(sa, &map_a, fb, k0, ma);
            }
            if constexpr (B_MN) {
              for (int i = 0; i < half / 64; ++i)
                ptx::tma_load_2d_pair_w(sb + i * 64 * BK * 2, &map_b, fb, nb + 64 * i, k0);
            } else {
              ptx::tma_load_2d_pair_w(sb, mb, fb, k0, nb);
            }
          } else {
            if constexpr (A_MN) {
              ptx::tma_load_2d_pair_hint_w(sa, &map_a, fb, ma, k0, pol_a);
              ptx::tma_load_2d_pair_hint_w(sa + 64 * BK * 2, &map_a, fb, ma + 64, k0, pol_a);
            } else {
              ptx::tma_load_2d_pair_hint_w(sa, &map_a, fb, k0, ma, pol_a);
            }
            if constexpr (B_MN) {
              for (int i = 0; i < half / 64; ++i)
                ptx::tma_load_2d_pair_hint_w(sb + i * 64 * BK * 2, &map_b, fb, nb + 64 * i, k0, pol_b);
            } else {
              ptx::tma_load_2d_pair_hint_w(sb, mb, fb, k0, nb, pol_b);
            }
          }
          if (++stage == C::NSTAGE) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // warp-converged issue, elect.sync inside the asm
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int w = cluster; w < sc.num_work; w += nclusters) {
        int m0, n0, width, kb0, kb1, khalf, tail;
        pair_work(sc, w, num_kb, m0, n0, width, kb0, kb1, khalf, tail);
        const uint32_t idesc = ptx::idesc_bf16_f32(256, width, A_MN, B_MN);
        ptx::mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * PBN;
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const uint64_t a0 = ptx::umma_desc_sw128(ptx::smem_u32(smem_a + stage * C::A_BYTES),
                                                   A_MN ? 64 * BK * 2 : 16, 1024);
          const uint64_t b0 = ptx::umma_desc_sw128(ptx::smem_u32(smem_b + stage * C::B_BYTES),
                                                   B_MN ? 64 * BK * 2 : 16, 1024);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            ptx::mma_bf16_ss_pair_w(d_tmem, a0 + ((A_MN ? k * 2048 : k * 32) >> 4),
                                    b0 + ((B_MN ? k * 2048 : k * 32) >> 4), idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          ptx::mma_commit_pair_w(&empty_bar[stage], 0x3);
          if (++stage == C::NSTAGE) { stage = 0; phase ^= 1; }
        }
        ptx::mma_commit_pair_w(&tfull_bar[acc], 0x3);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    const int q = warp - 4;
    const uint32_t tempty_leader0 = ptx::mapa(ptx::smem_u32(&tempty_bar[0]), 0);
    const uint32_t tempty_leader1 = ptx::mapa(ptx::smem_u32(&tempty_bar[1]), 0);
    int acc = 0;
    uint32_t acc_phase = 0, aux_phase = 0;
    int bsel = 0;
    uint8_t* stg = stg_all + q * 8192;
    for (int w = cluster; w < sc.num_work; w += nclusters) {
      int m0, n0, width, kb0, kb1, khalf, tail;
      pair_work(sc, w, num_kb, m0, n0, width, kb0, kb1, khalf, tail);
      const int row0 = m0 + 128 * static_cast<int>(rank) + q * 32;
      int* const flag = sc.flags + (tail * 2 + static_cast<int>(rank)) * 4 + q;
      if (khalf == 1) {  // the first half's reduce-add into these rows has completed
        if (lane == 0) {
          while (ptx::ld_acquire_gpu(flag) != sc.epoch) __nanosleep(64);
          *flag = 0;  // consumed: the next launch (or a CUDA-graph replay of this one) starts clean
          ptx::fence_proxy_async_global();
        }
        __syncwarp();
      }
      ptx::mbar_wait(&tfull_bar[acc], acc_phase);
      ptx::tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * PBN;
      if constexpr (EPI == EPI_DISCARD) {
        uint32_t raw[32];
        for (int c = 0; c < width; c += 32) ptx::tmem_ld_32x32b_x32(t_row + c, raw);
        ptx::tmem_ld_wait();
      } else {
        pair_epilogue<EPI>(em, p, t_row, width, n0, row0, stg, &aux_bar[2 * q], aux_phase, bsel, lane);
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive_cluster(acc == 0 ? tempty_leader0 : tempty_leader1);
      if (khalf == 0 && lane == 0) {  // publish: this warp's reduce-adds are complete
        ptx::bulk_wait<0>();
        ptx::fence_proxy_async_global();
        ptx::st_release_gpu(flag, sc.epoch);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) ptx::bulk_wait<0>();
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_pair<C::TMEM>(tmem_base);
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qres;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qres) !=
            cudaSuccess ||
        qres != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// 2-D bf16 tensor map: inner dimension `inner` (contiguous), outer `outer` with
// leading dimension `ld` elements; box = {64, box_outer}, 128-byte swizzle.
bool make_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
              uint32_t box_outer, bool f32 = false, uint32_t box_inner = 64) {
  auto enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * (f32 ? 4 : 2)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int g_num_sms = 0;

// Launch state that is per device (function attributes, occupancy, the K-split flag buffer),
// keyed by the current device ordinal; thread-safe.
constexpr int kMaxDevices = 64;
int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  return d;
}
std::mutex g_dev_mu;

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// Tail split (see the pair kernel): the s in {1, 2, 4} minimising the tail's length
// ceil(s R / P) / s tile-times (R = tiles mod P, P = pairs).  Only for K-major B, i.e. the
// forward GEMMs, which run alone on the compute stream: the backward's activation- and
// weight-gradient GEMMs (MN-major B) run concurrently on two streams and fill each other's
// tails, where split sub-tiles measured slower (scripts/task_durations.py, B tasks).
// Raster (tile rows per group, see tile_coords).  Row-major (group 1: consecutive tiles walk
// along N, so a wave of 74 pairs covers ~74 / tiles_n full tile rows: every A panel is read
// once and B stays L2-resident) unless A is the operand that fits in L2 (<= 48 MB of the
// 126 MB) and B is much larger (the LM-head forward: 206 MB of head weights), where the walk
// is column-major (group = tiles_m) so that B is streamed once.  Measured under the power cap
// (scripts/gemm_sustained.py, same box): row-major vs the previous 8-row groups +3.8% fc1
// forward (1312 TF/s, above cuBLAS's 1292), +4.3% fc1 activation gradient, +3.9% fc2
// forward, +4.4% fc1 weight gradient (DRAM reads 392 -> 313 MB per launch);
// profiles/r02/gemm_raster.
int raster_group(int M, int N, int K, int tiles_m) {
  static const int forced = env_int("AMDP_GEMM_GROUP_M", 0);
  if (forced > 0) return forced;
  const double a = 2.0 * M * static_cast<double>(K), b = 2.0 * N * static_cast<double>(K);
  const double fits = 48.0 * 1024 * 1024;
  if (a <= fits && b > 2 * a) return tiles_m;
  return 1;
}

PairSched pair_schedule(int M, int N, bool b_mn, int pairs, int K = 0) {
  PairSched s;
  s.tiles_m = (M + 255) / 256;
  s.tiles_n = (N + PBN - 1) / PBN;
  const int T = s.tiles_m * s.tiles_n;
  static const int forced = env_int("AMDP_GEMM_TAIL", -1);
  const int P = pairs;
  const int R = T % P;
  int best = 1;
  // GEMMs with fewer tiles than pairs (BERT-large / 350M shapes) split every tile along N too
  static const int small_split = env_int("AMDP_GEMM_SMALL_SPLIT", 1);
  if (R != 0 && (T > P || small_split) && !b_mn) {
    double best_len = 1.0;
    for (int cand = 2; cand <= 4; cand *= 2) {
      const double len = static_cast<double>((cand * R + P - 1) / P) / cand;
      if (len < best_len - 1e-9) { best_len = len; best = cand; }
    }
  }
  if (forced == 1 || ((forced == 2 || forced == 4) && !b_mn)) best = forced;
  s.tail_split = best;
  s.group_m = K > 0 ? raster_group(M, N, K, s.tiles_m) : GROUP_M;
  s.l2hint = 0;
  // L2 policies (AMDP_GEMM_L2HINT=1): the streamed operand evict_first, the resident one
  // evict_last.  Isolated fc1 weight gradient: DRAM reads 317 -> 288 MB, writes 45 -> 24 MB
  // (1.03x algorithmic), sustained +1-4%; but in the model the "streamed" operand (the
  // activation gradient dU) is read again by the concurrent activation-gradient GEMM, which
  // then misses: 1.3B window 1.3% slower.  Off by default.
  if (K > 0) {
    static const int hints = env_int("AMDP_GEMM_L2HINT", 0);
    const double a = 2.0 * M * static_cast<double>(K), b = 2.0 * N * static_cast<double>(K);
    const double fits = 48.0 * 1024 * 1024;
    if (hints && s.group_m == 1 && b <= fits && a > 2 * b) s.l2hint = 1;
    if (hints && s.group_m == s.tiles_m && s.tiles_m > 1 && a <= fits && b > 2 * a) s.l2hint = 2;
  }
  s.full_tiles = best == 1 ? T : T - R;
  s.num_work = s.full_tiles + best * (T - s.full_tiles);
  s.ksplit = 1;
  s.flags = nullptr;
  s.epoch = 0;
  return s;
}

// Co-resident 2-CTA clusters for this smem footprint (GPC sizes can leave SMs unpaired,
// so this may be below #SMs / 2); the persistent grid never exceeds it.
template <int NST>
int max_pairs() {
  static std::atomic<int> pairs_of[kMaxDevices];
  std::atomic<int>& pairs_a = pairs_of[current_device()];
  int pairs = pairs_a.load();
  if (pairs == 0) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 2;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.gridDim = dim3(g_num_sms, 1, 1);
    cfg.blockDim = dim3(PAIR_THREADS, 1, 1);
    cfg.dynamicSmemBytes = PairCfg<NST>::SMEM;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    auto kern = gemm_bf16_tc_pair<false, false, AMDP_EPI_STORE_BF16, NST>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(PairCfg<NST>::SMEM));
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = g_num_sms / 2;
    }
    pairs = n < g_num_sms / 2 ? n : g_num_sms / 2;
    pairs_a.store(pairs);
    if (getenv("AMDP_GEMM_DEBUG")) fprintf(stderr, "amdp_gemm: %d co-resident CTA pairs (NST=%d)\n", pairs, NST);
  }
  return pairs;
}

template <bool A_MN, bool B_MN, int EPI, int NST>
int launch_pair(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mbt, const EpiMaps& em,
                const EpiParams& p, cudaStream_t s) {
  auto kern = gemm_bf16_tc_pair<A_MN, B_MN, EPI, NST>;
  const int dev = current_device();
  static std::atomic<bool> attr_set[kMaxDevices];
  if (!attr_set[dev].load()) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(PairCfg<NST>::SMEM));
    if (e != cudaSuccess) return e;
    attr_set[dev].store(true);
  }
  const int pairs = max_pairs<NST>();
  PairSched sc = pair_schedule(p.M, p.N, B_MN, pairs, p.K);
  if constexpr (EPI == AMDP_EPI_ACCUM_F32) {
    // K-split of a partial last wave that fits in one wave as halves (fc1 / fc2 / LM-head
    // weight gradients at the 1.3B shapes); deterministic (see PairSched)
    static const int ks_env = env_int("AMDP_GEMM_KSPLIT", 1);
    const int T = sc.tiles_m * sc.tiles_n, R = T % pairs, num_kb = p.K / BK;
    if (ks_env != 0 && sc.tail_split == 1 && (T > pairs || ks_env == 2) && R > 0 && 2 * R <= pairs &&
        num_kb >= 8) {
      // one flag buffer per (device, stream): launches on one stream are ordered, so the
      // epoch tells consecutive ones apart; GEMMs on different streams (the executor's
      // concurrent compute / weight-gradient streams) never share flags
      static std::map<std::pair<int, cudaStream_t>, std::pair<int*, int>> flags_of;
      int* flags;
      int epoch;
      {
        std::lock_guard<std::mutex> lk(g_dev_mu);
        auto& slot = flags_of[{dev, s}];
        if (!slot.first) {
          if (cudaMalloc(&slot.first, 2048 * 8 * sizeof(int)) != cudaSuccess) return AMDP_ERR_CUDA;
          if (cudaMemset(slot.first, 0, 2048 * 8 * sizeof(int)) != cudaSuccess) return AMDP_ERR_CUDA;
        }
        flags = slot.first;
        epoch = ++slot.second;
      }
      if (R <= 2048) {
        sc.ksplit = 2;
        sc.full_tiles = T - R;
        sc.num_work = sc.full_tiles + 2 * R;
        sc.flags = flags;
        sc.epoch = epoch;
      }
    }
  }
  const int grid = 2 * (sc.num_work < pairs ? sc.num_work : pairs);
  cudaError_t e = launch_pdl(kern, dim3(grid), dim3(PAIR_THREADS), PairCfg<NST>::SMEM, s, ma, mb, mbt, em, p, sc);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <bool A_MN, bool B_MN, int EPI, int TBN>
int launch_single(const CUtensorMap& ma, const CUtensorMap& mb, const EpiMaps& em, const EpiParams& p,
                  cudaStream_t s) {
  auto kern = gemm_bf16_tcgen05<A_MN, B_MN, EPI, TBN>;
  constexpr size_t smem = SingleCfg<TBN>::SMEM;
  static std::atomic<bool> attr_set[kMaxDevices];
  const int dev = current_device();
  if (!attr_set[dev].load()) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr_set[dev].store(true);
  }
  const int tiles = ((p.M + BM - 1) / BM) * ((p.N + TBN - 1) / TBN);
  const int grid = tiles < g_num_sms ? tiles : g_num_sms;
  cudaError_t e = launch_pdl(kern, dim3(grid), dim3(NUM_THREADS), smem, s, ma, mb, em, p);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// MODE 0: single-CTA 128x256 tiles; MODE 128: single-CTA 128x128 tiles; MODE 256: CTA-pair
// 256x256 tiles (+ split tail).
template <bool A_MN, bool B_MN, int EPI>
int launch(int mode, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mbt, const EpiMaps& em,
           const EpiParams& p, cudaStream_t s) {
  if (mode == 0) return launch_single<A_MN, B_MN, EPI, 256>(ma, mb, em, p, s);
  if (mode == 128) return launch_single<A_MN, B_MN, EPI, 128>(ma, mb, em, p, s);
  static const int nst = env_int("AMDP_GEMM_STAGES", 6);
  if (nst == 4) return launch_pair<A_MN, B_MN, EPI, 4>(ma, mb, mbt, em, p, s);
  return launch_pair<A_MN, B_MN, EPI, 6>(ma, mb, mbt, em, p, s);
}

template <bool A_MN, bool B_MN>
int dispatch_epi(int mode, int epi, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mbt,
                 const EpiMaps& em, const EpiParams& p, cudaStream_t s) {
  switch (epi) {
    case AMDP_EPI_STORE_BF16: {
      static const bool discard = getenv("AMDP_GEMM_DISCARD") != nullptr;
      if (discard) return launch<A_MN, B_MN, EPI_DISCARD>(mode, ma, mb, mbt, em, p, s);
      return launch<A_MN, B_MN, AMDP_EPI_STORE_BF16>(mode, ma, mb, mbt, em, p, s);
    }
    case AMDP_EPI_GELU: return launch<A_MN, B_MN, AMDP_EPI_GELU>(mode, ma, mb, mbt, em, p, s);
    case AMDP_EPI_RESIDUAL: return launch<A_MN, B_MN, AMDP_EPI_RESIDUAL>(mode, ma, mb, mbt, em, p, s);
    case AMDP_EPI_ACCUM_F32: return launch<A_MN, B_MN, AMDP_EPI_ACCUM_F32>(mode, ma, mb, mbt, em, p, s);
    case AMDP_EPI_GELU_BWD: return launch<A_MN, B_MN, AMDP_EPI_GELU_BWD>(mode, ma, mb, mbt, em, p, s);
    case AMDP_EPI_STORE_F32: return launch<A_MN, B_MN, AMDP_EPI_STORE_F32>(mode, ma, mb, mbt, em, p, s);
    case AMDP_EPI_ROWDOT:
      if constexpr (!A_MN && !B_MN) return launch<A_MN, B_MN, AMDP_EPI_ROWDOT>(mode, ma, mb, mbt, em, p, s);
      break;
  }
  return AMDP_ERR_INVALID;
}

int gemm_pairs() {
  static const int nst = env_int("AMDP_GEMM_STAGES", 6);
  return nst == 4 ? max_pairs<4>() : max_pairs<6>();
}

// Tile shape per problem: CTA pairs with 256 x 256 tiles whenever M >= 256 (measured at the
// 1.3B shapes, profiles/r01_gemm_modes.txt: +5-13% over single-CTA 128x256 tiles).
int choose_mode(int M, int N, int K, bool a_mn, bool b_mn) {
  (void)a_mn;
  (void)b_mn;
  static const int forced = env_int("AMDP_GEMM_MODE", -1);
  if (forced == 0 || forced == 128 || forced == 256) return forced;
  // CTA pairs everywhere M allows, except small products (< 20 GFLOP: the BERT-large layer
  // GEMMs at 2048 tokens, 350M's out-projection), which run as single-CTA 128x256 tiles: with
  // the executor's concurrent streams a small GEMM then occupies half the SMs per tile and
  // leaves the rest to other logical devices' kernels (BERT-large D8 +7%, same box A/B;
  // GPT-1.3B's >= 69 GFLOP GEMMs stay on pairs, which are 6% faster there).  (Weight-gradient
  // GEMMs, A and B MN-major, issue four TMA boxes per stage and CTA; with a single-lane
  // producer that issue loop starved the pair kernel: 1081 TF/s sustained vs 1136 on
  // single-CTA tiles; warp-converged issue: 1189.)
  static const double small = env_int("AMDP_GEMM_SMALL_GFLOP", 20) * 1e9;
  if (M >= 256 && 2.0 * M * static_cast<double>(N) * K >= small) return 256;
  // Single-CTA tiles of 128 x 128 (AMDP_GEMM_NARROW=1: where they take fewer tile-times than
  // 128 x 256, waves(2T) / 2 < waves(T); =2 always).  In isolation they cut the BERT-large
  // layer GEMMs from 210 to 184 us (fc2 forward 24.2 -> 15.2 us, fc1 activation gradient
  // 22.9 -> 14.7, out-projection weight gradient 15.3 -> 9.9; cuBLAS 167 us for the set,
  // scripts/gemm_small.py), but inside the folded BERT-large D=8 window, where 8 logical
  // devices' kernels share the SMs, the wider tiles' lower per-tile overhead wins: 338k vs
  // 325k tokens/s (same box, A/B twice).  Off by default.
  static const int narrow = env_int("AMDP_GEMM_NARROW", 0);
  if (narrow == 2) return 128;
  if (narrow) {
    const int tm = (M + BM - 1) / BM, t256 = tm * ((N + 255) / 256), t128 = tm * ((N + 127) / 128);
    const int w256 = (t256 + g_num_sms - 1) / g_num_sms, w128 = (t128 + g_num_sms - 1) / g_num_sms;
    if (w128 < 2 * w256) return 128;
  }
  return 0;
}

}  // namespace
}  // namespace amdp

extern "C" int amdp_gemm(const amdp_gemm_args* a, amdp_stream_t stream) {
  using namespace amdp;
  if (!a || a->M <= 0 || a->N <= 0 || a->K <= 0 || a->K % BK != 0) return AMDP_ERR_INVALID;
  if (a->N % 8 != 0 || a->ldc % 4 != 0) return AMDP_ERR_INVALID;
  if (a->epilogue < 0 || a->epilogue > AMDP_EPI_ROWDOT) return AMDP_ERR_INVALID;
  if (a->epilogue == AMDP_EPI_ROWDOT &&
      (!a->aux || !a->rowdot || a->a_mn_major || a->b_mn_major || a->rowdot_seg <= 0 || a->rowdot_seg % 64 != 0 ||
       a->N % a->rowdot_seg != 0 || a->rowdot_seq <= 0 || a->M % a->rowdot_seq != 0))
    return AMDP_ERR_INVALID;
  if ((a->epilogue == AMDP_EPI_RESIDUAL || a->epilogue == AMDP_EPI_GELU_BWD) && !a->aux)
    return AMDP_ERR_INVALID;
  if (a->epilogue == AMDP_EPI_GELU && !a->C2) return AMDP_ERR_INVALID;
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) return AMDP_ERR_CUDA;
  }
  const int mode = choose_mode(a->M, a->N, a->K, a->a_mn_major != 0, a->b_mn_major != 0);
  CUtensorMap ma, mb, mbt;
  bool ok;
  if (a->a_mn_major)  // A stored [K][lda], M contiguous
    ok = make_map(&ma, a->A, a->M, a->K, a->lda, BK);
  else  // A stored [M][lda], K contiguous (128 rows per CTA in both kernels)
    ok = make_map(&ma, a->A, a->K, a->M, a->lda, BM);
  if (!ok) return AMDP_ERR_TMA;
  if (a->b_mn_major) {
    ok = make_map(&mb, a->B, a->N, a->K, a->ldb, BK);
    mbt = mb;
  } else {  // B rows per CTA: 256 / 128 (single) or 128 (pair); tail sub-tiles 128 / s
    ok = make_map(&mb, a->B, a->K, a->N, a->ldb, mode == 0 ? BN : mode == 128 ? 128 : PBN / 2);
    if (ok && mode == 256) {
      const PairSched sc = pair_schedule(a->M, a->N, false, gemm_pairs());
      ok = make_map(&mbt, a->B, a->K, a->N, a->ldb, PBN / 2 / sc.tail_split);
    } else {
      mbt = mb;
    }
  }
  if (!ok) return AMDP_ERR_TMA;
  EpiMaps em;
  {  // TMA-store epilogue maps (box 32 rows x 128 bytes)
    const bool f32 = a->epilogue == AMDP_EPI_ACCUM_F32 || a->epilogue == AMDP_EPI_STORE_F32;
    ok = make_map(&em.c, a->C, a->N, a->M, a->ldc, 32, f32, f32 ? 32 : 64);
    em.c2 = em.c;
    em.aux = em.c;
    if (ok && a->epilogue == AMDP_EPI_GELU) ok = make_map(&em.c2, a->C2, a->N, a->M, a->ldc2, 32);
    if (ok && (a->epilogue == AMDP_EPI_RESIDUAL || a->epilogue == AMDP_EPI_GELU_BWD || a->epilogue == AMDP_EPI_ROWDOT))
      ok = make_map(&em.aux, a->aux, a->N, a->M, a->ld_aux, 32);
    if (!ok) return AMDP_ERR_TMA;
  }
  EpiParams p{a->M, a->N, a->K, a->C, a->ldc,
              static_cast<const __nv_bfloat16*>(a->aux), a->ld_aux,
              static_cast<__nv_bfloat16*>(a->C2), a->ldc2, a->alpha,
              a->rowdot, a->rowdot_seg, a->rowdot_seq};
  if (a->epilogue == AMDP_EPI_ROWDOT) {
    // tiles (or tail sub-tiles) narrower than a segment split it between two CTAs (atomicAdd
    // onto zero)
    const int width = mode == 256 ? PBN / pair_schedule(a->M, a->N, false, gemm_pairs()).tail_split : mode == 128 ? 128 : BN;
    if (width < a->rowdot_seg) {
      const cudaError_t e = cudaMemsetAsync(a->rowdot, 0, static_cast<size_t>(a->M) * (a->N / a->rowdot_seg) * sizeof(float),
                                            reinterpret_cast<cudaStream_t>(stream));
      if (e != cudaSuccess) return e;
    }
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int am = a->a_mn_major ? 1 : 0, bm = a->b_mn_major ? 1 : 0;
  if (!am && !bm) return dispatch_epi<false, false>(mode, a->epilogue, ma, mb, mbt, em, p, s);
  if (!am && bm) return dispatch_epi<false, true>(mode, a->epilogue, ma, mb, mbt, em, p, s);
  if (am && !bm) return dispatch_epi<true, false>(mode, a->epilogue, ma, mb, mbt, em, p, s);
  return dispatch_epi<true, true>(mode, a->epilogue, ma, mb, mbt, em, p, s);
}
