// Tensor-pipe cost per tcgen05.mma (K16) for the operand shapes the attention kernels issue:
// one CTA, one issuing thread, R rounds of 8 MMAs into one TMEM accumulator, cycles/instruction.
#include <cstdio>
#include <cuda_runtime.h>
#include "kernels/sm100_ptx.cuh"
using namespace amdp;
enum { SS_KK = 0, SS_KMN = 1, TS_MN = 2, SS_KK_N256 = 3, TS_MN_N64 = 4, SS_KK_N64 = 5, DQ_MIX = 6, DQ128_MIX = 7, TS_KK = 8, W_SS_N64 = 9, W_TS_N64 = 10, W_SS_N128 = 11 };
template <int MODE>
__global__ void probe(int rounds, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc<512>(&slot);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (MODE >= W_SS_N64 && threadIdx.x < 32) {  // warp-converged issue (elect.sync in the asm)
    const uint32_t a = ptx::smem_u32(sm), b = a + 32768;
    constexpr int N = MODE == W_SS_N128 ? 128 : 64;
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, N, false, MODE == W_TS_N64);
    const uint64_t da = ptx::umma_desc_sw128(a, 16, 1024), db = ptx::umma_desc_sw128(b, 16, 1024);
    const uint64_t dbm = ptx::umma_desc_sw128(b, 16384, 1024);
    long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (MODE == W_TS_N64)
          ptx::mma_bf16_ts_w(tmem + 256, tmem + kk * 8, dbm + ((kk * 2048) >> 4), id, 1u);
        else
          ptx::mma_bf16_ss_w(tmem + 256, da + (((kk & 3) * 32) >> 4), db + (((kk & 3) * 32) >> 4), id, 1u);
      }
    }
    ptx::mma_commit_w(&bar);
    ptx::mbar_wait(&bar, 0);
    if (threadIdx.x == 0) out[0] = clock64() - t0;
  } else if (MODE < W_SS_N64 && threadIdx.x == 0) {
    const uint32_t a = ptx::smem_u32(sm), b = a + 32768;
    constexpr int N = MODE == SS_KK_N256 ? 256 : ((MODE == TS_MN_N64 || MODE == SS_KK_N64) ? 64 : 128);
    constexpr bool bmn = MODE == SS_KMN || MODE == TS_MN || MODE == TS_MN_N64;
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, N, false, bmn);
    long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
      if (MODE == DQ128_MIX) {  // current dQ block: S (TS N128) | dP (SS N128) | dQ (TS N128, B MN-major)
        constexpr uint32_t id_s = ptx::idesc_bf16_f32(128, 128, false, false);
        constexpr uint32_t id_g = ptx::idesc_bf16_f32(128, 128, false, true);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma_bf16_ts(tmem, tmem + 448 + (kk & 7) * 8, ptx::umma_desc_sw128(b + (kk & 3) * 32, 16, 1024), id_s, kk > 0);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma_bf16_ss(tmem + 128, ptx::umma_desc_sw128(a + (kk & 3) * 32, 16, 1024),
                           ptx::umma_desc_sw128(b + (kk & 3) * 32, 16, 1024), id_s, kk > 0);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma_bf16_ts(tmem + 256, tmem + 384 + kk * 8, ptx::umma_desc_sw128(b + kk * 2048, 16384, 1024), id_g, 1u);
        continue;
      }
      if (MODE == TS_KK) {
        constexpr uint32_t id_s = ptx::idesc_bf16_f32(128, 128, false, false);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma_bf16_ts(tmem, tmem + 448 + (kk & 7) * 8, ptx::umma_desc_sw128(b + (kk & 3) * 32, 16, 1024), id_s, 1u);
        continue;
      }
      if (MODE == DQ_MIX) {  // dQ kernel block: S, dP (M128 N64 K128, SS) + dQ (M128 N128 K64, TS)
        constexpr uint32_t id64 = ptx::idesc_bf16_f32(128, 64, false, false);
        constexpr uint32_t idg = ptx::idesc_bf16_f32(128, 128, false, true);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          ptx::mma_bf16_ss(tmem, ptx::umma_desc_sw128(a + (kk & 3) * 32, 16, 1024),
                           ptx::umma_desc_sw128(b + (kk & 3) * 32, 16, 1024), id64, 1u);
          ptx::mma_bf16_ss(tmem + 64, ptx::umma_desc_sw128(a + 16384 + (kk & 3) * 32, 16, 1024),
                           ptx::umma_desc_sw128(b + 8192 + (kk & 3) * 32, 16, 1024), id64, 1u);
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          ptx::mma_bf16_ts(tmem + 384, tmem + 128 + kk * 8, ptx::umma_desc_sw128(b + kk * 2048, 8192, 1024), idg, 1u);
        continue;
      }
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (MODE == TS_MN || MODE == TS_MN_N64)
          ptx::mma_bf16_ts(tmem + 256, tmem + kk * 8, ptx::umma_desc_sw128(b + kk * 2048, 16384, 1024), id, 1u);
        else if (bmn)
          ptx::mma_bf16_ss(tmem + 256, ptx::umma_desc_sw128(a + (kk & 3) * 32, 16, 1024),
                           ptx::umma_desc_sw128(b + kk * 2048, 16384, 1024), id, 1u);
        else
          ptx::mma_bf16_ss(tmem + 256, ptx::umma_desc_sw128(a + (kk & 3) * 32, 16, 1024),
                           ptx::umma_desc_sw128(b + (kk & 3) * 32, 16, 1024), id, 1u);
      }
    }
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    long long t1 = clock64();
    *out = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}
template <int MODE>
void run(const char* name, long long* d) {
  auto k = probe<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int rounds = 512;
  k<<<1, 128, 100 * 1024>>>(rounds, d); cudaDeviceSynchronize();
  k<<<1, 128, 100 * 1024>>>(rounds, d); cudaError_t e = cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %6.1f cycles per K16 MMA  (%s)\n", name, double(c) / (rounds * 8), cudaGetErrorString(e));
}
// Issue-queue depth: how long the issuing thread takes to push 64 MMAs (N128: 64 cyc each)
// compared with their completion.
__global__ void issue_depth(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc<512>(&slot);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = ptx::smem_u32(sm), b = a + 32768;
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, 128, false, false);
    long long t0 = clock64(), tk[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        ptx::mma_bf16_ss(tmem, ptx::umma_desc_sw128(a + (kk & 3) * 32, 16, 1024),
                         ptx::umma_desc_sw128(b + (kk & 3) * 32, 16, 1024), id, 1u);
      tk[r] = clock64();
    }
    ptx::mma_commit(&bar);
    long long t1 = clock64();
    ptx::mbar_wait(&bar, 0);
    long long t2 = clock64();
    for (int r = 0; r < 8; ++r) out[r] = tk[r] - t0;
    out[8] = t1 - t0; out[9] = t2 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}
// TS MMAs (M128 N128, A from TMEM) while LOADERS warps stream tcgen05.ld from other TMEM
// columns: does the softmax's TMEM traffic slow the tensor pipe?
__global__ void ts_contention(int rounds, int loaders, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); stop = 0; }
  if (threadIdx.x < 32) ptx::tmem_alloc<512>(&slot);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    const uint32_t b = ptx::smem_u32(sm) + 32768;
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, 128, false, true);
    long long t0 = clock64();
    for (int r = 0; r < rounds; ++r)
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        ptx::mma_bf16_ts(tmem + 256, tmem + 384 + kk * 8, ptx::umma_desc_sw128(b + kk * 2048, 16384, 1024), id, 1u);
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    out[0] = clock64() - t0;
    stop = 1;
  } else if (warp >= 4 && warp < 4 + loaders) {
    const uint32_t lanes = static_cast<uint32_t>((warp & 3) * 32) << 16;
    uint32_t acc = 0;
    long long n = 0;
    while (!stop) {
      uint32_t v[32];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        ptx::tmem_ld_32x32b_x32(tmem + lanes + c * 32, v);
        ptx::tmem_ld_wait();
        acc += v[0] ^ v[31];
      }
      ++n;
    }
    if ((threadIdx.x & 31) == 0) out[1 + (warp - 4)] = n;
    if (acc == 0x12345) out[20] = acc;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}
int main() {
  long long* d; cudaMalloc(&d, 200);
  {
    cudaFuncSetAttribute(ts_contention, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int loaders : {0, 4, 8}) {
      const int rounds = 256;
      for (int i = 0; i < 2; ++i) { ts_contention<<<1, 384, 100 * 1024>>>(rounds, loaders, d); cudaDeviceSynchronize(); }
      long long h[12]; cudaMemcpy(h, d, 96, cudaMemcpyDeviceToHost);
      long long tot = 0; for (int w = 0; w < loaders; ++w) tot += h[1 + w];
      printf("TS M128 N128 with %d tcgen05.ld warps: %.1f cycles/MMA; loader bytes/cycle %.1f\n", loaders,
             double(h[0]) / (rounds * 8), loaders ? double(tot) * 16384.0 / h[0] : 0.0);
    }
  }
  {
    cudaFuncSetAttribute(issue_depth, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int i = 0; i < 2; ++i) { issue_depth<<<1, 128, 100 * 1024>>>(d); cudaDeviceSynchronize(); }
    long long h[10]; cudaMemcpy(h, d, 80, cudaMemcpyDeviceToHost);
    printf("issue of 64 x (M128 N128 K16) MMAs: after each 8:");
    for (int r = 0; r < 8; ++r) printf(" %lld", h[r]);
    printf("; commit issued %lld; all complete %lld cycles\n", h[8], h[9]);
  }
  run<SS_KK>("SS M128 N128 K/K-major", d);
  run<SS_KK_N256>("SS M128 N256 K/K-major", d);
  run<SS_KMN>("SS M128 N128 B MN-major", d);
  run<TS_MN>("TS M128 N128 B MN-major", d);
  run<TS_MN_N64>("TS M128 N64 B MN-major", d);
  run<SS_KK_N64>("SS M128 N64 K/K-major", d);
  run<DQ_MIX>("dQ block (16 SS N64 + 4 TS N128) per 8", d);
  run<TS_KK>("TS M128 N128 B K-major", d);
  run<DQ128_MIX>("dQ128 block (8 TS + 8 SS + 8 TS, N128) per 8", d);
  run<W_SS_N64>("warp-issue SS M128 N64", d);
  run<W_TS_N64>("warp-issue TS M128 N64", d);
  run<W_SS_N128>("warp-issue SS M128 N128", d);
  return 0;
}
