// Tensor-pipe cost per tcgen05.mma (K16) for the operand shapes the attention kernels issue:
// one CTA, one issuing thread, R rounds of 8 MMAs into one TMEM accumulator, cycles/instruction.
#include <cstdio>
#include <cuda_runtime.h>
#include "kernels/sm100_ptx.cuh"
using namespace amdp;
enum { SS_KK = 0, SS_KMN = 1, TS_MN = 2, SS_KK_N256 = 3, TS_MN_N64 = 4 };
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
  if (threadIdx.x == 0) {
    const uint32_t a = ptx::smem_u32(sm), b = a + 32768;
    constexpr int N = MODE == SS_KK_N256 ? 256 : (MODE == TS_MN_N64 ? 64 : 128);
    constexpr bool bmn = MODE == SS_KMN || MODE == TS_MN || MODE == TS_MN_N64;
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, N, false, bmn);
    long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
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
int main() {
  long long* d; cudaMalloc(&d, 8);
  run<SS_KK>("SS M128 N128 K/K-major", d);
  run<SS_KK_N256>("SS M128 N256 K/K-major", d);
  run<SS_KMN>("SS M128 N128 B MN-major", d);
  run<TS_MN>("TS M128 N128 B MN-major", d);
  run<TS_MN_N64>("TS M128 N64 B MN-major", d);
  return 0;
}
