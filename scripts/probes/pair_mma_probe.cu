// Tensor-pipe cost per cta_group::2 tcgen05.mma (M256 N256 K16) with K-major vs MN-major
// operands: one CTA pair, the even CTA issues R rounds of 8 MMAs into one TMEM accumulator
// from fixed shared-memory tiles (no TMA), cycles per instruction.
#include <cstdio>
#include <cuda_runtime.h>
#include "kernels/sm100_ptx.cuh"
using namespace amdp;
template <bool A_MN, bool B_MN>
__global__ void __cluster_dims__(2, 1, 1) probe(int rounds, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  const uint32_t rank = ptx::cluster_rank();
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc_pair<512>(&slot);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (rank == 0 && threadIdx.x < 32) {
    constexpr int BK = 64;
    const uint32_t a = ptx::smem_u32(sm), b = a + 32768;
    constexpr uint32_t id = ptx::idesc_bf16_f32(256, 256, A_MN, B_MN);
    const uint64_t da = ptx::umma_desc_sw128(a, A_MN ? 64 * BK * 2 : 16, 1024);
    const uint64_t db = ptx::umma_desc_sw128(b, B_MN ? 64 * BK * 2 : 16, 1024);
    long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int kk = k & 3;
        ptx::mma_bf16_ss_pair_w(tmem, da + ((A_MN ? kk * 2048 : kk * 32) >> 4), db + ((B_MN ? kk * 2048 : kk * 32) >> 4),
                                id, 1u);
      }
    }
    ptx::mma_commit_pair_w(&bar, 0x1);
    ptx::mbar_wait(&bar, 0);
    if (threadIdx.x == 0) out[0] = clock64() - t0;
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc_pair<512>(tmem); }
}
template <bool A_MN, bool B_MN>
void run(const char* name, long long* d) {
  auto k = probe<A_MN, B_MN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int rounds = 512;
  for (int i = 0; i < 2; ++i) { k<<<2, 128, 100 * 1024>>>(rounds, d); cudaDeviceSynchronize(); }
  cudaError_t e = cudaGetLastError();
  long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("%-24s %6.1f cycles per M256 N256 K16 pair MMA (%s)\n", name, double(c) / (rounds * 8), cudaGetErrorString(e));
}
int main() {
  long long* d; cudaMalloc(&d, 64);
  run<false, false>("A K-major, B K-major", d);
  run<true, false>("A MN-major, B K-major", d);
  run<false, true>("A K-major, B MN-major", d);
  run<true, true>("A MN-major, B MN-major", d);
  return 0;
}
