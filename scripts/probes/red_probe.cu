// L2 reduction bandwidth: fp32 add of a [rows x 128] partial into a global accumulator,
// (a) warp-coalesced red.global.add.f32, (b) red.global.add.v4.f32, (c) TMA-free bulk
// cp.reduce.async.bulk (1-D, smem -> global, add.f32).  Each CTA reduces `reps` 32 KB tiles
// into accumulator rows chosen round-robin over a 64 MB buffer (so traffic mostly hits L2).
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>
__global__ void red_scalar(float* acc, int reps, int nrows) {
  for (int r = 0; r < reps; ++r) {
    const int row0 = ((blockIdx.x * reps + r) * 64) % nrows;
    // 64 rows x 128 floats; 128 threads: thread t handles column t of all 64 rows
    for (int i = 0; i < 64; ++i)
      atomicAdd(acc + static_cast<size_t>(row0 + i) * 128 + threadIdx.x, 1.0f);
  }
}
__global__ void red_v4(float* acc, int reps, int nrows) {
  for (int r = 0; r < reps; ++r) {
    const int row0 = ((blockIdx.x * reps + r) * 64) % nrows;
    // 64 rows x 128 floats = 2048 float4; 128 threads x 16
    for (int i = 0; i < 16; ++i) {
      const int e = i * 128 + threadIdx.x;  // float4 index
      float* p = acc + static_cast<size_t>(row0) * 128 + 4 * e;
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
    }
  }
}
__global__ void red_bulk(float* acc, int reps, int nrows) {
  __shared__ __align__(128) float tile[64 * 128];
  for (int i = threadIdx.x; i < 64 * 128; i += blockDim.x) tile[i] = 1.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int r = 0; r < reps; ++r) {
      const int row0 = ((blockIdx.x * reps + r) * 64) % nrows;
      float* dst = acc + static_cast<size_t>(row0) * 128;
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
                   "r"(static_cast<uint32_t>(__cvta_generic_to_shared(tile))), "r"(32768) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
}
int main() {
  const int nrows = 64 * 2048;  // 32 MB accumulator
  float* acc; cudaMalloc(&acc, size_t(nrows) * 128 * 4); cudaMemset(acc, 0, size_t(nrows) * 128 * 4);
  const int grid = 148 * 2, reps = 64;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const double bytes = double(grid) * reps * 32768;
  for (int k = 0; k < 3; ++k) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (k == 0) red_scalar<<<grid, 128>>>(acc, reps, nrows);
      if (k == 1) red_v4<<<grid, 128>>>(acc, reps, nrows);
      if (k == 2) red_bulk<<<grid, 128>>>(acc, reps, nrows);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("%s: %.1f GB/s of fp32 reduction (%s)\n", k == 0 ? "red.f32 coalesced" : k == 1 ? "red.v4.f32" : "cp.reduce.async.bulk",
                      bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
