// Throughput of ex2.approx (MUFU) vs FFMA on one SM: 1 CTA, W warps, 8 independent chains/thread.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ex2(float* out, int iters, long long* cyc) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_ffma(float* out, int iters, long long* cyc) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 4096 * 4); cudaMallocManaged(&cyc, 8);
  const int iters = 4096;
  for (int warps : {1, 2, 4, 8, 16}) {
    k_ex2<<<1, 32 * warps>>>(out, iters, cyc); cudaDeviceSynchronize();
    k_ex2<<<1, 32 * warps>>>(out, iters, cyc); cudaDeviceSynchronize();
    double ops = 8.0 * iters * 32 * warps;
    double e = ops / *cyc;
    k_ffma<<<1, 32 * warps>>>(out, iters, cyc); cudaDeviceSynchronize();
    double f = ops / *cyc;
    printf("warps=%2d ex2 lanes/clk/SM=%.2f  ffma lanes/clk/SM=%.2f\n", warps, e, f);
  }
  return 0;
}
