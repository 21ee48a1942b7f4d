// Shared device helpers for the memory-bound AMDP stage kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <utility>

#include "amdp_kernels.h"

namespace amdp {

using bf16 = __nv_bfloat16;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// 8 bf16 <-> 8 fp32 through one 16-byte vector.
__device__ __forceinline__ void load8(const bf16* p, float (&f)[8]) {
  uint4 q = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    float2 t = __bfloat1622float2(h[e]);
    f[2 * e] = t.x;
    f[2 * e + 1] = t.y;
  }
}
__device__ __forceinline__ void store8(bf16* p, const float (&f)[8]) {
  uint4 q;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
  for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
  *reinterpret_cast<uint4*>(p) = q;
}

// tanh-GELU of the bf16-rounded pre-activation, with every operation spelled out (no FMA
// contraction choices left to the compiler), shared by the fc1 GEMM epilogue and the
// recompute kernel so that the recomputed f = gelu(u) is bit-identical to the stored one.
// tanh on the SFU (tanh.approx.f32, max rel. error ~2^-11); the result is rounded to bf16.
__device__ __forceinline__ float gelu_tanh_bf16in(float acc) {
  const float x = __bfloat162float(__float2bfloat16_rn(acc));
  const float x3 = __fmul_rn(__fmul_rn(x, x), x);
  const float arg = __fmul_rn(0.7978845608028654f, __fmaf_rn(0.044715f, x3, x));
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(arg));
  return __fmul_rn(__fmul_rn(0.5f, x), __fadd_rn(1.f, t));
}

// splitmix64: the counter-based generator shared with the CPU oracle
// (oracle/gpt_oracle.py restates it bit-for-bit).
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Device side of programmatic dependent launch (see sm100_ptx.cuh for the tcgen05 kernels).
// 2^x on the FMA pipe for a pair (round-to-nearest split, degree-3 fit of 2^f on [-1/2, 1/2],
// rel. err 7.7e-5, far below the bf16 rounding of P): takes part of the exponentials off the
// 16/clk/SM MUFU unit (attention forward and backward softmax).
__device__ __forceinline__ float2 ex2_fma2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 t = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));
  // f = x - (t - M) = x + (M - t), both steps exact
  const float2 f = __fadd2_rn(x, __ffma2_rn(t, make_float2(-1.f, -1.f), make_float2(12582912.f, 12582912.f)));
  float2 p = __ffma2_rn(f, make_float2(0.05508868f, 0.05508868f), make_float2(0.24260405f, 0.24260405f));
  p = __ffma2_rn(p, f, make_float2(0.69327623f, 0.69327623f));
  p = __ffma2_rn(p, f, make_float2(0.99992895f, 0.99992895f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Launch with programmatic stream serialization (PDL): the kernel's launch and prologue
// overlap the previous kernel's tail; every kernel launched this way calls grid_dep_wait()
// before its first global-memory access.  AMDP_PDL=0 turns it off (plain serialization).
inline bool pdl_enabled() {
  static const int on = getenv("AMDP_PDL") ? atoi(getenv("AMDP_PDL")) : 1;
  return on != 0;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Per-device one-time flag (function attributes are per device): true the first time it is
// called for (key, current device).  key: a distinct static object per kernel instantiation.
inline bool first_on_device(std::atomic<uint64_t>& mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  const uint64_t bit = 1ull << dev;
  return (mask.fetch_or(bit) & bit) == 0;
}

// Sort of a minibatch's (token, position) keys for the deterministic token-table gradient
// (bf16 and fp32 paths): one CTA, bitonic in shared memory.  Key = token << 14 | position,
// so ntok <= 16384 and vocab < 2^18.
namespace {
constexpr int kEmbPosBits = 14;
__global__ void __launch_bounds__(1024) embedding_sort_kernel(const int32_t* __restrict__ tok, int ntok,
                                                              uint32_t* __restrict__ sorted) {
  extern __shared__ uint32_t keys[];
  grid_dep_wait();
  grid_dep_trigger();
  int n2 = 1;
  while (n2 < ntok) n2 <<= 1;
  for (int i = threadIdx.x; i < n2; i += blockDim.x)
    keys[i] = i < ntok ? (static_cast<uint32_t>(tok[i]) << kEmbPosBits) | static_cast<uint32_t>(i) : 0xffffffffu;
  __syncthreads();
  for (int size = 2; size <= n2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < n2 / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool up = (lo & size) == 0;
        const uint32_t a = keys[lo], b = keys[hi];
        if ((a > b) == up) {
          keys[lo] = b;
          keys[hi] = a;
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < ntok; i += blockDim.x) sorted[i] = keys[i];
}

}  // namespace

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace amdp
