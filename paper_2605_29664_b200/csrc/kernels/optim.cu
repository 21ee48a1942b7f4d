// Fused per-window optimizer step and small device utilities.
//
// One HBM pass per parameter: read g (fp32 window-accumulated gradient), theta, m, v;
// write theta, m, v, the bf16 working copy, and zero g for the next window.
// Algorithmic traffic: 4+4+4+4 read + 4+4+4+2+4 write = 34 B/param.
// The AdamType branch restates ppsim::detail::apply_update (optim.hpp:256-266):
// no bias correction, no weight decay, clamped preconditioner, fp64 in the
// reference, fp32 here.
#include <cmath>

#include "common.cuh"

namespace amdp {
namespace {

struct OptK {
  int kind;
  float lr, b1, b2, eps, wd, cmin, cmax, gscale;
  float bc1, bc2;  // AdamW bias corrections 1/(1-b1^t), 1/(1-b2^t)
};

__device__ __forceinline__ void opt_elem(const OptK& o, float& th, float& m, float& v, float g) {
  g *= o.gscale;
  switch (o.kind) {
    case AMDP_OPT_SGD:
      th -= o.lr * g;
      break;
    case AMDP_OPT_MOMENTUM:
      m = o.b1 * m + (1.f - o.b1) * g;
      th -= o.lr * m;
      break;
    case AMDP_OPT_REF_ADAMTYPE: {
      m = o.b1 * m + (1.f - o.b1) * g;
      v = o.b2 * v + (1.f - o.b2) * g * g;
      float pre = 1.f / (sqrtf(v) + o.eps);
      pre = fminf(fmaxf(pre, o.cmin), o.cmax);
      th -= o.lr * pre * m;
      break;
    }
    default: {  // AdamW
      m = o.b1 * m + (1.f - o.b1) * g;
      v = o.b2 * v + (1.f - o.b2) * g * g;
      const float mh = m * o.bc1, vh = v * o.bc2;
      th -= o.lr * (mh / (sqrtf(vh) + o.eps) + o.wd * th);
      break;
    }
  }
}

// USE_M / USE_V: whether the rule keeps momentum / second moment.  Unused state is neither
// read nor written (its pointer may be null), so no buffer is ever aliased.
template <bool USE_M, bool USE_V>
__global__ void __launch_bounds__(256) opt_kernel(OptK o, float* __restrict__ theta,
                                                  float* __restrict__ m, float* __restrict__ v,
                                                  float* __restrict__ grad, bf16* __restrict__ w,
                                                  int64_t n) {
  grid_dep_wait();  // PDL: predecessor's outputs visible from here
  grid_dep_trigger();
  const int64_t n4 = n / 4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += stride) {
    float4 t = reinterpret_cast<float4*>(theta)[i];
    float4 mm = USE_M ? reinterpret_cast<float4*>(m)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 vv = USE_V ? reinterpret_cast<float4*>(v)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 g = reinterpret_cast<float4*>(grad)[i];
    opt_elem(o, t.x, mm.x, vv.x, g.x);
    opt_elem(o, t.y, mm.y, vv.y, g.y);
    opt_elem(o, t.z, mm.z, vv.z, g.z);
    opt_elem(o, t.w, mm.w, vv.w, g.w);
    reinterpret_cast<float4*>(theta)[i] = t;
    if (USE_M) reinterpret_cast<float4*>(m)[i] = mm;
    if (USE_V) reinterpret_cast<float4*>(v)[i] = vv;
    reinterpret_cast<float4*>(grad)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    __nv_bfloat162 lo = __floats2bfloat162_rn(t.x, t.y), hi = __floats2bfloat162_rn(t.z, t.w);
    uint2 packed;
    packed.x = *reinterpret_cast<uint32_t*>(&lo);
    packed.y = *reinterpret_cast<uint32_t*>(&hi);
    reinterpret_cast<uint2*>(w)[i] = packed;
  }
  // tail
  for (int64_t i = n4 * 4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    float t = theta[i], mm = USE_M ? m[i] : 0.f, vv = USE_V ? v[i] : 0.f;
    opt_elem(o, t, mm, vv, grad[i]);
    theta[i] = t;
    if (USE_M) m[i] = mm;
    if (USE_V) v[i] = vv;
    grad[i] = 0.f;
    w[i] = __float2bfloat16_rn(t);
  }
}

__global__ void sumsq_kernel(const float* __restrict__ x, int64_t n, float* out) {
  float s = 0.f;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    s += x[i] * x[i];
  s = warp_sum(s);
  __shared__ float part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) atomicAdd(out, t);
  }
}

// theta_i = stddev * N(0,1) from Box-Muller over two splitmix64 draws keyed by
// (seed, i); computed in fp64, rounded once to fp32 (master) and bf16 (copy).
__global__ void fill_normal_kernel(bf16* w, float* f32, int64_t n, uint64_t key, float stddev) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r1 = splitmix64(key + 2 * static_cast<uint64_t>(i));
    const uint64_t r2 = splitmix64(key + 2 * static_cast<uint64_t>(i) + 1);
    const double u1 = (static_cast<double>(r1 >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = static_cast<double>(r2 >> 11) * 0x1.0p-53;
    const double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    const float val = static_cast<float>(static_cast<double>(stddev) * z);
    if (f32) f32[i] = val;
    if (w) w[i] = __float2bfloat16_rn(val);
  }
}

__global__ void fill_const_kernel(float* x, int64_t n, float value) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[i] = value;
}

int grid_for(int64_t work, int per_sm) {
  int64_t b = (work + 255) / 256;
  const int64_t cap = static_cast<int64_t>(per_sm) * num_sms();
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return static_cast<int>(b);
}

}  // namespace
}  // namespace amdp

using namespace amdp;

extern "C" int amdp_optimizer_step(const amdp_opt_args* a, float* master, float* m, float* v,
                                   float* grad, uint16_t* weight_bf16, int64_t n,
                                   amdp_stream_t stream) {
  if (!a || n < 0 || !master || !grad || !weight_bf16) return AMDP_ERR_INVALID;
  if (a->kind < AMDP_OPT_SGD || a->kind > AMDP_OPT_ADAMW) return AMDP_ERR_INVALID;
  if (a->kind != AMDP_OPT_SGD && !m) return AMDP_ERR_INVALID;
  if ((a->kind == AMDP_OPT_REF_ADAMTYPE || a->kind == AMDP_OPT_ADAMW) && !v)
    return AMDP_ERR_INVALID;
  if (n == 0) return 0;
  if (a->kind == AMDP_OPT_SGD) m = nullptr;
  if (a->kind == AMDP_OPT_SGD || a->kind == AMDP_OPT_MOMENTUM) v = nullptr;
  if ((reinterpret_cast<uintptr_t>(master) | reinterpret_cast<uintptr_t>(grad) |
       reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) % 16 != 0 ||
      reinterpret_cast<uintptr_t>(weight_bf16) % 8 != 0)
    return AMDP_ERR_INVALID;
  OptK o;
  o.kind = a->kind;
  o.lr = a->lr;
  o.b1 = a->beta1;
  o.b2 = a->beta2;
  o.eps = a->eps;
  o.wd = a->weight_decay;
  o.cmin = a->clamp_min;
  o.cmax = a->clamp_max;
  o.gscale = a->grad_scale;
  const int step = a->step < 1 ? 1 : a->step;
  o.bc1 = static_cast<float>(1.0 / (1.0 - std::pow(static_cast<double>(a->beta1), step)));
  o.bc2 = static_cast<float>(1.0 / (1.0 - std::pow(static_cast<double>(a->beta2), step)));
  const dim3 grid(grid_for(n / 4 + 1, 8));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  bf16* w = reinterpret_cast<bf16*>(weight_bf16);
  if (a->kind == AMDP_OPT_SGD)
    launch_pdl(opt_kernel<false, false>, grid, dim3(256), 0, s, o, master, nullptr, nullptr, grad, w, n);
  else if (a->kind == AMDP_OPT_MOMENTUM)
    launch_pdl(opt_kernel<true, false>, grid, dim3(256), 0, s, o, master, m, nullptr, grad, w, n);
  else
    launch_pdl(opt_kernel<true, true>, grid, dim3(256), 0, s, o, master, m, v, grad, w, n);
  return cudaGetLastError();
}

extern "C" int amdp_sumsq(const float* x, int64_t n, float* out, amdp_stream_t stream) {
  if (n < 0 || !out) return AMDP_ERR_INVALID;
  if (n == 0) return 0;
  sumsq_kernel<<<grid_for(n, 4), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(x, n, out);
  return cudaGetLastError();
}

extern "C" int amdp_fill_normal_bf16_f32(uint16_t* w_bf16, float* w_f32, int64_t n,
                                         uint64_t seed, float stddev, amdp_stream_t stream) {
  if (n < 0) return AMDP_ERR_INVALID;
  if (n == 0) return 0;
  fill_normal_kernel<<<grid_for(n, 8), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<bf16*>(w_bf16), w_f32, n, splitmix64(seed), stddev);
  return cudaGetLastError();
}

extern "C" int amdp_fill_const_f32(float* x, int64_t n, float value, amdp_stream_t stream) {
  if (n < 0) return AMDP_ERR_INVALID;
  if (n == 0) return 0;
  fill_const_kernel<<<grid_for(n, 8), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(x, n,
                                                                                         value);
  return cudaGetLastError();
}

extern "C" const char* amdp_version(void) { return "amdp-b200 0.1 sm_100a"; }
