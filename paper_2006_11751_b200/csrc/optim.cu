// Global-norm clip + Adam (optimizer_step, policy.hpp:431-455) over the flat
// fp32 parameter vector.  Two launches, no host round trip:
//   1. sum of squares (fp64 partials, deterministic last-block reduce) + finite
//      check -> d_norm_out[0] = ||g||, d_norm_out[1] = clip scale;
//   2. fused elementwise update reading the scale from device memory; writes
//      theta, m, v and (optionally) the bf16 inference copy the policy forward
//      reads (the "publish" of ParamStore, policy.hpp:487-494, without a copy).
// HBM-bound: 4 B grad + 3x(4 B read + 4 B write) + 2 B bf16 = 30 B / parameter.
#include <cuda_bf16.h>

#include "appo_common.cuh"

namespace appo_b200 {
namespace {

__global__ void __launch_bounds__(256)
    sumsq_kernel(int64_t n, const float* __restrict__ g, double* partials, unsigned* counter,
                 double* norm_out, float clip, int* flags, const int* peer_flags) {
  APPO_PDL_ENTRY();
  // data-parallel: adopt the other ranks' rejection flags (read by adam_kernel)
  if (peer_flags && blockIdx.x == 0 && threadIdx.x < kNumFlags && peer_flags[threadIdx.x])
    atomicOr(flags + threadIdx.x, peer_flags[threadIdx.x]);
  double acc = 0.0;
  bool bad = false;
  const int64_t n4 = (reinterpret_cast<uintptr_t>(g) & 15) ? 0 : (n >> 2);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {  // four loads in flight per thread
    float4 x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = __ldg(g4 + i + k * stride);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      bad |= !(finitef(x[k].x) && finitef(x[k].y) && finitef(x[k].z) && finitef(x[k].w));
      acc += (double)x[k].x * x[k].x + (double)x[k].y * x[k].y + (double)x[k].z * x[k].z +
             (double)x[k].w * x[k].w;
    }
  }
  for (; i < n4; i += stride) {
    const float4 x = __ldg(g4 + i);
    bad |= !(finitef(x.x) && finitef(x.y) && finitef(x.z) && finitef(x.w));
    acc += (double)x.x * x.x + (double)x.y * x.y + (double)x.z * x.z + (double)x.w * x.w;
  }
  for (int64_t i = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    bad |= !finitef(g[i]);
    acc += (double)g[i] * g[i];
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags + kFlagNumeric, 1);
  // block reduce
  __shared__ double sh[32];
  __shared__ bool last;
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
    partials[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {  // whole last block: strided partial sums, fixed-order tree (deterministic)
    __threadfence();
    double t = 0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x)
      t += ((volatile double*)partials)[b];
    t = warp_sum(t);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = t;
    __syncthreads();
  }
  // the step's accept/reject decision, frozen here for both Adam launches
  // (the rest of Adam may run on the learner side stream after the next
  // step's first kernels have raised flags of their own)
  if (last && threadIdx.x < kNumFlags)
    flags[kNumFlags + threadIdx.x] = ((volatile int*)flags)[threadIdx.x];
  if (last && threadIdx.x == 0) {
    double s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
    const double norm = sqrt(s);
    double scale = 1.0;
    if (clip > 0.0f && norm > (double)clip) scale = (double)clip / norm;
    norm_out[0] = norm;
    norm_out[1] = scale;
    *counter = 0;
  }
}

__global__ void __launch_bounds__(256)
    adam_kernel(int64_t n, float* __restrict__ theta, float* __restrict__ m,
                float* __restrict__ v, const float* __restrict__ g,
                const double* __restrict__ norm_in, float lr, float b1, float b2, float eps,
                float bc1, float bc2, __nv_bfloat16* __restrict__ bf16, float* __restrict__ f32,
                const int* flags, unsigned* applied) {
  APPO_PDL_ENTRY();
  if (flags[kFlagNumeric] | flags[kFlagContract] | flags[kFlagQueue]) {
    // the step threw before Adam: parameters untouched, but the publish target
    // still receives the current parameters so the published copy stays valid
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
      const float th = theta[i];
      if (bf16) bf16[i] = __float2bfloat16_rn(th);
      if (f32) f32[i] = th;
    }
    return;
  }
  if (applied && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(applied, 1u);
  const float scale = (float)norm_in[1];
  auto upd = [&](float th, float& mi, float& vi, float gr) {
    const float gi = gr * scale;
    mi = b1 * mi + (1.0f - b1) * gi;
    vi = b2 * vi + (1.0f - b2) * gi * gi;
    return th - lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
  };
  // float4 body (16-byte aligned vectors, 8-byte aligned bf16 copy), scalar tail
  const bool vec = ((reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(theta) |
                     reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v) |
                     reinterpret_cast<uintptr_t>(f32)) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(bf16) & 7) == 0;
  const int64_t n4 = vec ? (n >> 2) : 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 gg = reinterpret_cast<const float4*>(g)[i];
    float4 th = reinterpret_cast<float4*>(theta)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    th.x = upd(th.x, mm.x, vv.x, gg.x);
    th.y = upd(th.y, mm.y, vv.y, gg.y);
    th.z = upd(th.z, mm.z, vv.z, gg.z);
    th.w = upd(th.w, mm.w, vv.w, gg.w);
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    reinterpret_cast<float4*>(theta)[i] = th;
    if (bf16) {
      const __nv_bfloat162 lo = __floats2bfloat162_rn(th.x, th.y);
      const __nv_bfloat162 hi = __floats2bfloat162_rn(th.z, th.w);
      uint2 pk;
      pk.x = *reinterpret_cast<const uint32_t*>(&lo);
      pk.y = *reinterpret_cast<const uint32_t*>(&hi);
      reinterpret_cast<uint2*>(bf16)[i] = pk;
    }
    if (f32) reinterpret_cast<float4*>(f32)[i] = th;
  }
  for (int64_t i = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float mi = m[i], vi = v[i];
    const float th = upd(theta[i], mi, vi, g[i]);
    m[i] = mi;
    v[i] = vi;
    theta[i] = th;
    if (bf16) bf16[i] = __float2bfloat16_rn(th);
    if (f32) f32[i] = th;
  }
}

}  // namespace

// module anchor for preload_library_kernels (slotq.cu)
const void* kanchor_optim() { return reinterpret_cast<const void*>(&sumsq_kernel); }

static int adam_range(Ctx* c, int64_t n, float* theta, float* m, float* v, const float* g,
                      int64_t t, float lr, float b1, float b2, float eps, double* d_norm_out,
                      uint16_t* bf16_copy, float* f32_copy, unsigned* applied) {
  if (n <= 0) return APPO_OK;
  const float bc1 = (float)(1.0 - pow((double)b1, (double)t));
  const float bc2 = (float)(1.0 - pow((double)b2, (double)t));
  const int64_t nv = (n + 3) / 4;  // float4 groups (the kernel falls back to scalars if unaligned)
  const int grid2 = (int)((nv + 255) / 256 < 148 * 16 ? (nv + 255) / 256 : 148 * 16);
  c->next_bytes = (double)n * (4 + 24 + (bf16_copy ? 2 : 0) + (f32_copy ? 4 : 0));
  APPO_LAUNCH(c, adam_kernel, grid2, 256, 0, n, theta, m, v, g, d_norm_out, lr, b1, b2, eps, bc1,
              bc2, reinterpret_cast<__nv_bfloat16*>(bf16_copy), f32_copy, c->d_flags + kNumFlags,
              applied);
  return APPO_OK;
}

int launch_adam_rest(Ctx* c, int64_t n, int64_t lo, float* theta, float* m, float* v,
                     const float* g, int64_t t, float lr, float b1, float b2, float eps,
                     double* d_norm_out, uint16_t* bf16_copy, float* f32_copy) {
  return adam_range(c, n - lo, theta + lo, m + lo, v + lo, g + lo, t, lr, b1, b2, eps, d_norm_out,
                    bf16_copy ? bf16_copy + lo : nullptr, f32_copy ? f32_copy + lo : nullptr,
                    nullptr);
}

int launch_adam(Ctx* c, int64_t n, float* theta, float* m, float* v, const float* g, int64_t t,
                float lr, float b1, float b2, float eps, float clip, double* d_norm_out,
                uint16_t* bf16_copy, float* f32_copy, unsigned* applied, const int* peer_flags,
                int64_t n_head) {
  if (n == 0) return APPO_OK;
  const int grid = 148 * 4;  // partials fit kRedSlots; enough loads in flight for HBM
  c->next_bytes = (double)n * 4;
  APPO_LAUNCH(c, sumsq_kernel, grid, 256, 0, n, g, c->d_red, c->d_counter + 1, d_norm_out, clip,
              c->d_flags, peer_flags);
  return adam_range(c, n_head >= 0 && n_head < n ? n_head : n, theta, m, v, g, t, lr, b1, b2, eps,
                    d_norm_out, bf16_copy, f32_copy, applied);
}

}  // namespace appo_b200
