// Off-policy returns, loss reduction and categorical-head kernels.
//
// V-trace / n-step / GAE are the same backward linear recurrence
//   a_t = delta_t + k_t * a_{t+1},   a_T = terminal
// (offpolicy.hpp:83-98 for V-trace with a = v - V, k = disc*c;
//  offpolicy.hpp:107-113 for n-step with a = ret, k = disc, terminal = boot;
//  GAE with k = disc*lambda).  One warp owns one trajectory: each lane composes
// the affine maps of its ceil(T/32) consecutive steps, a 5-step shuffle scan
// composes the lanes right-to-left, and a second pass over the lane's chunk
// writes the outputs.  HBM-bound: V-trace moves 17 B in + 8 B out per element
// (16 B more with rho/c outputs).
#include "appo_common.cuh"
#include "returns.cuh"

namespace appo_b200 {

namespace {

struct ReturnsArgs {
  int n_traj, T;
  const float* r;
  const float* v;
  const float* boot;
  const float* tl;
  const float* bl;
  const uint8_t* d;
  float gamma, rho_bar, c_bar, lambda;
  float* out0;  // vtrace: v_s      nstep: ret   gae: adv
  float* out1;  // vtrace: pg_adv   gae: ret (optional)
  float* out2;  // vtrace: rho (optional)
  float* out3;  // vtrace: c (optional)
  int* flags;
};

template <int MODE>
__device__ __forceinline__ void step_coeffs(const ReturnsArgs& a, const float* r, const float* v,
                                            const float* tl, const float* bl, const uint8_t* d,
                                            float boot, int t, int T, float& k, float& delta,
                                            float& rho, float& c, float& disc) {
  disc = d[t] ? 0.0f : a.gamma;
  if (MODE == kVTrace) {
    float lr = tl[t] - bl[t];
    lr = fminf(fmaxf(lr, -20.0f), 20.0f);  // importance_ratio clamp, offpolicy.hpp:50-54
    const float ratio = expf(lr);
    rho = fminf(a.rho_bar, ratio);
    c = fminf(a.c_bar, ratio);
    const float vnext = (t + 1 < T) ? v[t + 1] : boot;
    delta = rho * (r[t] + disc * vnext - v[t]);
    k = disc * c;
  } else if (MODE == kNStep) {
    delta = r[t];
    k = disc;
  } else {
    const float vnext = (t + 1 < T) ? v[t + 1] : boot;
    delta = r[t] + disc * vnext - v[t];
    k = disc * a.lambda;
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) returns_kernel(ReturnsArgs a) {
  APPO_PDL_ENTRY();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= a.n_traj) return;
  const int T = a.T;
  const size_t base = (size_t)warp * T;
  const float* r = a.r + base;
  const float* v = (MODE != kNStep) ? a.v + base : nullptr;
  const float* tl = (MODE == kVTrace) ? a.tl + base : nullptr;
  const float* bl = (MODE == kVTrace) ? a.bl + base : nullptr;
  const uint8_t* d = a.d + base;
  const float boot = a.boot[warp];

  const int per = (T + 31) >> 5;
  const int t0 = min(lane * per, T);
  const int t1 = min(t0 + per, T);

  // validation (offpolicy.hpp:70-75): non-finite inputs -> NumericError
  if (MODE == kVTrace) {
    bool bad = !finitef(boot);
    for (int t = t0; t < t1; ++t)
      bad |= !finitef(r[t]) || !finitef(v[t]) || !finitef(tl[t]) || !finitef(bl[t]);
    if (bad) atomicOr(a.flags + kFlagNumeric, 1);
  }

  // pass 1: compose this lane's chunk, map(x) = D + K x
  float K = 1.0f, D = 0.0f;
  for (int t = t1 - 1; t >= t0; --t) {
    float k, delta, rho, c, disc;
    step_coeffs<MODE>(a, r, v, tl, bl, d, boot, t, T, k, delta, rho, c, disc);
    D = delta + k * D;
    K = k * K;
  }
  // inclusive right-to-left scan over lanes: (Ki,Di) o (Kj,Dj) = (Ki Kj, Di + Ki Dj)
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const float Kn = __shfl_down_sync(0xffffffffu, K, off);
    const float Dn = __shfl_down_sync(0xffffffffu, D, off);
    if (lane + off < 32) {
      D = D + K * Dn;
      K = K * Kn;
    }
  }
  float Kx = __shfl_down_sync(0xffffffffu, K, 1);
  float Dx = __shfl_down_sync(0xffffffffu, D, 1);
  if (lane == 31) {
    Kx = 1.0f;
    Dx = 0.0f;
  }
  const float terminal = (MODE == kNStep) ? boot : 0.0f;
  float a_next = Dx + Kx * terminal;  // a at step t1

  // pass 2: outputs for this chunk
  for (int t = t1 - 1; t >= t0; --t) {
    float k, delta, rho, c, disc;
    step_coeffs<MODE>(a, r, v, tl, bl, d, boot, t, T, k, delta, rho, c, disc);
    const float at = delta + k * a_next;
    if (MODE == kVTrace) {
      const float vnext_corr = (t + 1 < T) ? (v[t + 1] + a_next) : boot;  // v_{t+1}
      a.out0[base + t] = v[t] + at;
      a.out1[base + t] = rho * (r[t] + disc * vnext_corr - v[t]);
      if (a.out2) a.out2[base + t] = rho;
      if (a.out3) a.out3[base + t] = c;
    } else if (MODE == kNStep) {
      a.out0[base + t] = at;
    } else {
      a.out0[base + t] = at;
      if (a.out1) a.out1[base + t] = at + v[t];
    }
    a_next = at;
  }
}

// T <= 32 (the configs' T = 32): lane t owns step t, every input of a
// trajectory is loaded once into registers (V_{t+1} by shuffle), so a
// trajectory costs one memory round trip.  Warps are persistent and take
// kRetU consecutive trajectories per pass, all loaded before any is scanned
// (kRetU round trips in flight per warp: at 65,536 x 32 two loads per warp
// left the kernel latency-bound at 0.37 of HBM).
constexpr int kRetU = 4;
template <int MODE>
__global__ void __launch_bounds__(256, 4) returns32_kernel(ReturnsArgs a) {
  APPO_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int T = a.T;
  const bool on = lane < T;
  for (int i0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kRetU; i0 < a.n_traj;
       i0 += nw * kRetU) {
    ReturnsStepIn x[kRetU];
#pragma unroll
    for (int u = 0; u < kRetU; ++u) {
      const int i = i0 + u;
      const bool ok = on && i < a.n_traj;
      const size_t o = (size_t)i * T + lane;
      x[u].r = ok ? __ldcs(a.r + o) : 0.0f;
      x[u].v = (MODE != kNStep && ok) ? __ldcs(a.v + o) : 0.0f;
      x[u].tl = (MODE == kVTrace && ok) ? __ldcs(a.tl + o) : 0.0f;
      x[u].bl = (MODE == kVTrace && ok) ? __ldcs(a.bl + o) : 0.0f;
      x[u].d = ok ? a.d[o] : 1;
      x[u].boot = i < a.n_traj ? __ldg(a.boot + i) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < kRetU; ++u) {
      const int i = i0 + u;
      if (i >= a.n_traj) break;  // warp-uniform
      // validation (offpolicy.hpp:70-75): non-finite inputs -> NumericError
      if (MODE == kVTrace) {
        const bool bad =
            __any_sync(0xffffffffu, (lane == 0 && !finitef(x[u].boot)) ||
                                        (on && (!finitef(x[u].r) || !finitef(x[u].v) ||
                                                !finitef(x[u].tl) || !finitef(x[u].bl))));
        if (bad && lane == 0) atomicOr(a.flags + kFlagNumeric, 1);
      }
      const ReturnsStepOut y =
          returns_warp32<MODE>(x[u], lane, T, a.gamma, a.rho_bar, a.c_bar, a.lambda);
      if (on) {
        const size_t o = (size_t)i * T + lane;
        __stcs(a.out0 + o, y.o0);
        if (MODE == kVTrace) {
          __stcs(a.out1 + o, y.o1);
          if (a.out2) __stcs(a.out2 + o, y.rho);
          if (a.out3) __stcs(a.out3 + o, y.c);
        } else if (MODE == kGAE) {
          if (a.out1) __stcs(a.out1 + o, y.o1);
        }
      }
    }
  }
}

// T == 32, 16-byte aligned rows: 8 lanes per trajectory, lane c owns steps
// 4c .. 4c+3 as float4 (one 16-byte load per input and store per output), so a
// warp takes 4 trajectories per pass.  Each lane composes its 4 affine maps
// locally, a 3-step shuffle scan over the 8-lane group composes the chunks
// right to left, and a second pass over the 4 steps writes the outputs.  The
// lane-per-step form above spends ~180 warp instructions per trajectory and
// was issue-bound at 0.38 of HBM on 65,536 x 32.
template <int MODE>
__global__ void __launch_bounds__(256, 4) returns32v_kernel(ReturnsArgs a) {
  APPO_PDL_ENTRY();
  const int lane = threadIdx.x & 31, c = lane & 7;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 4; i0 < a.n_traj; i0 += nw * 4) {
    const int i = i0 + (lane >> 3);
    const bool ok = i < a.n_traj;  // uniform over the 8-lane group
    const size_t o4 = (size_t)i * 8 + c;  // float4 index of steps 4c.. of trajectory i
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f), v = r, tl = r, bl = r;
    uint32_t dd = 0x01010101u;
    float boot = 0.0f;
    if (ok) {
      r = __ldcs(reinterpret_cast<const float4*>(a.r) + o4);
      if (MODE != kNStep) v = __ldcs(reinterpret_cast<const float4*>(a.v) + o4);
      if (MODE == kVTrace) {
        tl = __ldcs(reinterpret_cast<const float4*>(a.tl) + o4);
        bl = __ldcs(reinterpret_cast<const float4*>(a.bl) + o4);
      }
      dd = __ldcs(reinterpret_cast<const unsigned int*>(a.d) + o4);
      boot = __ldg(a.boot + i);
    }
    if (MODE == kVTrace) {  // validation (offpolicy.hpp:70-75): non-finite -> NumericError
      const bool bad = ok && (!finitef(boot) || !finitef(r.x) || !finitef(r.y) || !finitef(r.z) ||
                              !finitef(r.w) || !finitef(v.x) || !finitef(v.y) || !finitef(v.z) ||
                              !finitef(v.w) || !finitef(tl.x) || !finitef(tl.y) ||
                              !finitef(tl.z) || !finitef(tl.w) || !finitef(bl.x) ||
                              !finitef(bl.y) || !finitef(bl.z) || !finitef(bl.w));
      if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.flags + kFlagNumeric, 1);
    }
    const float rv[4] = {r.x, r.y, r.z, r.w}, vv[4] = {v.x, v.y, v.z, v.w};
    const float tv[4] = {tl.x, tl.y, tl.z, tl.w}, bv[4] = {bl.x, bl.y, bl.z, bl.w};
    // V_{t+1}: the next chunk's first value, the bootstrap after the last step
    float vn3 = __shfl_down_sync(0xffffffffu, v.x, 1);
    if (c == 7) vn3 = boot;
    const float vnext[4] = {vv[1], vv[2], vv[3], vn3};
    float k[4], delta[4], rho[4], cc[4], disc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      disc[q] = ((dd >> (8 * q)) & 0xffu) ? 0.0f : a.gamma;
      if (MODE == kVTrace) {
        const float lr = fminf(fmaxf(tv[q] - bv[q], -20.0f), 20.0f);  // offpolicy.hpp:50-54
        const float ratio = expf(lr);
        rho[q] = fminf(a.rho_bar, ratio);
        cc[q] = fminf(a.c_bar, ratio);
        delta[q] = rho[q] * (rv[q] + disc[q] * vnext[q] - vv[q]);
        k[q] = disc[q] * cc[q];
      } else if (MODE == kNStep) {
        delta[q] = rv[q];
        k[q] = disc[q];
      } else {
        delta[q] = rv[q] + disc[q] * vnext[q] - vv[q];
        k[q] = disc[q] * a.lambda;
      }
    }
    // this chunk's map (K, D): a_{4c} = D + K a_{4c+4}
    float K = k[3], D = delta[3];
#pragma unroll
    for (int q = 2; q >= 0; --q) {
      D = delta[q] + k[q] * D;
      K = k[q] * K;
    }
    // inclusive right-to-left scan over the 8 chunks of the trajectory
#pragma unroll
    for (int off = 1; off < 8; off <<= 1) {
      const float Kn = __shfl_down_sync(0xffffffffu, K, off, 8);
      const float Dn = __shfl_down_sync(0xffffffffu, D, off, 8);
      if (c + off < 8) {
        D = D + K * Dn;
        K = K * Kn;
      }
    }
    float Kx = __shfl_down_sync(0xffffffffu, K, 1, 8);
    float Dx = __shfl_down_sync(0xffffffffu, D, 1, 8);
    if (c == 7) {
      Kx = 1.0f;
      Dx = 0.0f;
    }
    const float terminal = (MODE == kNStep) ? boot : 0.0f;
    float an = Dx + Kx * terminal;  // a_{4c+4}
    // V-trace: v_s of the step after the chunk's last (V + a there; the
    // bootstrap after the trajectory's last step)
    float vs_next = (c == 7) ? boot : (vn3 + an);
    float o0[4], o1[4];
#pragma unroll
    for (int q = 3; q >= 0; --q) {
      const float at = delta[q] + k[q] * an;
      if (MODE == kVTrace) {
        o0[q] = vv[q] + at;
        o1[q] = rho[q] * (rv[q] + disc[q] * vs_next - vv[q]);
        vs_next = o0[q];
      } else if (MODE == kNStep) {
        o0[q] = at;
      } else {
        o0[q] = at;
        o1[q] = at + vv[q];
      }
      an = at;
    }
    if (ok) {
      __stcs(reinterpret_cast<float4*>(a.out0) + o4, make_float4(o0[0], o0[1], o0[2], o0[3]));
      if (MODE == kVTrace) {
        __stcs(reinterpret_cast<float4*>(a.out1) + o4, make_float4(o1[0], o1[1], o1[2], o1[3]));
        if (a.out2)
          __stcs(reinterpret_cast<float4*>(a.out2) + o4, make_float4(rho[0], rho[1], rho[2], rho[3]));
        if (a.out3)
          __stcs(reinterpret_cast<float4*>(a.out3) + o4, make_float4(cc[0], cc[1], cc[2], cc[3]));
      } else if (MODE == kGAE) {
        if (a.out1)
          __stcs(reinterpret_cast<float4*>(a.out1) + o4, make_float4(o1[0], o1[1], o1[2], o1[3]));
      }
    }
  }
}

template <int MODE>
int launch_returns(Ctx* c, const ReturnsArgs& a) {
  if (a.n_traj == 0 || a.T == 0) return APPO_OK;
  const int warps_per_block = 8;
  const int grid = (a.n_traj + warps_per_block - 1) / warps_per_block;
  const double n = (double)a.n_traj * a.T;
  c->next_bytes = MODE == kVTrace ? n * (17 + 8 + (a.out2 ? 4 : 0) + (a.out3 ? 4 : 0)) + a.n_traj * 4.0
                  : MODE == kNStep ? n * 9 + a.n_traj * 4.0
                                   : n * (13 + (a.out1 ? 8 : 4)) + a.n_traj * 4.0;
  const auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (a.T == 32 && a16(a.r) && (MODE == kNStep || a16(a.v)) &&
      (MODE != kVTrace || (a16(a.tl) && a16(a.bl) && a16(a.out1) && a16(a.out2) &&
                           a16(a.out3))) &&
      (MODE != kGAE || a16(a.out1)) && a16(a.out0) &&
      (reinterpret_cast<uintptr_t>(a.d) & 3) == 0) {
    // chunked float4 form: 4 trajectories per warp pass, persistent
    const int gv = (a.n_traj + 31) / 32;
    const int grid_v = gv < c->num_sms * 4 ? gv : c->num_sms * 4;  // 4 resident per SM
    APPO_LAUNCH(c, returns32v_kernel<MODE>, grid_v, warps_per_block * 32, 0, a);
    return APPO_OK;
  }
  if (a.T <= 32) {
    // persistent, kRetU trajectories per warp pass: 4 resident blocks of 8
    // warps per SM (__launch_bounds__(256, 4): <= 64 registers)
    const int gu = (a.n_traj + warps_per_block * kRetU - 1) / (warps_per_block * kRetU);
    const int g32 = gu < c->num_sms * 4 ? gu : c->num_sms * 4;
    APPO_LAUNCH(c, returns32_kernel<MODE>, g32, warps_per_block * 32, 0, a);
    return APPO_OK;
  }
  APPO_LAUNCH(c, returns_kernel<MODE>, grid, warps_per_block * 32, 0, a);
  return APPO_OK;
}

// ---------------------------------------------------------------- reductions

// Block-reduce NV doubles; partials[blockIdx][NV]; the last block to finish
// reduces the partials in block order (deterministic) and calls fin(sums).
template <int NV>
__device__ __forceinline__ bool block_reduce_last(double (&acc)[NV], double* partials,
                                                  unsigned* counter, double (&total)[NV]) {
  __shared__ double sh[32][NV];
  __shared__ bool is_last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) acc[j] = warp_sum(acc[j]);
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) sh[wid][j] = acc[j];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double s = 0;
      for (int w = 0; w < nw; ++w) s += sh[w][j];
      partials[blockIdx.x * NV + j] = s;
    }
    __threadfence();
    const unsigned prev = atomicAdd(counter, 1u);
    is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return false;
  __threadfence();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double s = 0;
      for (unsigned b = 0; b < gridDim.x; ++b) s += ((volatile double*)partials)[b * NV + j];
      total[j] = s;
    }
    *counter = 0;  // re-arm for the next launch on this stream
  }
  return threadIdx.x == 0;
}

// total_loss (offpolicy.hpp:146-168): out = {policy, value, entropy, total}
__global__ void __launch_bounds__(256)
    total_loss_kernel(int n, const float* __restrict__ ratios, const float* __restrict__ adv,
                      const float* __restrict__ values, const float* __restrict__ vt,
                      const float* __restrict__ ent, float lo, float hi, float vc, float ec,
                      double* partials, unsigned* counter, double* out, int* flags) {
  APPO_PDL_ENTRY();
  double acc[3] = {0, 0, 0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double r = ratios[i], A = adv[i];
    const double cl = fmin(fmax(r, (double)lo), (double)hi);
    acc[0] -= fmin(r * A, cl * A);
    const double ve = (double)values[i] - (double)vt[i];
    acc[1] += ve * ve;
    acc[2] += ent[i];
  }
  double tot[3];
  if (block_reduce_last<3>(acc, partials, counter, tot)) {
    const double inv = n > 0 ? 1.0 / n : 0.0;
    out[0] = tot[0] * inv;
    out[1] = vc * tot[1] * inv;
    out[2] = tot[2] * inv;
    out[3] = out[0] + out[1] - ec * out[2];
    if (!isfinite(out[3])) atomicOr(flags + kFlagNumeric, 1);
  }
}

// Stable softmax statistics of one head's logits [n]: max and partition sum
// (softmax_heads, policy.hpp:210-228).
__device__ __forceinline__ void head_softmax(const float* lg, int n, double& mx, double& z) {
  mx = lg[0];
  for (int i = 1; i < n; ++i) mx = fmax(mx, (double)lg[i]);
  z = 0;
  for (int i = 0; i < n; ++i) z += exp((double)lg[i] - mx);
}

// log_prob_and_entropy (policy.hpp:262-281) over factored heads: joint logp of
// the stored action [B][n_heads] = sum of per-head log max(p, 1e-300); entropy =
// sum of per-head entropies.  Logits row = concatenated heads.
__global__ void logp_entropy_kernel(int B, HeadsSpec hs, const float* __restrict__ logits,
                                    const int32_t* __restrict__ actions, float* logp, float* ent,
                                    int* flags) {
  APPO_PDL_ENTRY();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int ld = hs.off[hs.n];
  double lp = 0, h = 0;
  for (int j = 0; j < hs.n; ++j) {
    const int n = hs.off[j + 1] - hs.off[j];
    const float* lg = logits + (size_t)b * ld + hs.off[j];
    const int act = actions[(size_t)b * hs.n + j];
    if (act < 0 || act >= n) {  // APPO_CHECK "action index out of range for head"
      atomicOr(flags + kFlagContract, 1);
      return;
    }
    double mx, z;
    head_softmax(lg, n, mx, z);
    for (int i = 0; i < n; ++i) {
      const double p = exp((double)lg[i] - mx) / z;
      if (p > 0) h -= p * log(p);
    }
    lp += log(fmax(exp((double)lg[act] - mx) / z, 1e-300));
  }
  logp[b] = (float)lp;
  ent[b] = (float)h;
}

// sample_action (policy.hpp:232-258): per head, inverse CDF with the first i
// where u < cum (fallback n-1); joint logp = sum of log max(p, 1e-300).  The
// uniform of (row b, head j) is counter-based: U(key, counter0 + b*n_heads + j).
__global__ void sample_kernel(int B, HeadsSpec hs, const float* __restrict__ logits, uint64_t key,
                              uint64_t counter0, int32_t* actions, float* logp) {
  APPO_PDL_ENTRY();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int ld = hs.off[hs.n];
  double lp = 0;
  for (int j = 0; j < hs.n; ++j) {
    const int n = hs.off[j + 1] - hs.off[j];
    const float* lg = logits + (size_t)b * ld + hs.off[j];
    double mx, z;
    head_softmax(lg, n, mx, z);
    const double u = uniform01(key, counter0 + (uint64_t)b * hs.n + j);
    double cum = 0;
    int chosen = n - 1;
    for (int i = 0; i < n; ++i) {
      cum += exp((double)lg[i] - mx) / z;
      if (u < cum) {
        chosen = i;
        break;
      }
    }
    actions[(size_t)b * hs.n + j] = chosen;
    lp += log(fmax(exp((double)lg[chosen] - mx) / z, 1e-300));
  }
  logp[b] = (float)lp;
}

}  // namespace

// module anchor for preload_library_kernels (slotq.cu)
const void* kanchor_offpolicy() { return reinterpret_cast<const void*>(&logp_entropy_kernel); }

int launch_vtrace(Ctx* c, int n_traj, int T, const float* r, const float* v, const float* boot,
                  const float* tl, const float* bl, const uint8_t* d, float gamma, float rho_bar,
                  float c_bar, float* v_out, float* pg_out, float* rho_out, float* c_out) {
  ReturnsArgs a{n_traj, T, r, v, boot, tl, bl, d, gamma, rho_bar, c_bar, 0.f,
                v_out, pg_out, rho_out, c_out, c->d_flags};
  return launch_returns<kVTrace>(c, a);
}
int launch_nstep(Ctx* c, int n_traj, int T, const float* r, const float* boot, const uint8_t* d,
                 float gamma, float* ret) {
  ReturnsArgs a{n_traj, T, r, nullptr, boot, nullptr, nullptr, d, gamma, 1.f, 1.f, 0.f,
                ret, nullptr, nullptr, nullptr, c->d_flags};
  return launch_returns<kNStep>(c, a);
}
int launch_gae(Ctx* c, int n_traj, int T, const float* r, const float* v, const float* boot,
               const uint8_t* d, float gamma, float lambda, float* adv, float* ret) {
  ReturnsArgs a{n_traj, T, r, v, boot, nullptr, nullptr, d, gamma, 1.f, 1.f, lambda,
                adv, ret, nullptr, nullptr, c->d_flags};
  return launch_returns<kGAE>(c, a);
}

int launch_total_loss(Ctx* c, int n, const float* ratios, const float* adv, const float* values,
                      const float* vt, const float* ent, float lo, float hi, float vc, float ec,
                      double* d_out4) {
  int grid = (n + 255) / 256;
  grid = grid < 1 ? 1 : (grid > 296 ? 296 : grid);
  APPO_LAUNCH(c, total_loss_kernel, grid, 256, 0, n, ratios, adv, values, vt, ent, lo, hi, vc,
              ec, c->d_red, c->d_counter, d_out4, c->d_flags);
  return APPO_OK;
}

int launch_logp_entropy(Ctx* c, int B, const HeadsSpec& hs, const float* logits,
                        const int32_t* actions, float* logp, float* ent) {
  if (B == 0) return APPO_OK;
  APPO_LAUNCH(c, logp_entropy_kernel, (B + 127) / 128, 128, 0, B, hs, logits, actions, logp, ent,
              c->d_flags);
  return APPO_OK;
}

int launch_sample(Ctx* c, int B, const HeadsSpec& hs, const float* logits, uint64_t key,
                  uint64_t counter0, int32_t* actions, float* logp) {
  if (B == 0) return APPO_OK;
  APPO_LAUNCH(c, sample_kernel, (B + 127) / 128, 128, 0, B, hs, logits, key, counter0, actions,
              logp);
  return APPO_OK;
}

}  // namespace appo_b200
