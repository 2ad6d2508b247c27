// One trajectory of V-trace / n-step / GAE per warp for T <= 32 (lane t owns
// step t).  The three are the same backward linear recurrence
//   a_t = delta_t + k_t * a_{t+1},   a_T = terminal
// (offpolicy.hpp:83-98 V-trace with a = v - V, k = disc*c; offpolicy.hpp:
// 107-113 n-step with a = ret, k = disc, terminal = boot; GAE with k =
// disc*lambda), solved by a 5-step right-to-left shuffle scan of the affine
// maps (K, D).  Shared by returns32_kernel (offpolicy.cu) and the fused
// per-trajectory loss kernel (traj_loss.cu) so both compute the same floats.
#pragma once
#include <stdint.h>

namespace appo_b200 {

enum ReturnsMode { kVTrace = 0, kNStep = 1, kGAE = 2 };

struct ReturnsStepIn {
  float r, v, tl, bl, boot;  // boot: the trajectory's bootstrap value (all lanes)
  uint8_t d;
};
struct ReturnsStepOut {
  float o0;  // vtrace: v_s      nstep: ret   gae: adv
  float o1;  // vtrace: pg_adv   gae: ret
  float rho, c;
};

// Whole warp; lanes >= T take part in the scan with the identity map.
template <int MODE>
__device__ __forceinline__ ReturnsStepOut returns_warp32(const ReturnsStepIn& x, int lane, int T,
                                                         float gamma, float rho_bar, float c_bar,
                                                         float lambda) {
  const bool on = lane < T;
  float vnext = __shfl_down_sync(0xffffffffu, x.v, 1);
  if (lane == T - 1) vnext = x.boot;
  const float disc = x.d ? 0.0f : gamma;
  float k = 1.0f, delta = 0.0f, rho = 0.0f, c = 0.0f;
  if (on) {
    if (MODE == kVTrace) {
      const float lr = fminf(fmaxf(x.tl - x.bl, -20.0f), 20.0f);  // offpolicy.hpp:50-54
      const float ratio = expf(lr);
      rho = fminf(rho_bar, ratio);
      c = fminf(c_bar, ratio);
      delta = rho * (x.r + disc * vnext - x.v);
      k = disc * c;
    } else if (MODE == kNStep) {
      delta = x.r;
      k = disc;
    } else {
      delta = x.r + disc * vnext - x.v;
      k = disc * lambda;
    }
  }
  // inclusive right-to-left scan of the affine maps (K, D): a_t = D + K a_T
  float K = k, D = delta;
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
  const float terminal = (MODE == kNStep) ? x.boot : 0.0f;
  const float a_next = Dx + Kx * terminal;  // a_{t+1}
  const float at = delta + k * a_next;
  ReturnsStepOut o;
  o.rho = rho;
  o.c = c;
  if (MODE == kVTrace) {
    const float vnext_corr = (lane + 1 < T) ? (vnext + a_next) : x.boot;  // v_{t+1}
    o.o0 = x.v + at;
    o.o1 = rho * (x.r + disc * vnext_corr - x.v);
  } else if (MODE == kNStep) {
    o.o0 = at;
    o.o1 = 0.0f;
  } else {
    o.o0 = at;
    o.o1 = at + x.v;
  }
  return o;
}

}  // namespace appo_b200
