// The learner's loss block fused per trajectory: policy / value heads over
// the trajectory's T core rows and its bootstrap row, the target
// log-probability, V-trace (and GAE when the advantage source asks for it),
// the PPO / value / entropy loss with its gradient wrt logits and value, and
// the heads backward (dcore rows + this trajectory's partial head-weight
// gradients) -- one CTA per trajectory.  The trajectory's core rows and the
// head weights are bulk-copied into shared memory once and read from there by
// the heads and by the heads backward; everything between the stages stays in
// shared memory or registers.  Replaces heads_fwd -> returns32 -> ppo_loss ->
// heads_bwd_fused (four dependent launches) in the learner step; the
// per-trajectory head-gradient partials are summed in trajectory order by
// heads_grad_reduce_kernel (model_kernels.cu), so the result is deterministic.
//
// Reference: heads softmax_heads / log_prob_and_entropy (policy.hpp:232-281),
// vtrace (offpolicy.hpp:61-100), gae as n-step - V (offpolicy.hpp:104-114),
// the loss and its logits / value gradient (policy.hpp:323-375), learner use
// orchestrator.hpp:803-863.  Envelope: T <= 32 (lane t owns step t), A <= 7
// (A + 1 <= 8 lanes per sample), no batch-wide advantage normalisation (that
// needs the whole batch before the loss: the unfused path runs it).
#include "appo_common.cuh"
#include "model_kernels.cuh"
#include "returns.cuh"
#include "sm100.cuh"

namespace appo_b200 {
namespace {

// 16 warps: two or three core rows per warp in the heads, 8 lanes per sample
// in the loss (warps 0-7), a thread per head-gradient column in the backward
// (1024 threads cap registers at 64: the fp64 loss state then spills)
constexpr int kTlThreads = 512;
constexpr int kTlA1 = 8;  // A + 1 <= 8
// dynamic shared memory: core rows [33][512] fp32, head rows [8][512] fp32
// (policy rows, the value row at A, zero rows above), the copy barrier
constexpr int kTlRowsOff = 0;
constexpr int kTlWOff = 33 * kHidden * 4;
constexpr int kTlBarOff = kTlWOff + kTlA1 * kHidden * 4;
constexpr int kTlSmem = kTlBarOff + 16;

struct TrajLossArgs {
  int n_traj, T, A;
  int64_t B;
  const float* core;  // [B + n_traj][512]: steps s = i*T + t, bootstrap rows B + i
  const float* wpi;   // [A][512]
  const float* bpi;   // [A]
  const float* wv;    // [512]
  const float* bv;    // [1]
  const int32_t* act;
  const float* rew;
  const float* blogp;
  const uint8_t* done;
  const int64_t* ver;
  int64_t cur_version;
  float gamma, rho_bar, c_bar, lambda;
  LossHP hp;
  // outputs
  float* logits;  // [B + n_traj][A]
  float* values;  // [B + n_traj]
  float* vt;      // [B] V-trace targets
  float* pg;      // [B] V-trace policy-gradient advantages
  float* adv;     // [B] GAE advantages (GAE mode)
  float* dcore;   // [B][512]
  float* part;    // [n_traj][(A+1)*512 + A+1] head-gradient partials
  double* partials;
  unsigned* counter;
  double* stats;
  int* flags;
};

// packed fp32 pairs (fma.rn.f32x2: two FMAs per issue slot)
__device__ __forceinline__ uint64_t tl_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 tl_unpack(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ uint64_t tl_ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// the 8 dot products of one row (policy rows, value row at A) reduce-scattered
// over the warp: 9 shuffles; lanes 4k .. 4k+3 end with sum k
__device__ __forceinline__ float tl_reduce8(const float (&v)[kTlA1], int lane) {
  const bool u4 = lane & 16, u3 = lane & 8, u2 = lane & 4;
  float t4[4], t2[2];
#pragma unroll
  for (int m = 0; m < 4; ++m)
    t4[m] = (u4 ? v[m + 4] : v[m]) + __shfl_xor_sync(0xffffffffu, u4 ? v[m] : v[m + 4], 16);
#pragma unroll
  for (int m = 0; m < 2; ++m)
    t2[m] = (u3 ? t4[m + 2] : t4[m]) + __shfl_xor_sync(0xffffffffu, u3 ? t4[m] : t4[m + 2], 8);
  float t1 = (u2 ? t2[1] : t2[0]) + __shfl_xor_sync(0xffffffffu, u2 ? t2[0] : t2[1], 4);
  t1 += __shfl_xor_sync(0xffffffffu, t1, 2);
  t1 += __shfl_xor_sync(0xffffffffu, t1, 1);
  return t1;
}

template <bool GAE>
__global__ void __launch_bounds__(kTlThreads) traj_loss_kernel(TrajLossArgs a) {
  __shared__ float s_logit[33][kTlA1];
  __shared__ float s_val[33];
  __shared__ float s_tlogp[32];
  __shared__ float s_vt[32], s_adv[32];
  __shared__ __align__(16) float s_dl[32][kTlA1];  // dlogits, dV at A, zeros above
  __shared__ __align__(16) float s_sw[kTlA1][kHidden];  // rows 16..31's head-gradient sums
  __shared__ double s_red[8][6];
  __shared__ bool s_last;

  extern __shared__ __align__(16) uint8_t tl_smem[];
  float* s_rows = reinterpret_cast<float*>(tl_smem + kTlRowsOff);  // [33][512]
  float* s_w = reinterpret_cast<float*>(tl_smem + kTlWOff);        // [8][512]
  uint64_t* bar = reinterpret_cast<uint64_t*>(tl_smem + kTlBarOff);

  const int i = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = a.T, A = a.A, A1 = A + 1;
  const int64_t s0 = (int64_t)i * T;

  if (tid == 0) {
    sm100::mbar_init(bar, 1);
    sm100::fence_barrier_init();
  }
  APPO_PDL_ENTRY();
  if (tid == 0) {
    // the T step rows are contiguous; the bootstrap row and the policy rows follow
    const uint32_t rb = (uint32_t)T * kHidden * 4, hb = kHidden * 4;
    sm100::mbar_arrive_expect_tx(bar, rb + hb + (uint32_t)A * hb);
    sm100::bulk_load_1d(s_rows, a.core + s0 * kHidden, rb, bar);
    sm100::bulk_load_1d(s_rows + 32 * kHidden, a.core + (a.B + i) * kHidden, hb, bar);
    sm100::bulk_load_1d(s_w, a.wpi, (uint32_t)A * hb, bar);
  }
  // the value row (odd parameter offset: not 16-byte aligned) and zero rows
  for (int x = tid; x < (kTlA1 - A) * kHidden; x += kTlThreads)
    s_w[A * kHidden + x] = x < kHidden ? a.wv[x] : 0.0f;
  // per-sample scalars: the returns warps' inputs and the loss threads' (8
  // lanes per sample, threads 0..8T-1)
  float x_r = 0.0f, x_bl = 0.0f;
  uint8_t x_d = 1;
  if (warp < 2 && lane < T) {
    x_r = a.rew[s0 + lane];
    x_bl = a.blogp[s0 + lane];
    x_d = a.done[s0 + lane];
  }
  const int lt = tid >> 3, sub = tid & 7;  // loss mapping
  const bool lon = lt < T;
  int l_act = 0;
  float l_bl = 0.0f;
  int64_t l_ver = 0;
  if (lon) {
    l_act = a.act[s0 + lt];
    l_bl = a.blogp[s0 + lt];
    if (sub == 0) l_ver = a.ver[s0 + lt];
  }
  const float bv = a.bv[0];
  const float bp = (lane >> 2) < A ? a.bpi[(lane >> 2) & 7] : 0.0f;
  __syncthreads();  // value / zero rows; the barrier init
  sm100::mbar_wait(bar, 0);

  // ---- heads: a warp takes rows rr and rr + 16 together (each head row
  //      loaded once for both), packed FMAs; rows t < T are the steps, row
  //      32 of s_rows the bootstrap row (rr = T) ----
  for (int rr0 = warp; rr0 <= T; rr0 += 32) {
    const int rr1 = rr0 + 16;
    const bool two = rr1 <= T;
    const float4* h0p = reinterpret_cast<const float4*>(s_rows + (rr0 < T ? rr0 : 32) * kHidden);
    const float4* h1p = reinterpret_cast<const float4*>(s_rows + (rr1 < T ? rr1 : 32) * kHidden);
    uint64_t acc0[kTlA1], acc1[kTlA1];
#pragma unroll
    for (int k = 0; k < kTlA1; ++k) acc0[k] = acc1[k] = 0;
#pragma unroll 1
    for (int q = 0; q < kHidden / 128; ++q) {
      const int j4 = lane + 32 * q;
      const float4 h0 = h0p[j4];
      const float4 h1 = two ? h1p[j4] : make_float4(0.f, 0.f, 0.f, 0.f);
      const uint64_t h0a = tl_pack(h0.x, h0.y), h0b = tl_pack(h0.z, h0.w);
      const uint64_t h1a = tl_pack(h1.x, h1.y), h1b = tl_pack(h1.z, h1.w);
#pragma unroll
      for (int k = 0; k < kTlA1; ++k) {
        const float4 w = reinterpret_cast<const float4*>(s_w + k * kHidden)[j4];
        const uint64_t wa = tl_pack(w.x, w.y), wb = tl_pack(w.z, w.w);
        acc0[k] = tl_ffma2(wb, h0b, tl_ffma2(wa, h0a, acc0[k]));
        acc1[k] = tl_ffma2(wb, h1b, tl_ffma2(wa, h1a, acc1[k]));
      }
    }
    const int k = lane >> 2;
#pragma unroll 1
    for (int which = 0; which < (two ? 2 : 1); ++which) {
      float v[kTlA1];
#pragma unroll
      for (int m = 0; m < kTlA1; ++m) {
        const float2 f = tl_unpack(which ? acc1[m] : acc0[m]);
        v[m] = f.x + f.y;
      }
      const float t1 = tl_reduce8(v, lane);
      const int rr = which ? rr1 : rr0;
      const int64_t row = rr < T ? s0 + rr : a.B + i;
      if ((lane & 3) == 0) {
        if (k < A) {
          const float lgf = t1 + bp;
          s_logit[rr][k] = lgf;
          a.logits[row * A + k] = lgf;
        } else if (k == A) {
          const float val = t1 + bv;
          s_val[rr] = val;
          a.values[row] = val;
        }
      }
    }
  }
  __syncthreads();

  // ---- fp64 log-softmax per sample (lane group of 8; as ppo_loss_kernel):
  //      the target log-probability for V-trace, kept in registers for the loss
  double p = 0.0, lp = 0.0, H = 0.0, logp = 0.0;
  int ac = 0;
  const unsigned gm = 0xffu << (lane & ~7);
  if (lon) {
    if (sub == 0 && (l_act < 0 || l_act >= A)) atomicOr(a.flags + kFlagContract, 1);
    ac = min(max(l_act, 0), A - 1);
    const bool mine = sub < A;
    const double l = mine ? (double)s_logit[lt][sub] : -1e300;
    double mx = l;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(gm, mx, o, 8));
    const double ex = mine ? exp(l - mx) : 0.0;
    double z = ex;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) z += __shfl_xor_sync(gm, z, o, 8);
    const double lz = log(z);
    p = ex / z;
    lp = (l - mx) - lz;
    H = (mine && p > 0) ? -p * lp : 0.0;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) H += __shfl_xor_sync(gm, H, o, 8);
    const double lpa = __shfl_sync(gm, lp, ac, 8);
    logp = fmax(lpa, -690.7755278982137);  // log(1e-300) floor
    if (sub == 0) s_tlogp[lt] = (float)logp;
  }
  __syncthreads();

  // ---- returns: warp 0 V-trace, warp 1 GAE (the advantage source) ----
  if (warp == 0 || (GAE && warp == 1)) {
    ReturnsStepIn x;
    x.r = x_r;
    x.v = lane < T ? s_val[lane] : 0.0f;
    x.tl = lane < T ? s_tlogp[lane] : 0.0f;
    x.bl = x_bl;
    x.boot = s_val[T];
    x.d = x_d;
    if (warp == 0) {
      // validation (offpolicy.hpp:70-75): non-finite inputs -> NumericError
      const bool bad = __any_sync(0xffffffffu, (lane == 0 && !finitef(x.boot)) ||
                                                   (lane < T && (!finitef(x.r) || !finitef(x.v) ||
                                                                 !finitef(x.tl) || !finitef(x.bl))));
      if (bad && lane == 0) atomicOr(a.flags + kFlagNumeric, 1);
      const ReturnsStepOut y =
          returns_warp32<kVTrace>(x, lane, T, a.gamma, a.rho_bar, a.c_bar, 0.0f);
      if (lane < T) {
        s_vt[lane] = y.o0;
        a.vt[s0 + lane] = y.o0;
        a.pg[s0 + lane] = y.o1;
        if (!GAE) s_adv[lane] = y.o1;
      }
    } else {
      const ReturnsStepOut y = returns_warp32<kGAE>(x, lane, T, a.gamma, 1.0f, 1.0f, a.lambda);
      if (lane < T) {
        s_adv[lane] = y.o0;
        a.adv[s0 + lane] = y.o0;
      }
    }
  }
  __syncthreads();

  // ---- loss + gradient wrt logits / value (policy.hpp:323-375) ----
  if (warp < 8) {
    double acc[6] = {0, 0, 0, 0, 0, -1e300};
    if (lon) {
      double d = logp - (double)l_bl;
      d = fmin(fmax(d, -20.0), 20.0);
      const double ratio = exp(d);
      const double A_s = s_adv[lt];
      const double cl = fmin(fmax(ratio, (double)a.hp.clip_low), (double)a.hp.clip_high);
      const double sur = fmin(ratio * A_s, cl * A_s);
      const double dsur = (ratio * A_s <= cl * A_s) ? A_s : 0.0;  // ties -> unclipped
      const double invB = 1.0 / (double)a.B;
      const double dL_dlogp = -invB * dsur * ratio;
      const double verr = (double)s_val[lt] - (double)s_vt[lt];
      if (sub < A) {
        const double dlp = (sub == ac ? 1.0 : 0.0) - p;
        const double dH = p > 0 ? -p * (lp + H) : 0.0;
        s_dl[lt][sub] = (float)(dL_dlogp * dlp - a.hp.entropy_coef * invB * dH);
      } else if (sub == A) {
        s_dl[lt][A] = (float)(a.hp.value_coef * invB * 2.0 * verr);
      } else {
        s_dl[lt][sub] = 0.0f;
      }
      if (sub == 0) {
        const double lag = (double)(a.cur_version - l_ver);
        acc[0] = -sur;
        acc[1] = verr * verr;
        acc[2] = H;
        acc[3] = ratio;
        acc[4] = lag;
        acc[5] = lag;
      }
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) acc[k] = warp_sum(acc[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[5] = fmax(acc[5], __shfl_xor_sync(0xffffffffu, acc[5], o));
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < 6; ++k) s_red[warp][k] = acc[k];
  }
  __syncthreads();  // s_dl, s_red

  // per-trajectory stat partials; the last CTA reduces them in trajectory order
  if (tid == 0) {
    for (int k = 0; k < 6; ++k) {
      double t = k == 5 ? -1e300 : 0.0;
      for (int w = 0; w < 8; ++w) t = k == 5 ? fmax(t, s_red[w][k]) : t + s_red[w][k];
      a.partials[i * 6 + k] = t;
    }
    __threadfence();
    s_last = atomicAdd(a.counter, 1u) == gridDim.x - 1;
  }

  // ---- heads backward: dcore rows and the head-weight gradient partials;
  //      thread (half, jp) owns columns 2jp, 2jp + 1 of rows [16 half, 16 half
  //      + 16): packed FMAs, the halves' sums added through shared memory ----
  {
    const int jp = tid & 255, half = tid >> 8;
    const int c0 = 2 * jp;
    uint64_t w2[kTlA1], sw2[kTlA1];
#pragma unroll
    for (int k = 0; k < kTlA1; ++k) {
      w2[k] = *reinterpret_cast<const uint64_t*>(s_w + k * kHidden + c0);
      sw2[k] = 0;
    }
    const int t1 = min(T, 16 * half + 16);
#pragma unroll 2
    for (int t = 16 * half; t < t1; ++t) {
      const uint64_t cv = *reinterpret_cast<const uint64_t*>(s_rows + t * kHidden + c0);
      const float4 ga = *reinterpret_cast<const float4*>(&s_dl[t][0]);
      const float4 gb = *reinterpret_cast<const float4*>(&s_dl[t][4]);
      const float g[kTlA1] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
      uint64_t dc = 0;
#pragma unroll
      for (int k = 0; k < kTlA1; ++k) {
        const uint64_t g2 = tl_pack(g[k], g[k]);
        dc = tl_ffma2(g2, w2[k], dc);
        sw2[k] = tl_ffma2(g2, cv, sw2[k]);
      }
      *reinterpret_cast<uint64_t*>(a.dcore + (s0 + t) * kHidden + c0) = dc;
    }
    if (half == 1)
#pragma unroll
      for (int k = 0; k < kTlA1; ++k) *reinterpret_cast<uint64_t*>(&s_sw[k][c0]) = sw2[k];
    __syncthreads();  // also publishes s_last
    float* pb = a.part + (size_t)i * (A1 * kHidden + A1);
    if (half == 0) {
#pragma unroll
      for (int k = 0; k < kTlA1; ++k)
        if (k < A1) {
          const float2 x = tl_unpack(sw2[k]);
          const float2 y = *reinterpret_cast<const float2*>(&s_sw[k][c0]);
          pb[k * kHidden + c0] = x.x + y.x;  // per-trajectory stride is odd: no float2
          pb[k * kHidden + c0 + 1] = x.y + y.y;
        }
    } else if (jp < A1) {
      float sb = 0.0f;  // head bias gradients: column sums of dlogits / dV
      for (int t = 0; t < T; ++t) sb += s_dl[t][jp];
      pb[A1 * kHidden + jp] = sb;
    }
  }

  if (s_last && tid < 32) {
    // fixed order: lane b sums trajectories b, b + 32, ..; then a lane tree
    __threadfence();
    double t[6] = {0, 0, 0, 0, 0, -1e300};
    for (int b = lane; b < (int)gridDim.x; b += 32)
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const double x = __ldcg(a.partials + b * 6 + k);
        t[k] = k == 5 ? fmax(t[k], x) : t[k] + x;
      }
#pragma unroll
    for (int k = 0; k < 5; ++k) t[k] = warp_sum(t[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t[5] = fmax(t[5], __shfl_xor_sync(0xffffffffu, t[5], o));
    if (lane == 0) {
      const double invB = 1.0 / (double)a.B;
      double* st = a.stats;
      st[0] = t[0] * invB;
      st[1] = a.hp.value_coef * t[1] * invB;
      st[2] = t[2] * invB;
      st[3] = st[0] + st[1] - a.hp.entropy_coef * st[2];
      st[4] = t[3] * invB;
      st[6] = t[4] * invB;
      st[7] = t[5];
      if (!isfinite(st[3])) atomicOr(a.flags + kFlagNumeric, 1);
      *a.counter = 0;
    }
  }
}

}  // namespace

// module anchor for preload_library_kernels (slotq.cu)
const void* kanchor_traj_loss() { return reinterpret_cast<const void*>(&traj_loss_kernel<false>); }

bool traj_loss_supported(int n_traj, int T, int A, bool normalize_adv) {
  static const bool off = [] {
    const char* v = getenv("APPO_TRAJ_LOSS");
    return v && v[0] == '0';
  }();
  return !off && !normalize_adv && n_traj >= 1 && n_traj * 6 <= kRedSlots && n_traj <= 320 &&
         T >= 1 && T <= 32 && A >= 1 && A + 1 <= kTlA1;
}

int k_traj_loss(Ctx* c, int n_traj, int T, int A, const float* core, const float* wpi,
                const float* bpi, const float* wv, const float* bv, const int32_t* act,
                const float* rew, const float* blogp, const uint8_t* done, const int64_t* ver,
                int64_t cur_version, float gamma, float rho_bar, float c_bar, bool gae,
                float lambda, const LossHP& hp, float* logits, float* values, float* vt, float* pg,
                float* adv, float* dcore, float* part, double* stats, float* gwpi, float* gbpi,
                float* gwv, float* gbv, bool reduce_heads) {
  APPO_REQUIRE(traj_loss_supported(n_traj, T, A, false), APPO_ERR_CONTRACT,
               "traj_loss: outside the fused kernel's envelope");
  APPO_REQUIRE(((reinterpret_cast<uintptr_t>(core) | reinterpret_cast<uintptr_t>(wpi)) & 15) == 0,
               APPO_ERR_CONTRACT, "traj_loss: core / policy head must be 16-byte aligned");
  TrajLossArgs a;
  a.n_traj = n_traj;
  a.T = T;
  a.A = A;
  a.B = (int64_t)n_traj * T;
  a.core = core;
  a.wpi = wpi;
  a.bpi = bpi;
  a.wv = wv;
  a.bv = bv;
  a.act = act;
  a.rew = rew;
  a.blogp = blogp;
  a.done = done;
  a.ver = ver;
  a.cur_version = cur_version;
  a.gamma = gamma;
  a.rho_bar = rho_bar;
  a.c_bar = c_bar;
  a.lambda = lambda;
  a.hp = hp;
  a.logits = logits;
  a.values = values;
  a.vt = vt;
  a.pg = pg;
  a.adv = adv;
  a.dcore = dcore;
  a.part = part;
  a.partials = c->d_red;
  a.counter = c->d_counter + 2;
  a.stats = stats;
  a.flags = c->d_flags;
  const double B = (double)n_traj * T;
  // in: core rows (T + 1 per trajectory, staged once),
  // step scalars; out: logits, values, vt, pg, dcore, partials
  c->next_bytes = (B + n_traj) * kHidden * 4 + B * (4 + 4 + 4 + 1 + 8) +
                  (B + n_traj) * (A + 1) * 4 + B * 8 + B * kHidden * 4 +
                  (double)n_traj * (A + 1) * (kHidden + 1) * 4;
  c->next_name = "traj_loss_kernel";
  static int attr_bytes[64] = {};
  const int dev = c->device & 63;
  if (attr_bytes[dev] < kTlSmem) {
    APPO_CUDA_TRY(cudaFuncSetAttribute(traj_loss_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kTlSmem));
    APPO_CUDA_TRY(cudaFuncSetAttribute(traj_loss_kernel<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kTlSmem));
    attr_bytes[dev] = kTlSmem;
  }
  if (gae)
    APPO_LAUNCH(c, traj_loss_kernel<true>, n_traj, kTlThreads, kTlSmem, a);
  else
    APPO_LAUNCH(c, traj_loss_kernel<false>, n_traj, kTlThreads, kTlSmem, a);
  c->next_name = nullptr;
  if (!reduce_heads) return APPO_OK;  // the caller launches it (learner side stream)
  return k_heads_grad_reduce(c, A, n_traj, part, gwpi, gbpi, gwv, gbv);
}

}  // namespace appo_b200
