// SIMT kernels around the tcgen05 GEMMs of the model: im2col (fallbacks),
// the GRU cell (inference: fused with heads + sampling; training: with saved
// gates and done-masked recurrence), heads forward/backward, the fused PPO
// loss, slot gathers, column sums for bias gradients.
//
// All of these are HBM/latency-bound elementwise or small-reduction kernels:
// coalesced along the innermost (channel / hidden) dimension, 16-byte vector
// accesses where the layout allows it.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "model_kernels.cuh"

namespace appo_b200 {
namespace {

__device__ __forceinline__ float bf2f(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }
__device__ __forceinline__ uint16_t f2bf(float f) {
  __nv_bfloat16 h = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t*>(&h);
}
__device__ __forceinline__ float sigmoidf_(float x) { return 1.0f / (1.0f + expf(-x)); }

__device__ __forceinline__ const uint8_t* obs_ptr(const ObsSrc& o, int64_t r) {
  if (!o.slot_ids) return o.base + r * o.img_stride;
  const int64_t B = (int64_t)o.n_traj * o.T;
  if (r < B) {
    const int64_t i = r / o.T, t = r % o.T;
    return o.base + (uint64_t)o.slot_ids[i] * o.slot_bytes + o.obs_off + t * o.obs_dim;
  }
  return o.base + (uint64_t)o.slot_ids[r - B] * o.slot_bytes + o.boot_off;
}

// conv1 im2col from u8 CHW images: col[r*P1 + y*W1 + x][(c*8 + kh)*8 + kw] = obs[c][4y+kh][4x+kw]
// (values kept as exact integers 0..255 in bf16; the 1/255 is folded into the
// GEMM epilogue scale).  One thread = one (row, c, kh): 8 bytes in, 16 B out.
__global__ void im2col_u8_kernel(ObsSrc src, int64_t R, int C, int H, int W, int H1, int W1,
                                 uint16_t* __restrict__ col) {
  APPO_PDL_ENTRY();
  const int64_t P1 = (int64_t)H1 * W1;
  const int64_t total = R * P1 * C * 8;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int ckh = (int)(g % (C * 8));
    const int64_t row = g / (C * 8);
    const int64_t r = row / P1;
    const int p = (int)(row % P1);
    const int y = p / W1, x = p % W1;
    const int c = ckh >> 3, kh = ckh & 7;
    const uint8_t* img = obs_ptr(src, r);
    const uint8_t* s = img + ((int64_t)c * H + (y * 4 + kh)) * W + x * 4;
    const uint32_t lo = *reinterpret_cast<const uint32_t*>(s);
    const uint32_t hi = *reinterpret_cast<const uint32_t*>(s + 4);
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t word = j < 2 ? lo : hi;
      const int sh = (j & 1) * 16;
      const float f0 = (float)((word >> sh) & 0xFF);
      const float f1 = (float)((word >> (sh + 8)) & 0xFF);
      w[j] = (uint32_t)f2bf(f0) | ((uint32_t)f2bf(f1) << 16);
    }
    *reinterpret_cast<uint4*>(col + row * (C * 64) + ckh * 8) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// NHWC im2col: col[r*Po + y*Wo + x][(kh*k + kw)*Cin + ci] = act[r][sy+kh][sx+kw][ci]
// One thread = 8 channels (16 B).
__global__ void im2col_nhwc_kernel(const uint16_t* __restrict__ act, int64_t R, int Hi, int Wi,
                                   int Cin, int k, int s, int Ho, int Wo,
                                   uint16_t* __restrict__ col) {
  APPO_PDL_ENTRY();
  const int cg = Cin / 8;
  const int64_t Po = (int64_t)Ho * Wo;
  const int64_t total = R * Po * k * k * cg;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(g % cg);
    int64_t rest = g / cg;
    const int kk = (int)(rest % (k * k));
    const int64_t row = rest / (k * k);
    const int64_t r = row / Po;
    const int p = (int)(row % Po);
    const int y = p / Wo, x = p % Wo, kh = kk / k, kw = kk % k;
    const uint4 v = *reinterpret_cast<const uint4*>(
        act + (((r * Hi) + (y * s + kh)) * Wi + (x * s + kw)) * Cin + c8 * 8);
    *reinterpret_cast<uint4*>(col + row * (int64_t)(k * k * Cin) + kk * Cin + c8 * 8) = v;
  }
}

// Operands derived from a published copy in ONE launch (after the Adam step
// that wrote it): blocks 0..nb-2 rearrange the conv3 / conv2 weights for the
// sub-pixel dgrad (k_publish_derived layout), the last block writes the conv1
// fp16 weights and offset-corrected bias.
__global__ void __launch_bounds__(256)
    publish_derived_kernel(const uint16_t* __restrict__ wb, const float* __restrict__ pf,
                           int64_t off_c1w, int64_t off_c1b, int K1, int64_t off_c2w,
                           int64_t off_c3w, uint16_t* __restrict__ c1h, float* __restrict__ c1b,
                           uint16_t* __restrict__ wt2, uint16_t* __restrict__ wt3) {
  APPO_PDL_ENTRY();
  constexpr int kC1Blocks = 4;  // conv1 operands: 8 output channels (a warp each) per block
  if (blockIdx.x >= gridDim.x - kC1Blocks) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cb = blockIdx.x - (gridDim.x - kC1Blocks);
    for (int co = cb * 8 + warp; co < 32 && warp < 8; co += 32) {
      float acc = 0.0f;
      for (int k = lane; k < K1; k += 32) {
        const __half h = __float2half_rn(pf[off_c1w + (size_t)co * K1 + k]);
        c1h[(size_t)co * K1 + k] = __half_as_ushort(h);
        acc += __half2float(h);
      }
      acc = warp_sum(acc);
      if (lane == 0) c1b[co] = pf[off_c1b + co] - (1024.0f / 255.0f) * acc;
    }
    return;
  }
  // wt3: Co=128, k=3, Ci=64 (4*64*512 elements); wt2: Co=64, k=4, Ci=32 (4*32*256)
  const int n3 = 4 * 64 * 512, n2 = 4 * 32 * 256;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n3 + n2;
       g += (gridDim.x - kC1Blocks) * blockDim.x) {
    const bool is3 = g < n3;
    const int e = is3 ? g : g - n3;
    const int Co = is3 ? 128 : 64, k = is3 ? 3 : 4, Ci = is3 ? 64 : 32;
    const int kmax = 4 * Co;
    const int kk = e % kmax, ci = (e / kmax) % Ci, cls = e / (kmax * Ci);
    const int tap = kk / Co, co = kk % Co;
    const int kh = (cls >> 1) + 2 * (tap >> 1), kw = (cls & 1) + 2 * (tap & 1);
    const uint16_t* w = wb + (is3 ? off_c3w : off_c2w);
    const uint16_t v = (kh < k && kw < k) ? w[(((size_t)co * k + kh) * k + kw) * Ci + ci] : (uint16_t)0;
    (is3 ? wt3 : wt2)[e] = v;
  }
}

// contiguous rows: 4 values per thread, no index division
__global__ void f32_to_bf16_vec_kernel(int64_t n4, const float4* __restrict__ src,
                                       uint2* __restrict__ dst) {
  APPO_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldg(src + i);
    dst[i] = make_uint2(((uint32_t)f2bf(v.y) << 16) | f2bf(v.x),
                        ((uint32_t)f2bf(v.w) << 16) | f2bf(v.z));
  }
}

__global__ void f32_to_bf16_kernel(int64_t n, const float* __restrict__ src, int64_t src_ld,
                                   uint16_t* __restrict__ dst, int64_t dst_ld, int cols) {
  APPO_PDL_ENTRY();
  const int64_t total = n * cols;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = g / cols;
    const int c = (int)(g % cols);
    dst[r * dst_ld + c] = f2bf(src[r * src_ld + c]);
  }
}

// GRU cell (PyTorch gate order r, z, n) + heads + sampling for inference.
// One warp per env; lane owns hidden units j = 4 lane + 128 q (float4 loads
// and stores of every operand row).
__global__ void __launch_bounds__(256)
    gru_infer_kernel(int B, int A, const float* __restrict__ gi, const float* __restrict__ gh,
                     const float* __restrict__ h_in, const float* __restrict__ wpi,
                     const float* __restrict__ bpi, const float* __restrict__ wv,
                     const float* __restrict__ bv, uint64_t key, uint64_t counter0,
                     float* __restrict__ h_out, int32_t* __restrict__ actions,
                     float* __restrict__ logp, float* __restrict__ values,
                     float* __restrict__ logits_out) {
  APPO_PDL_ENTRY();
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= B) return;
  const float4* gib = reinterpret_cast<const float4*>(gi + (int64_t)b * kGates);
  const float4* ghb = reinterpret_cast<const float4*>(gh + (int64_t)b * kGates);
  const float4* hib = reinterpret_cast<const float4*>(h_in + (int64_t)b * kHidden);
  float4* hob = reinterpret_cast<float4*>(h_out + (int64_t)b * kHidden);
  constexpr int H4 = kHidden / 4;
  float acc[kMaxActions + 1];
#pragma unroll
  for (int a = 0; a <= kMaxActions; ++a) acc[a] = 0.0f;
#pragma unroll
  for (int q = 0; q < kHidden / 128; ++q) {
    const int j4 = lane + 32 * q;  // float4 index: units 4 j4 .. 4 j4 + 3
    const float4 ir = __ldg(gib + j4), iz = __ldg(gib + H4 + j4), in_ = __ldg(gib + 2 * H4 + j4);
    const float4 hr = __ldg(ghb + j4), hz = __ldg(ghb + H4 + j4), hn = __ldg(ghb + 2 * H4 + j4);
    const float4 hp = __ldg(hib + j4);
    const float xr[4] = {ir.x + hr.x, ir.y + hr.y, ir.z + hr.z, ir.w + hr.w};
    const float xz[4] = {iz.x + hz.x, iz.y + hz.y, iz.z + hz.z, iz.w + hz.w};
    const float xi[4] = {in_.x, in_.y, in_.z, in_.w};
    const float xh[4] = {hn.x, hn.y, hn.z, hn.w};
    const float xp[4] = {hp.x, hp.y, hp.z, hp.w};
    float h[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float r = sigmoidf_(xr[k]);
      const float z = sigmoidf_(xz[k]);
      const float n = tanhf(xi[k] + r * xh[k]);
      h[k] = (1.0f - z) * n + z * xp[k];
    }
    hob[j4] = make_float4(h[0], h[1], h[2], h[3]);
#pragma unroll
    for (int a = 0; a < kMaxActions; ++a)
      if (a < A) {
        const float4 w = __ldg(reinterpret_cast<const float4*>(wpi + a * kHidden) + j4);
        acc[a] += w.x * h[0] + w.y * h[1] + w.z * h[2] + w.w * h[3];
      }
    // wv sits at an odd offset of the parameter vector: scalar loads
    acc[kMaxActions] += __ldg(wv + 4 * j4) * h[0] + __ldg(wv + 4 * j4 + 1) * h[1] +
                        __ldg(wv + 4 * j4 + 2) * h[2] + __ldg(wv + 4 * j4 + 3) * h[3];
  }
#pragma unroll
  for (int a = 0; a < kMaxActions; ++a)
    if (a < A) acc[a] = warp_sum(acc[a]);
  acc[kMaxActions] = warp_sum(acc[kMaxActions]);
  if (lane == 0) {
    double lg[kMaxActions];
    double mx = -1e300;
    for (int a = 0; a < A; ++a) {
      lg[a] = (double)(acc[a] + bpi[a]);
      mx = fmax(mx, lg[a]);
      if (logits_out) logits_out[(int64_t)b * A + a] = (float)lg[a];
    }
    values[b] = acc[kMaxActions] + bv[0];
    double z = 0;
    for (int a = 0; a < A; ++a) z += exp(lg[a] - mx);
    const double u = uniform01(key, counter0 + (uint64_t)b);
    double cum = 0;
    int chosen = A - 1;
    for (int a = 0; a < A; ++a) {
      cum += exp(lg[a] - mx) / z;
      if (u < cum) {
        chosen = a;
        break;
      }
    }
    actions[b] = chosen;
    logp[b] = (float)log(fmax(exp(lg[chosen] - mx) / z, 1e-300));
  }
}

// Stage h for GRU step t: hbf/hin rows <- hcur (fp32 -> bf16 + fp32 copy).
__global__ void stage_h_kernel(int n_traj, int T, int t, const float* __restrict__ hcur,
                               float* __restrict__ hin, uint16_t* __restrict__ hbf) {
  APPO_PDL_ENTRY();
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_traj * kHidden) return;
  const int i = g / kHidden, j = g % kHidden;
  const int64_t row = (t < T) ? (int64_t)i * T + t : (int64_t)n_traj * T + i;
  const float h = hcur[g];
  hin[row * kHidden + j] = h;
  hbf[row * kHidden + j] = f2bf(h);
}

// Training GRU cell at step t for all trajectories; saves gates for BPTT
// and advances hcur with the reset-after-done mask (orchestrator.hpp:402).
__global__ void gru_train_kernel(int n_traj, int T, int t, const float* __restrict__ gi,
                                 const float* __restrict__ gh, const uint8_t* __restrict__ done,
                                 float* __restrict__ hcur, float* __restrict__ core,
                                 uint16_t* __restrict__ core_bf, float* __restrict__ gates) {
  APPO_PDL_ENTRY();
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_traj * kHidden) return;
  const int i = g / kHidden, j = g % kHidden;
  const int64_t row = (t < T) ? (int64_t)i * T + t : (int64_t)n_traj * T + i;
  const float* gir = gi + row * kGates;
  const float* ghr = gh + (int64_t)i * kGates;
  const float r = sigmoidf_(gir[j] + ghr[j]);
  const float z = sigmoidf_(gir[kHidden + j] + ghr[kHidden + j]);
  const float ghn = ghr[2 * kHidden + j];
  const float n = tanhf(gir[2 * kHidden + j] + r * ghn);
  const float hprev = hcur[g];
  const float h = (1.0f - z) * n + z * hprev;
  core[row * kHidden + j] = h;
  core_bf[row * kHidden + j] = f2bf(h);
  float* gs = gates + row * 4 * kHidden;
  gs[j] = r;
  gs[kHidden + j] = z;
  gs[2 * kHidden + j] = n;
  gs[3 * kHidden + j] = ghn;
  if (t < T) hcur[g] = done[(int64_t)i * T + t] ? 0.0f : h;
}

// Heads forward, warp per row; rows < B also get the target log-probability of
// the stored action and the policy entropy (log_prob_and_entropy,
// policy.hpp:262-281, learner use orchestrator.hpp:803-814) in fp64.
// AMAX: compile-time bound on the action count (8 covers the Doom head's 6;
// the loops over actions are unrolled to it, predicated by the runtime A).
template <int AMAX>
__global__ void __launch_bounds__(256)
    heads_fwd_kernel(int64_t R, int A, const float* __restrict__ core,
                     const float* __restrict__ wpi, const float* __restrict__ bpi,
                     const float* __restrict__ wv, const float* __restrict__ bv,
                     float* __restrict__ logits, float* __restrict__ values, int64_t B,
                     const int32_t* __restrict__ act, float* __restrict__ tlogp,
                     float* __restrict__ ent, int* flags) {
  APPO_PDL_ENTRY();
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= R) return;
  float acc[AMAX + 1];
#pragma unroll
  for (int a = 0; a <= AMAX; ++a) acc[a] = 0.0f;
  // lane owns units 4 j4 .. 4 j4 + 3, j4 = lane + 32 q (float4 rows; wv sits at
  // an odd parameter offset: scalar loads)
  const float4* crow = reinterpret_cast<const float4*>(core + row * kHidden);
#pragma unroll
  for (int q = 0; q < kHidden / 128; ++q) {
    const int j4 = lane + 32 * q;
    const float4 h = __ldg(crow + j4);
#pragma unroll
    for (int a = 0; a < AMAX; ++a)
      if (a < A) {
        const float4 w = __ldg(reinterpret_cast<const float4*>(wpi + a * kHidden) + j4);
        acc[a] += w.x * h.x + w.y * h.y + w.z * h.z + w.w * h.w;
      }
    acc[AMAX] += __ldg(wv + 4 * j4) * h.x + __ldg(wv + 4 * j4 + 1) * h.y +
                        __ldg(wv + 4 * j4 + 2) * h.z + __ldg(wv + 4 * j4 + 3) * h.w;
  }
#pragma unroll
  for (int a = 0; a < AMAX; ++a)
    if (a < A) acc[a] = warp_sum(acc[a]);
  acc[AMAX] = warp_sum(acc[AMAX]);
  // lane a < A holds logit a (all lanes hold the sums after warp_sum)
  float my = 0.0f;
#pragma unroll
  for (int a = 0; a < AMAX; ++a)
    if (a == lane) my = acc[a];
  const float lgf = lane < A ? my + bpi[lane] : -INFINITY;
  if (lane < A) logits[row * A + lane] = lgf;
  if (lane == 0) values[row] = acc[AMAX] + bv[0];
  if (act && row < B) {
    const int ac = act[row];
    if (ac < 0 || ac >= A) {
      if (lane == 0) atomicOr(flags + kFlagContract, 1);
      return;
    }
    // log_prob_and_entropy in fp64, one action per lane
    double mx = lane < A ? (double)lgf : -1e300;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const double e = lane < A ? exp((double)lgf - mx) : 0.0;
    const double z = warp_sum(e);
    const double pr = e / z;
    const double hterm = (lane < A && pr > 0) ? -pr * log(pr) : 0.0;
    const double h = warp_sum(hterm);
    const double pa = __shfl_sync(0xffffffffu, pr, ac);
    if (lane == 0) {
      tlogp[row] = (float)log(fmax(pa, 1e-300));
      ent[row] = (float)h;
    }
  }
}

// Gather per-step scalars and h0 from trajectory slots (layout v2) in FIFO
// order: s = i*T + t (orchestrator.hpp:781-795).  One block per trajectory.
__global__ void gather_slots_kernel(int n_traj, int T, const uint8_t* __restrict__ region,
                                    uint64_t slot_bytes, const int32_t* __restrict__ slot_ids,
                                    SlotOffsets off, int32_t* __restrict__ act,
                                    float* __restrict__ rew, float* __restrict__ blogp,
                                    uint8_t* __restrict__ done, int64_t* __restrict__ ver,
                                    float* __restrict__ h0, int* flags) {
  APPO_PDL_ENTRY();
  const int i = blockIdx.x;
  if (i >= n_traj) return;
  const uint8_t* slot = region + (uint64_t)slot_ids[i] * slot_bytes;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const int64_t s = (int64_t)i * T + t;
    act[s] = reinterpret_cast<const int32_t*>(slot + off.actions)[t];
    const float rw = reinterpret_cast<const float*>(slot + off.rewards)[t];
    const float lp = reinterpret_cast<const float*>(slot + off.logp)[t];
    rew[s] = rw;
    blogp[s] = lp;
    done[s] = slot[off.dones + t];
    ver[s] = reinterpret_cast<const int64_t*>(slot + off.versions)[t];
    if (!finitef(rw) || !finitef(lp)) atomicOr(flags + kFlagNumeric, 1);
  }
  for (int j = threadIdx.x; j < kHidden; j += blockDim.x)
    h0[(int64_t)i * kHidden + j] = reinterpret_cast<const float*>(slot + off.hidden)[j];
}

// Advantage normalisation (orchestrator.hpp:838-845), one block.
__global__ void normalize_kernel(int n, float* __restrict__ adv) {
  APPO_PDL_ENTRY();
  __shared__ double sh[32];
  __shared__ double mean_s, sd_s;
  double s = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += adv[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    mean_s = t / n;
  }
  __syncthreads();
  const double mean = mean_s;
  double q = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) q += (adv[i] - mean) * (adv[i] - mean);
  q = warp_sum(q);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = q;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    sd_s = sqrt(t / n) + 1e-8;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) adv[i] = (float)((adv[i] - mean) / sd_s);
}

// Fused PPO / value / entropy loss and its gradient wrt logits and value
// (policy.hpp:323-375).  LPS lanes per sample (lane a owns action a, lane A the
// value gradient): the fp64 log-softmax / entropy run across the lane group
// instead of serially in one thread; partial sums (policy, value, entropy,
// ratio, lag) -> deterministic last-block reduce into stats[0..7].
template <int LPS>
__global__ void __launch_bounds__(256)
    ppo_loss_kernel(int B, int A, const float* __restrict__ logits,
                    const float* __restrict__ values, const int32_t* __restrict__ act,
                    const float* __restrict__ blogp, const float* __restrict__ adv,
                    const float* __restrict__ vt, LossHP hp, float* __restrict__ dlog,
                    uint16_t* __restrict__ dhead, double* partials, unsigned* counter,
                    double* stats, int* flags, const int64_t* __restrict__ ver, int64_t cur) {
  APPO_PDL_ENTRY();
  const int sub = threadIdx.x & (LPS - 1);
  const int s = (blockIdx.x * blockDim.x + threadIdx.x) / LPS;
  // policy, value, entropy, ratio sums; version-lag sum and max (orchestrator.hpp:790,862-863)
  double acc[6] = {0, 0, 0, 0, 0, -1e300};
  if (s < B) {  // whole lane groups: every lane of a group takes this branch together
    const unsigned gm = (LPS == 32 ? 0xffffffffu : ((1u << LPS) - 1u) << (threadIdx.x & 31 & ~(LPS - 1)));
    const int a_s = act[s];
    if (sub == 0 && (a_s < 0 || a_s >= A)) atomicOr(flags + kFlagContract, 1);
    const int ac = min(max(a_s, 0), A - 1);
    const bool mine = sub < A;
    const double l = mine ? (double)logits[(int64_t)s * A + sub] : -1e300;
    // fp64 log-softmax over the lane group: one exp per action, a single log
    double mx = l;
#pragma unroll
    for (int o = LPS / 2; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(gm, mx, o, LPS));
    const double ex = mine ? exp(l - mx) : 0.0;
    double z = ex;
#pragma unroll
    for (int o = LPS / 2; o > 0; o >>= 1) z += __shfl_xor_sync(gm, z, o, LPS);
    const double lz = log(z);
    const double p = ex / z;
    const double lp = (l - mx) - lz;
    double H = (mine && p > 0) ? -p * lp : 0.0;
#pragma unroll
    for (int o = LPS / 2; o > 0; o >>= 1) H += __shfl_xor_sync(gm, H, o, LPS);
    const double lpa = __shfl_sync(gm, lp, ac, LPS);
    const double logp = fmax(lpa, -690.7755278982137);  // log(1e-300) floor
    double d = logp - (double)blogp[s];
    d = fmin(fmax(d, -20.0), 20.0);
    const double ratio = exp(d);
    const double A_s = adv[s];
    const double cl = fmin(fmax(ratio, (double)hp.clip_low), (double)hp.clip_high);
    const double sur = fmin(ratio * A_s, cl * A_s);
    const double dsur = (ratio * A_s <= cl * A_s) ? A_s : 0.0;  // ties -> unclipped
    const double invB = 1.0 / B;
    const double dL_dlogp = -invB * dsur * ratio;
    const double verr = (double)values[s] - (double)vt[s];
    const double dV = hp.value_coef * invB * 2.0 * verr;
    float gsub = 0.0f;
    if (mine) {
      const double dlp = (sub == ac ? 1.0 : 0.0) - p;
      const double dH = p > 0 ? -p * (lp + H) : 0.0;
      gsub = (float)(dL_dlogp * dlp - hp.entropy_coef * invB * dH);
      dlog[(int64_t)s * (A + 1) + sub] = gsub;
    } else if (sub == A) {
      gsub = (float)dV;
      dlog[(int64_t)s * (A + 1) + A] = gsub;
    }
    // bf16 head-gradient row, 16 wide: dlogits, dV, zeros
#pragma unroll
    for (int col = sub; col < 16; col += LPS) dhead[(int64_t)s * 16 + col] = col <= A ? f2bf(gsub) : 0;
    if (sub == 0) {
      acc[0] = -sur;
      acc[1] = verr * verr;
      acc[2] = H;
      acc[3] = ratio;
      acc[4] = (double)(cur - ver[s]);
      acc[5] = (double)(cur - ver[s]);
    }
  }
  // block reduce + last block
  __shared__ double sh[8][6];
  __shared__ bool last;
#pragma unroll
  for (int k = 0; k < 5; ++k) acc[k] = warp_sum(acc[k]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc[5] = fmax(acc[5], __shfl_xor_sync(0xffffffffu, acc[5], o));
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int k = 0; k < 6; ++k) sh[threadIdx.x >> 5][k] = acc[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < 6; ++k) {
      double t = k == 5 ? -1e300 : 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = k == 5 ? fmax(t, sh[w][k]) : t + sh[w][k];
      partials[blockIdx.x * 6 + k] = t;
    }
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    // whole last block: thread b loads block b's partials (b, b + blockDim, ..
    // summed in that order), then a fixed-order tree over the threads
    // (deterministic; one memory round trip instead of a serial walk)
    __threadfence();
    double t[6] = {0, 0, 0, 0, 0, -1e300};
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x)
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const double x = __ldcg(partials + b * 6 + k);
        t[k] = k == 5 ? fmax(t[k], x) : t[k] + x;
      }
#pragma unroll
    for (int k = 0; k < 5; ++k) t[k] = warp_sum(t[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t[5] = fmax(t[5], __shfl_xor_sync(0xffffffffu, t[5], o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0)
#pragma unroll
      for (int k = 0; k < 6; ++k) sh[threadIdx.x >> 5][k] = t[k];
    __syncthreads();
  }
  if (last && threadIdx.x == 0) {
    double t[6] = {0, 0, 0, 0, 0, -1e300};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
      for (int k = 0; k < 6; ++k) t[k] = k == 5 ? fmax(t[k], sh[w][k]) : t[k] + sh[w][k];
    const double invB = 1.0 / B;
    stats[0] = t[0] * invB;
    stats[1] = hp.value_coef * t[1] * invB;
    stats[2] = t[2] * invB;
    stats[3] = stats[0] + stats[1] - hp.entropy_coef * stats[2];
    stats[4] = t[3] * invB;
    stats[6] = B > 0 ? t[4] * invB : 0.0;
    stats[7] = B > 0 ? t[5] : 0.0;
    if (!isfinite(stats[3])) atomicOr(flags + kFlagNumeric, 1);
    *counter = 0;
  }
}

// Heads backward in one kernel (policy.hpp:377-383 analogue for the heads):
// dcore[s][j] = sum_a dlog[s][a] * Wh[a][j] (Wh = policy rows then the value
// row) and the head gradients dWh[a][j] = sum_s dlog[s][a] * core[s][j],
// dbh[a] = sum_s dlog[s][a] in fp32.  Block = a range of rows x 512 columns
// (thread j), walked in chunks of kHbRows: the chunk's dlog rows are staged in
// shared memory and its core values loaded into registers up front (one
// memory round trip per chunk instead of one per row); per-block partials are
// summed in block order by heads_grad_reduce_kernel (deterministic).
constexpr int kHbRows = 16;
template <int AMAX>
__global__ void __launch_bounds__(512)
    heads_bwd_fused_kernel(int B, int A, const float* __restrict__ dlog,
                           const float* __restrict__ core, const float* __restrict__ wpi,
                           const float* __restrict__ wv, float* __restrict__ dcore,
                           float* __restrict__ part, unsigned* counter, float* gwpi, float* gbpi,
                           float* gwv, float* gbv) {
  APPO_PDL_ENTRY();
  __shared__ float sdl[kHbRows][AMAX + 1];
  const int j = threadIdx.x;
  const int A1 = A + 1;
  const int rows = (B + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * rows, r1 = min(B, r0 + rows);
  float w[AMAX + 1], sw[AMAX + 1], sb = 0.0f;
#pragma unroll
  for (int a = 0; a <= AMAX; ++a) {
    w[a] = a < A ? wpi[a * kHidden + j] : (a == A ? wv[j] : 0.0f);
    sw[a] = 0.0f;
  }
  for (int c0 = r0; c0 < r1; c0 += kHbRows) {
    const int nr = min(kHbRows, r1 - c0);
    __syncthreads();  // previous chunk's sdl reads done
    if (j < kHbRows * A1) {
      const int r = j / A1, a = j - r * A1;
      sdl[r][a] = r < nr ? dlog[(int64_t)(c0 + r) * A1 + a] : 0.0f;
    }
    float cv[kHbRows];
#pragma unroll
    for (int r = 0; r < kHbRows; ++r) cv[r] = r < nr ? core[(int64_t)(c0 + r) * kHidden + j] : 0.0f;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kHbRows; ++r) {
      if (r < nr) {
        float dc = 0.0f;
#pragma unroll
        for (int a = 0; a <= AMAX; ++a) {
          if (a < A1) {
            const float g = sdl[r][a];
            dc += g * w[a];
            sw[a] += g * cv[r];
          }
        }
        dcore[(int64_t)(c0 + r) * kHidden + j] = dc;
        if (j < A1) sb += sdl[r][j];
      }
    }
  }
  float* pb = part + (size_t)blockIdx.x * (A1 * kHidden + A1);
#pragma unroll
  for (int a = 0; a <= AMAX; ++a)
    if (a < A1) pb[a * kHidden + j] = sw[a];
  if (j < A1) pb[A1 * kHidden + j] = sb;
}

// Sums the per-block head-gradient partials in a fixed order: block = 32
// outputs x 8 warps, warp g sums blocks g, g+8, ... (loads issued 8 ahead),
// then the 8 warp sums are added in warp order (deterministic).
__global__ void __launch_bounds__(256)
    heads_grad_reduce_kernel(int A, int nb, const float* __restrict__ part, float* gwpi,
                             float* gbpi, float* gwv, float* gbv) {
  APPO_PDL_ENTRY();
  __shared__ float sh[8][33];
  const int A1 = A + 1;
  const int stride = A1 * kHidden + A1;
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int o = blockIdx.x * 32 + lane;
  float t = 0.0f;
  if (o < stride) {
    for (int b0 = g; b0 < nb; b0 += 64) {
      float x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        x[k] = b0 + 8 * k < nb ? __ldg(part + (size_t)(b0 + 8 * k) * stride + o) : 0.0f;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (b0 + 8 * k < nb) t += x[k];
    }
  }
  sh[g][lane] = t;
  __syncthreads();
  if (g != 0 || o >= stride) return;
  t = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; ++k) t += sh[k][lane];
  if (o < A * kHidden) gwpi[o] = t;
  else if (o < A1 * kHidden) gwv[o - A * kHidden] = t;
  else if (o - A1 * kHidden < A) gbpi[o - A1 * kHidden] = t;
  else gbv[0] = t;
}

// One reverse BPTT step at time t (oracle orc_learner_step): dh = dcore + keep*dnext;
// gate gradients -> dgi / dgh rows (bf16); dnext <- dh*z (the GEMM then adds dgh . W_hh).
__global__ void gru_bwd_kernel(int n_traj, int T, int t, const float* __restrict__ dcore,
                               const uint8_t* __restrict__ done, const float* __restrict__ gates,
                               const float* __restrict__ hin, float* __restrict__ dnext,
                               uint16_t* __restrict__ dgi, uint16_t* __restrict__ dgh) {
  APPO_PDL_ENTRY();
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_traj * kHidden) return;
  const int i = g / kHidden, j = g % kHidden;
  const int64_t s = (int64_t)i * T + t;
  const float keep = done[s] ? 0.0f : 1.0f;
  const float dh = dcore[s * kHidden + j] + keep * dnext[g];
  const float* gs = gates + s * 4 * kHidden;
  const float r = gs[j], z = gs[kHidden + j], n = gs[2 * kHidden + j], ghn = gs[3 * kHidden + j];
  const float hp = hin[s * kHidden + j];
  const float dn = dh * (1.0f - z);
  const float dz = dh * (hp - n);
  const float dan = dn * (1.0f - n * n);
  const float dr = dan * ghn;
  const float dgr = dr * r * (1.0f - r);
  const float dgz = dz * z * (1.0f - z);
  uint16_t* gi_row = dgi + s * kGates;
  uint16_t* gh_row = dgh + s * kGates;
  gi_row[j] = f2bf(dgr);
  gi_row[kHidden + j] = f2bf(dgz);
  gi_row[2 * kHidden + j] = f2bf(dan);
  gh_row[j] = f2bf(dgr);
  gh_row[kHidden + j] = f2bf(dgz);
  gh_row[2 * kHidden + j] = f2bf(dan * r);
  dnext[g] = dh * z;
}

// Column sums (bias gradients): partial[chunk][n] over row chunks, then reduce.
template <bool BF16>
__global__ void colsum_partial_kernel(int64_t M, int N, const void* __restrict__ src,
                                      int64_t ld, int rows_per_chunk, float* __restrict__ part) {
  APPO_PDL_ENTRY();
  const int n = blockIdx.x * 32 + (threadIdx.x & 31);
  const int grp = threadIdx.x >> 5;  // 8 row groups
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_chunk;
  const int64_t r1 = min(r0 + rows_per_chunk, M);
  float acc = 0.0f;
  if (n < N) {
    for (int64_t r = r0 + grp; r < r1; r += 8) {
      acc += BF16 ? bf2f(reinterpret_cast<const uint16_t*>(src)[r * ld + n])
                  : reinterpret_cast<const float*>(src)[r * ld + n];
    }
  }
  __shared__ float sh[8][32];
  sh[grp][threadIdx.x & 31] = acc;
  __syncthreads();
  if (grp == 0 && n < N) {
    float t = 0;
    for (int k = 0; k < 8; ++k) t += sh[k][threadIdx.x & 31];
    part[(int64_t)blockIdx.y * N + n] = t;
  }
}
__global__ void colsum_final_kernel(int N, int chunks, const float* __restrict__ part,
                                    float* __restrict__ out, int accumulate) {
  APPO_PDL_ENTRY();
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  float t = 0;
  for (int c = 0; c < chunks; ++c) t += part[(int64_t)c * N + n];
  out[n] = accumulate ? out[n] + t : t;
}

int grid_for(int64_t n, int block, int max_blocks) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  return (int)(g < max_blocks ? g : max_blocks);
}

}  // namespace

// module anchor for preload_library_kernels (slotq.cu)
const void* kanchor_model() { return reinterpret_cast<const void*>(&im2col_u8_kernel); }

int k_im2col_u8(Ctx* c, const ObsSrc& src, int64_t R, const Dims& d, uint16_t* col) {
  const int64_t n = R * d.P1 * d.C * 8;
  c->next_bytes = (double)R * d.obs_dim + (double)R * d.P1 * d.K1 * 2;
  APPO_LAUNCH(c, im2col_u8_kernel, grid_for(n, 256, c->num_sms * 32), 256, 0, src, R, d.C, d.H,
              d.W, d.H1, d.W1, col);
  return APPO_OK;
}
int k_im2col_nhwc(Ctx* c, const uint16_t* act, int64_t R, int Hi, int Wi, int Cin, int k, int s,
                  int Ho, int Wo, uint16_t* col) {
  const int64_t n = R * Ho * Wo * k * k * (Cin / 8);
  c->next_bytes = (double)R * Hi * Wi * Cin * 2 + (double)R * Ho * Wo * k * k * Cin * 2;
  APPO_LAUNCH(c, im2col_nhwc_kernel, grid_for(n, 256, c->num_sms * 32), 256, 0, act, R, Hi, Wi,
              Cin, k, s, Ho, Wo, col);
  return APPO_OK;
}
int k_publish_derived(Ctx* c, const uint16_t* wb, const float* pf, const Dims& d, uint16_t* c1h,
                      float* c1b, uint16_t* wt2, uint16_t* wt3) {
  APPO_LAUNCH(c, publish_derived_kernel, 148, 256, 0, wb, pf, d.off_c1w, d.off_c1b, d.K1, d.off_c2w,
              d.off_c3w, c1h, c1b, wt2, wt3);
  return APPO_OK;
}
int k_f32_to_bf16(Ctx* c, int64_t rows, const float* src, int64_t src_ld, uint16_t* dst,
                  int64_t dst_ld, int cols) {
  const int64_t n = rows * cols;
  if (src_ld == cols && dst_ld == cols && n % 4 == 0 &&
      ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    c->next_bytes = 6.0 * (double)n;
    APPO_LAUNCH(c, f32_to_bf16_vec_kernel, grid_for(n / 4, 256, c->num_sms * 16), 256, 0, n / 4,
                reinterpret_cast<const float4*>(src), reinterpret_cast<uint2*>(dst));
    return APPO_OK;
  }
  APPO_LAUNCH(c, f32_to_bf16_kernel, grid_for(rows * cols, 256, c->num_sms * 16), 256, 0, rows,
              src, src_ld, dst, dst_ld, cols);
  return APPO_OK;
}
int k_gru_infer(Ctx* c, int B, int A, const float* gi, const float* gh, const float* h_in,
                const float* wpi, const float* bpi, const float* wv, const float* bv,
                uint64_t key, uint64_t counter0, float* h_out, int32_t* actions, float* logp,
                float* values, float* logits) {
  APPO_REQUIRE(((reinterpret_cast<uintptr_t>(gi) | reinterpret_cast<uintptr_t>(gh) |
                 reinterpret_cast<uintptr_t>(h_in) | reinterpret_cast<uintptr_t>(h_out) |
                 reinterpret_cast<uintptr_t>(wpi)) & 15) == 0,
               APPO_ERR_CONTRACT, "policy_forward: hidden-state buffers must be 16-byte aligned");
  APPO_LAUNCH(c, gru_infer_kernel, (B + 7) / 8, 256, 0, B, A, gi, gh, h_in, wpi, bpi, wv, bv,
              key, counter0, h_out, actions, logp, values, logits);
  return APPO_OK;
}
int k_stage_h(Ctx* c, int n_traj, int T, int t, const float* hcur, float* hin, uint16_t* hbf) {
  APPO_LAUNCH(c, stage_h_kernel, (n_traj * kHidden + 255) / 256, 256, 0, n_traj, T, t, hcur, hin,
              hbf);
  return APPO_OK;
}
int k_gru_train(Ctx* c, int n_traj, int T, int t, const float* gi, const float* gh,
                const uint8_t* done, float* hcur, float* core, uint16_t* core_bf, float* gates) {
  APPO_LAUNCH(c, gru_train_kernel, (n_traj * kHidden + 255) / 256, 256, 0, n_traj, T, t, gi, gh,
              done, hcur, core, core_bf, gates);
  return APPO_OK;
}
int k_heads_fwd(Ctx* c, int64_t R, int A, const float* core, const float* wpi, const float* bpi,
                const float* wv, const float* bv, float* logits, float* values, int64_t B,
                const int32_t* act, float* tlogp, float* ent) {
  APPO_REQUIRE(((reinterpret_cast<uintptr_t>(core) | reinterpret_cast<uintptr_t>(wpi)) & 15) == 0,
               APPO_ERR_CONTRACT, "heads: core / policy head must be 16-byte aligned");
  c->next_name = "heads_fwd_kernel";
  if (A <= 8)
    APPO_LAUNCH(c, heads_fwd_kernel<8>, (int)((R + 7) / 8), 256, 0, R, A, core, wpi, bpi, wv, bv,
                logits, values, B, act, tlogp, ent, c->d_flags);
  else
    APPO_LAUNCH(c, heads_fwd_kernel<kMaxActions>, (int)((R + 7) / 8), 256, 0, R, A, core, wpi, bpi,
                wv, bv, logits, values, B, act, tlogp, ent, c->d_flags);
  c->next_name = nullptr;
  return APPO_OK;
}
int k_gather_slots(Ctx* c, int n_traj, int T, const uint8_t* region, uint64_t slot_bytes,
                   const int32_t* slot_ids, const SlotOffsets& off, int32_t* act, float* rew,
                   float* blogp, uint8_t* done, int64_t* ver, float* h0) {
  APPO_LAUNCH(c, gather_slots_kernel, n_traj, 128, 0, n_traj, T, region, slot_bytes, slot_ids,
              off, act, rew, blogp, done, ver, h0, c->d_flags);
  return APPO_OK;
}
int k_normalize(Ctx* c, int n, float* adv) {
  APPO_LAUNCH(c, normalize_kernel, 1, 1024, 0, n, adv);
  return APPO_OK;
}
int k_ppo_loss(Ctx* c, int B, int A, const float* logits, const float* values,
               const int32_t* act, const float* blogp, const float* adv, const float* vt,
               const LossHP& hp, float* dlog, uint16_t* dhead, double* stats, const int64_t* ver,
               int64_t cur) {
  // lane groups of 8 (A <= 7) or 16 per sample, 256-thread blocks
  const int lps = A < 8 ? 8 : 16;
  const int grid = (B + 256 / lps - 1) / (256 / lps);
  APPO_REQUIRE(grid * 6 <= kRedSlots, APPO_ERR_CONTRACT, "ppo_loss: batch too large");
  // in: logits, value, action, behaviour logp, advantage, v-target, version;
  // out: dlogits + dV (fp32) and the bf16 head-gradient row (16 wide)
  c->next_bytes = (double)B * (A * 4 + 28 + (A + 1) * 4 + 32);
  c->next_name = "ppo_loss_kernel";
  if (lps == 8)
    APPO_LAUNCH(c, ppo_loss_kernel<8>, grid, 256, 0, B, A, logits, values, act, blogp, adv, vt, hp,
                dlog, dhead, c->d_red, c->d_counter + 2, stats, c->d_flags, ver, cur);
  else
    APPO_LAUNCH(c, ppo_loss_kernel<16>, grid, 256, 0, B, A, logits, values, act, blogp, adv, vt,
                hp, dlog, dhead, c->d_red, c->d_counter + 2, stats, c->d_flags, ver, cur);
  c->next_name = nullptr;
  return APPO_OK;
}
int k_heads_bwd_fused(Ctx* c, int B, int A, const float* dlog, const float* core,
                      const float* wpi, const float* wv, float* dcore, float* part, float* gwpi,
                      float* gbpi, float* gwv, float* gbv) {
  int grid = (B + 15) / 16;  // 16 rows per block
  if (grid > 160) grid = 160;
  if (grid < 1) grid = 1;
  c->next_name = "heads_bwd_fused_kernel";
  if (A < 8)
    APPO_LAUNCH(c, heads_bwd_fused_kernel<7>, grid, 512, 0, B, A, dlog, core, wpi, wv, dcore,
                part, c->d_counter + 7, gwpi, gbpi, gwv, gbv);
  else
    APPO_LAUNCH(c, heads_bwd_fused_kernel<kMaxActions>, grid, 512, 0, B, A, dlog, core, wpi, wv,
                dcore, part, c->d_counter + 7, gwpi, gbpi, gwv, gbv);
  c->next_name = nullptr;
  return k_heads_grad_reduce(c, A, grid, part, gwpi, gbpi, gwv, gbv);
}
int k_heads_grad_reduce(Ctx* c, int A, int nb, const float* part, float* gwpi, float* gbpi,
                        float* gwv, float* gbv) {
  const int outs = (A + 1) * (kHidden + 1);
  APPO_LAUNCH(c, heads_grad_reduce_kernel, (outs + 31) / 32, 256, 0, A, nb, part, gwpi, gbpi,
              gwv, gbv);
  return APPO_OK;
}
int k_gru_bwd(Ctx* c, int n_traj, int T, int t, const float* dcore, const uint8_t* done,
              const float* gates, const float* hin, float* dnext, uint16_t* dgi, uint16_t* dgh) {
  APPO_LAUNCH(c, gru_bwd_kernel, (n_traj * kHidden + 255) / 256, 256, 0, n_traj, T, t, dcore,
              done, gates, hin, dnext, dgi, dgh);
  return APPO_OK;
}
int k_colsum(Ctx* c, int64_t M, int N, const void* src, int64_t ld, bool bf16, float* part,
             float* out, bool accumulate) {
  int chunks = (int)((M + 255) / 256);
  if (chunks > 256) chunks = 256;
  if (chunks < 1) chunks = 1;
  const int rows_per_chunk = (int)((M + chunks - 1) / chunks);
  dim3 grid((N + 31) / 32, chunks);
  if (bf16)
    APPO_LAUNCH(c, colsum_partial_kernel<true>, grid, 256, 0, M, N, src, ld, rows_per_chunk,
                part);
  else
    APPO_LAUNCH(c, colsum_partial_kernel<false>, grid, 256, 0, M, N, src, ld, rows_per_chunk,
                part);
  APPO_LAUNCH(c, colsum_final_kernel, (N + 255) / 256, 256, 0, N, chunks, part, out,
              accumulate ? 1 : 0);
  return APPO_OK;
}
}  // namespace appo_b200
