// Inference GRU step fused into its gate GEMMs (sm_100a tcgen05), SURVEY.md
// §2.2 K2/K3: the per-env gate pre-activations never leave TMEM.
//
// Tile = 128 envs x 64 hidden units (unit block ub).  Over K = 512 of x (the
// encoder output, bf16) one MMA chain of N = 192 accumulates [W_ir; W_iz; W_in]
// rows of the block into TMEM columns [r | z | n_i]; over K = 512 of h (bf16
// copy of h_in) two chains accumulate [W_hr; W_hz] into the same [r | z]
// columns and W_hn into a fourth block [n_h] (PyTorch's n = tanh(x W_in + b_in
// + r * (h W_hn + b_hn)) keeps the two n parts apart).  4 x 64 columns per
// tile, double-buffered = all 512 TMEM columns.  The epilogue applies the cell
// (fp32, as policy forward / oracle gru_fwd), writes h' and the tile's partial
// policy / value head dot products over its 64 units; heads_sample_kernel sums
// the 16 partials of an env (8 unit blocks x 2 epilogue halves), adds the head
// biases and samples (fp64 inverse CDF, as gru_infer_kernel).
//
//   warp 0      TMA: per K block the A block (x or h: 128 x 64) and the three
//               64-row gate slices of W_ih or W_hh (24 KB), 4-stage ring
//   warp 1      TMEM owner + MMA issuer
//   warps 2..9  epilogue: 2 warps per TMEM lane quarter, 32 units each
//
// Replaces the inference tail of forward_batch (policy.hpp:165-200; the
// reference's MLP core stands where the GRU is): the fp32
// gi / gh round trip of the unfused path (2 x 100 MB written and re-read per
// 16,384-env step).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "appo_common.cuh"
#include "gemm.cuh"
#include "model_kernels.cuh"
#include "sm100.cuh"

namespace appo_b200 {
namespace {

constexpr int GI_EPI_WARPS = 8;
constexpr int GI_THREADS = 32 * (2 + GI_EPI_WARPS);
constexpr int GI_UB = 64;                     // units per tile
constexpr int GI_NUB = kHidden / GI_UB;       // 8 unit blocks
constexpr int GI_NST = 4;                     // stages
constexpr int GI_A = 128 * 128;               // A block: 128 rows x 64 K (bf16, SW128)
constexpr int GI_B = 192 * 128;               // B block: 3 gate slices x 64 rows x 64 K
constexpr int GI_STAGE = GI_A + GI_B;         // 40 KB
constexpr int GI_SMEM = 1024 + GI_NST * GI_STAGE + 256 + 4 * kHidden * 4;  // + gate biases
constexpr int GI_PW = 8;                      // partial heads per (env, half-tile): A <= 7 logits + value

struct GiParams {
  int B, A;
  const float* h_in;      // fp32 [B][512]
  const float* b_ih;      // [1536]
  const float* b_hh;      // [1536]
  const float* wpi;       // [A][512]
  const float* wv;        // [512]
  float* h_out;           // fp32 [B][512]
  float* part;            // [GI_NUB * 2][B][GI_PW]
};

__device__ __forceinline__ void gi_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  sm100::tmem_ld16(taddr, r);
}
// fast-math gates (MUFU ex2 + fast divide, |err| ~1e-7: far below the bf16
// rounding of the GEMM operands), as the learner's GRU kernels
__device__ __forceinline__ float gi_sig(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }
__device__ __forceinline__ float gi_tanh(float x) { return 2.0f * gi_sig(2.0f * x) - 1.0f; }

__global__ void __launch_bounds__(GI_THREADS, 1)
    gru_infer_fused_kernel(const __grid_constant__ CUtensorMap map_x,
                           const __grid_constant__ CUtensorMap map_h,
                           const __grid_constant__ CUtensorMap map_wih,
                           const __grid_constant__ CUtensorMap map_whh,
                           const __grid_constant__ GiParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + GI_NST * GI_STAGE);
  uint64_t* full = bars;
  uint64_t* empty = full + GI_NST;
  uint64_t* acc_full = empty + GI_NST;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  // gate biases by unit: b_ir + b_hr, b_iz + b_hz, b_in, b_hn
  float* sbias = reinterpret_cast<float*>(smem + GI_NST * GI_STAGE + 256);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = (p.B + 127) / 128, units = tiles_m * GI_NUB;

  if (threadIdx.x == 0) {
    sm100::tma_prefetch(&map_x);
    sm100::tma_prefetch(&map_h);
    sm100::tma_prefetch(&map_wih);
    sm100::tma_prefetch(&map_whh);
    for (int s = 0; s < GI_NST; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&acc_full[s], 1);
      sm100::mbar_init(&acc_empty[s], GI_EPI_WARPS);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) {
    sm100::tmem_alloc(tmem_slot, 512);
    sm100::tmem_relinquish();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  APPO_PDL_ENTRY();  // x, h (bf16) and the published weights come from earlier kernels
  for (int j = threadIdx.x; j < kHidden; j += GI_THREADS) {
    sbias[j] = p.b_ih[j] + p.b_hh[j];
    sbias[kHidden + j] = p.b_ih[kHidden + j] + p.b_hh[kHidden + j];
    sbias[2 * kHidden + j] = p.b_ih[2 * kHidden + j];
    sbias[3 * kHidden + j] = p.b_hh[2 * kHidden + j];
  }
  __syncthreads();

  if (warp == 0) {
    // ---- TMA: 16 K blocks per tile (8 of x with W_ih, 8 of h with W_hh) ----
    int stage = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int tm = u / GI_NUB, ub = u % GI_NUB;
      for (int kb = 0; kb < 16; ++kb) {
        sm100::mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = smem + stage * GI_STAGE;
        uint8_t* sb = sa + GI_A;
        const bool hpart = kb >= 8;
        const int k0 = (kb & 7) * 64;
        sm100::mbar_arrive_expect_tx_warp(&full[stage], GI_STAGE);
        sm100::tma_load_3d_warp(sa, hpart ? &map_h : &map_x, &full[stage], k0, tm * 128, 0);
#pragma unroll
        for (int g = 0; g < 3; ++g)
          sm100::tma_load_3d_warp(sb + g * 64 * 128, hpart ? &map_whh : &map_wih, &full[stage], k0,
                                  g * kHidden + ub * GI_UB, 0);
        if (++stage == GI_NST) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---- MMA: x part -> [r | z | n_i] (N 192); h part -> [r | z] (N 128) + [n_h] (N 64) ----
    constexpr uint32_t id192 = sm100::make_idesc_bf16(128, 192, 0, 0);
    constexpr uint32_t id128 = sm100::make_idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t id64 = sm100::make_idesc_bf16(128, 64, 0, 0);
    int stage = 0, acc = 0;
    uint32_t phase = 0, accph = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      sm100::mbar_wait(&acc_empty[acc], accph ^ 1);
      sm100::tc_fence_after();
      const uint32_t d = tmem_base + acc * 256;
      for (int kb = 0; kb < 16; ++kb) {
        sm100::mbar_wait(&full[stage], phase);
        sm100::tc_fence_after();
        const uint32_t a0 = sm100::smem_u32(smem + stage * GI_STAGE), b0 = a0 + GI_A;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = sm100::make_sdesc(a0 + k * 32, 16, 1024);
          if (kb < 8) {
            sm100::umma_f16_warp(d, ad, sm100::make_sdesc(b0 + k * 32, 16, 1024), id192,
                                 (kb | k) ? 1u : 0u);
          } else {
            sm100::umma_f16_warp(d, ad, sm100::make_sdesc(b0 + k * 32, 16, 1024), id128, 1u);
            sm100::umma_f16_warp(d + 192, ad, sm100::make_sdesc(b0 + 128 * 128 + k * 32, 16, 1024),
                                 id64, (kb > 8 || k) ? 1u : 0u);
          }
        }
        sm100::umma_commit_warp(&empty[stage]);
        if (++stage == GI_NST) { stage = 0; phase ^= 1; }
      }
      sm100::umma_commit_warp(&acc_full[acc]);
      if (++acc == 2) { acc = 0; accph ^= 1; }
    }
  } else {
    // ---- epilogue: lanes = envs of quarter q, units part*32 .. +32 of the block ----
    const int ew = warp - 2, q = warp & 3, part = ew >> 2;
    int acc = 0;
    uint32_t accph = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int tm = u / GI_NUB, ub = u % GI_NUB;
      const int env = tm * 128 + q * 32 + lane;
      const bool ok = env < p.B;
      sm100::mbar_wait(&acc_full[acc], accph);
      sm100::tc_fence_after();
      float hp[GI_PW];
#pragma unroll
      for (int a = 0; a < GI_PW; ++a) hp[a] = 0.0f;
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        const int c0 = part * 32 + ch * 16;  // unit within the block
        const int j0 = ub * GI_UB + c0;      // hidden unit
        const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + acc * 256 + c0;
        uint32_t rr[16], rz[16], rni[16], rnh[16];
        gi_ld16(ta, rr);
        gi_ld16(ta + 64, rz);
        gi_ld16(ta + 128, rni);
        gi_ld16(ta + 192, rnh);
        sm100::tmem_ld_wait();
        float hprev[16];
        const float4* hsrc = reinterpret_cast<const float4*>(p.h_in + (size_t)(ok ? env : 0) * kHidden + j0);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4 v = __ldg(hsrc + k);
          hprev[4 * k] = v.x; hprev[4 * k + 1] = v.y; hprev[4 * k + 2] = v.z; hprev[4 * k + 3] = v.w;
        }
        float hn[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int j = j0 + k;
          const float r = gi_sig(__uint_as_float(rr[k]) + sbias[j]);
          const float z = gi_sig(__uint_as_float(rz[k]) + sbias[kHidden + j]);
          const float n = gi_tanh(__uint_as_float(rni[k]) + sbias[2 * kHidden + j] +
                                  r * (__uint_as_float(rnh[k]) + sbias[3 * kHidden + j]));
          hn[k] = (1.0f - z) * n + z * hprev[k];
        }
        if (ok) {
          float4* dst = reinterpret_cast<float4*>(p.h_out + (size_t)env * kHidden + j0);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            dst[k] = make_float4(hn[4 * k], hn[4 * k + 1], hn[4 * k + 2], hn[4 * k + 3]);
        }
        // partial heads over these 16 units (head rows are warp-uniform: broadcast loads)
#pragma unroll
        for (int a = 0; a < GI_PW - 1; ++a)
          if (a < p.A) {
            const float4* w4 = reinterpret_cast<const float4*>(p.wpi + (size_t)a * kHidden + j0);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float4 w = __ldg(w4 + k);
              hp[a] += w.x * hn[4 * k] + w.y * hn[4 * k + 1] + w.z * hn[4 * k + 2] + w.w * hn[4 * k + 3];
            }
          }
#pragma unroll
        for (int k = 0; k < 16; ++k) hp[GI_PW - 1] += __ldg(p.wv + j0 + k) * hn[k];
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&acc_empty[acc]);
      if (++acc == 2) { acc = 0; accph ^= 1; }
      if (ok) {
        float4* dst = reinterpret_cast<float4*>(p.part + ((size_t)(ub * 2 + part) * p.B + env) * GI_PW);
        dst[0] = make_float4(hp[0], hp[1], hp[2], hp[3]);
        dst[1] = make_float4(hp[4], hp[5], hp[6], hp[7]);
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem_base, 512);
  }
}

// Sum the 16 partial head rows of an env (fixed order), add the head biases,
// softmax + inverse-CDF sample in fp64 with the env's counter-based uniform
// (the same draw as gru_infer_kernel / the oracle).
__global__ void heads_sample_kernel(int B, int A, const float* __restrict__ part,
                                    const float* __restrict__ bpi, const float* __restrict__ bv,
                                    uint64_t key, uint64_t counter0, int32_t* __restrict__ actions,
                                    float* __restrict__ logp, float* __restrict__ values,
                                    float* __restrict__ logits_out) {
  APPO_PDL_ENTRY();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  float acc[GI_PW];
#pragma unroll
  for (int a = 0; a < GI_PW; ++a) acc[a] = 0.0f;
#pragma unroll 4
  for (int s = 0; s < 2 * GI_NUB; ++s) {
    const float4* src = reinterpret_cast<const float4*>(part + ((size_t)s * B + b) * GI_PW);
    const float4 v0 = __ldg(src), v1 = __ldg(src + 1);
    acc[0] += v0.x; acc[1] += v0.y; acc[2] += v0.z; acc[3] += v0.w;
    acc[4] += v1.x; acc[5] += v1.y; acc[6] += v1.z; acc[7] += v1.w;
  }
  double lg[GI_PW - 1];
  double mx = -1e300;
  for (int a = 0; a < A; ++a) {
    lg[a] = (double)(acc[a] + bpi[a]);
    mx = fmax(mx, lg[a]);
    if (logits_out) logits_out[(int64_t)b * A + a] = (float)lg[a];
  }
  values[b] = acc[GI_PW - 1] + bv[0];
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

}  // namespace

const void* kanchor_gru_infer() { return reinterpret_cast<const void*>(&gru_infer_fused_kernel); }

bool gru_infer_fused_supported(int B, int A) { return B > 0 && A >= 1 && A <= GI_PW - 1; }

int gru_infer_fused(Ctx* c, int B, int A, const uint16_t* x, const uint16_t* hbf,
                    const uint16_t* w_ih, const uint16_t* w_hh, const float* b_ih,
                    const float* b_hh, const float* h_in, const float* wpi, const float* bpi,
                    const float* wv, const float* bv, uint64_t key, uint64_t counter0,
                    float* part, float* h_out, int32_t* actions, float* logp, float* values,
                    float* logits) {
  APPO_REQUIRE(gru_infer_fused_supported(B, A), APPO_ERR_CONTRACT, "gru_infer_fused: shape");
  APPO_REQUIRE(((reinterpret_cast<uintptr_t>(h_in) | reinterpret_cast<uintptr_t>(h_out) |
                 reinterpret_cast<uintptr_t>(wpi) | reinterpret_cast<uintptr_t>(part)) & 15) == 0,
               APPO_ERR_CONTRACT, "gru_infer_fused: 16-byte alignment");
  CUtensorMap mx, mh, mwi, mwh;
  // activations [B][512] bf16, box {64 K, 128 rows}; weights [1536][512], box {64 K, 64 rows}
  int st = make_tmap_bf16_3d(&mx, x, kHidden, (uint64_t)B, 1, kHidden * 2, (uint64_t)B * kHidden * 2,
                             64, 128, 1);
  if (!st) st = make_tmap_bf16_3d(&mh, hbf, kHidden, (uint64_t)B, 1, kHidden * 2,
                                  (uint64_t)B * kHidden * 2, 64, 128, 1);
  if (!st) st = make_tmap_bf16_3d(&mwi, w_ih, kHidden, kGates, 1, kHidden * 2,
                                  (uint64_t)kGates * kHidden * 2, 64, 64, 1);
  if (!st) st = make_tmap_bf16_3d(&mwh, w_hh, kHidden, kGates, 1, kHidden * 2,
                                  (uint64_t)kGates * kHidden * 2, 64, 64, 1);
  if (st) return st;
  GiParams p{};
  p.B = B;
  p.A = A;
  p.h_in = h_in;
  p.b_ih = b_ih;
  p.b_hh = b_hh;
  p.wpi = wpi;
  p.wv = wv;
  p.h_out = h_out;
  p.part = part;
  static int attr_bytes[64] = {};
  const int dev = c->device & 63;
  if (attr_bytes[dev] < GI_SMEM) {
    APPO_CUDA_TRY(cudaFuncSetAttribute(gru_infer_fused_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, GI_SMEM));
    attr_bytes[dev] = GI_SMEM;
  }
  const int units = (B + 127) / 128 * GI_NUB;
  const int grid = c->num_sms < units ? c->num_sms : units;
  c->next_name = "gru_infer_fused_tcgen05";
  c->next_flops = 2.0 * B * 512.0 * (3 * 512 + 3 * 512);
  c->next_bytes = 2.0 * B * 512 * 2 + 4.0 * B * 512 * 2 + 4.0 * 16 * B * GI_PW;
  APPO_LAUNCH(c, gru_infer_fused_kernel, grid, GI_THREADS, GI_SMEM, mx, mh, mwi, mwh, p);
  c->next_name = "heads_sample_kernel";
  APPO_LAUNCH(c, heads_sample_kernel, (B + 127) / 128, 128, 0, B, A, part, bpi, bv, key, counter0,
              actions, logp, values, logits);
  return APPO_OK;
}

}  // namespace appo_b200
