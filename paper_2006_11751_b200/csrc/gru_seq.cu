// Persistent GRU recurrence for the learner: the T-step forward unroll (+ the
// bootstrap step) and the BPTT reverse sweep each run as ONE cooperative
// kernel; the per-step recurrent product runs on tcgen05.
//
// The trajectories are split in groups of 32 (GT).  A CTA owns 16 hidden units
// of one group; the only cross-CTA traffic is the per-step exchange of its
// group (h_{t+1} forward, the gate gradients dgh_t backward, bf16, L2-resident)
// behind one barrier per step among the group's CTAs.  What bounds a step is
// how fast one SM takes the exchange in from L2 (~40 B/cycle measured): the
// group split halves it relative to a CTA that stages all 64 trajectories.
//
//   forward : 32 CTAs per group x 16 units.  D = h_t W_hh[own gate rows]^T as
//             ONE M=128 UMMA chain whose rows are (K quarter q, trajectory) and
//             N = (quarter, 48 gate rows r,z,n of the units) = 192, K = 128:
//             the four diagonal blocks are the quarter partial sums (a quarter
//             of the MMA instructions of an M=32 chain, which tcgen05 lacks).
//             W slice resident (bf16, SW128 K-major), h_t staged by TMA per
//             K block.  The epilogue applies the cell (PyTorch r,z,n; oracle
//             gru_fwd) and stores the exchange first, the step's other outputs
//             after the barrier arrive.
//   backward: 32 CTAs per group x 16 units.  Gate gradients of own units
//             (oracle orc_learner_step BPTT) are published as dgh_t; after the
//             barrier dnext[i][j] = dh*z + sum_g dgh_t[i][g] W_hh[g][j] as one
//             M=128 chain (rows: quarter of 384 gates x trajectory, N = quarter
//             x 16 units = 64, K = 384) with W_hh[:, own]^T resident and the
//             group's dgh_t (96 KB) staged by TMA in three 32 KB parts; bias
//             gradients summed per group in a fixed order, then over the groups
//             by the last CTA of each unit block (deterministic).
// Per-cell state (h, b_hh, prefetched next-step inputs, dh*z) lives in
// registers because a thread owns the same (trajectory, unit) cells every step.
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "gemm.cuh"
#include "model.cuh"
#include "model_kernels.cuh"
#include "sm100.cuh"

namespace appo_b200 {
namespace {

constexpr int MAXTRAJ = 64;                // trajectories per learner step (2 groups)
constexpr int THR = 256;

constexpr int UPC_F = 16;                  // forward: units per CTA
constexpr int NCTA_F = kHidden / UPC_F;    // 32
constexpr int NG = 3 * UPC_F;              // 48 gate rows per CTA (forward N)


__device__ __forceinline__ uint16_t f2bf_(float f) {
  __nv_bfloat16 h = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t*>(&h);
}
// fast-math gates: MUFU ex2 + fast divide (|err| ~1e-7, far below the bf16
// operand rounding of the recurrent product)
__device__ __forceinline__ float sig_(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }
__device__ __forceinline__ float tanh_(float x) { return 2.0f * sig_(2.0f * x) - 1.0f; }
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// byte offset of 16-byte chunk c (8 bf16) of row r, K block kb in a K-major
// SW128 tile whose K blocks hold `rows` rows each
__device__ __forceinline__ uint32_t sw128(int rows, int r, int kb, int c) {
  return (uint32_t)(kb * rows * 128 + r * 128 + ((c ^ (r & 7)) << 4));
}

// Grid-wide barrier on a monotonically increasing counter (never reset: a
// launch waits for base + epoch * CTAs, the base passed by the host); all
// CTAs are co-resident (cooperative launch).
// Split form: arrive (release of everything the CTA stored before it), then
// work that no other CTA needs (deferred stores, prefetches), then wait.
__device__ __forceinline__ void grid_arrive(unsigned* counter) {
  __syncthreads();
  if (threadIdx.x == 0)
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
}
__device__ __forceinline__ void grid_wait(unsigned* counter, unsigned target) {
  if (threadIdx.x == 0) {
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
    } while ((int)(v - target) < 0);  // wrap-safe: the counters only grow
  }
  __syncthreads();
}

__device__ __forceinline__ void grid_barrier(unsigned* counter, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // release-add (cumulative over the CTA's writes ordered by the bar.sync)
    // instead of a full fence + relaxed atomic
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

// Issue cp.async copies of rows [n_rows] x 512 bf16 (global row stride ld
// elements, from column col0) into a 64-row SW128 K-major tile; rows >=
// n_rows are zero-filled.  Caller commits / waits.
#define FSTAMP(k)                                                     \
  do {                                                                \
    if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[t * 8 + (k)] = clock64(); \
  } while (0)
// ---- trajectory-group forward: 32 trajectories per CTA group --------------
// The exchange is bounded by how fast one SM can take h_t in from L2 (~40 B per
// cycle measured: 64 KB per step cost ~1.7k cycles), so the trajectories are
// split in groups of 32: CTA (group g, unit block uc) owns units 16uc..16uc+15
// of trajectories 32g..32g+31 and stages only its group's h_t (32 KB); the 32
// CTAs of a group synchronise among themselves (one counter per group).
// Recurrent product per step: one M=128 UMMA chain whose rows are (K quarter
// q, trajectory) and N = (K quarter, 48 gate rows) = 192, K = 128: the four
// diagonal blocks are the quarter partial sums.
constexpr int GT = 32;                      // trajectories per group
constexpr int GQ = 4;                       // K quarters (M = GQ * GT = 128)
constexpr int GKQ = kHidden / GQ;           // 128: K per quarter (2 SW128 K blocks)
constexpr int G_KB = 128 * 128;             // one 64-wide K block of the 128-row A tile
constexpr int G_A = 2 * G_KB;               // A tile: 32 KB
constexpr int G_NB = GQ * NG;               // 192 B rows
constexpr int G_B = 2 * G_NB * 128;         // 48 KB
// partial-sum rows padded to 52 floats: the lane-per-row float4 stores of the
// TMEM readout hit 8 distinct bank groups (a 48-float pitch put 16 lanes on
// one bank: 16-way conflicts on every store)
constexpr int GQS = NG + 4;
constexpr int G_FWD_SMEM = 1024 + G_A + G_B + GQ * GT * GQS * 4 + 64;

struct GFwdArgs {
  CUtensorMap hmap;      // 3-D map over hbuf_bf {512, n_traj, 2}, box {64, 32, 1}, SW128
  int n_traj, T;
  const float* gi;
  const uint16_t* whh;
  const float* bhh;
  const uint8_t* done;
  float* hbuf;
  uint16_t* hbuf_bf;
  float* core;
  uint16_t* core_bf;
  float* gates;
  float* hin;
  uint16_t* hbf;
  unsigned* bar;         // [groups] step counters
  unsigned base[4];      // counter values at launch, per group
  long long* prof;
};

__global__ void __launch_bounds__(THR, 1) gru_g_fwd_kernel(const __grid_constant__ GFwdArgs a) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* tA = sm;
  uint8_t* tB = sm + G_A;
  float* gq = reinterpret_cast<float*>(tB + G_B);                 // [GQ][GT][GQS] partial sums
  uint64_t* mbar = reinterpret_cast<uint64_t*>(gq + GQ * GT * GQS);
  uint64_t* kbar = mbar + 1;  // [2] one per K block (all four quarters of it)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(kbar + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = blockIdx.x / NCTA_F, uc = blockIdx.x % NCTA_F;
  const int j0 = uc * UPC_F, i0 = grp * GT;
  const int B = a.n_traj * a.T;
  unsigned* bar = a.bar + grp;
  const unsigned base = a.base[grp];

  // resident B: row q*NG + n = gate row n (g*16 + u) restricted to K quarter q
  for (int e = tid; e < G_NB * 16; e += THR) {  // 16 chunks of 16 B per 128-wide quarter row
    const int nn = e >> 4, c = e & 15;
    const int q = nn / NG, n = nn % NG;
    const int grow = (n / UPC_F) * kHidden + j0 + (n % UPC_F);
    *reinterpret_cast<uint4*>(tB + sw128(G_NB, nn, c >> 3, c & 7)) =
        reinterpret_cast<const uint4*>(a.whh + (int64_t)grow * kHidden + q * GKQ)[c];
  }
  if (tid == 0) {
    sm100::mbar_init(mbar, 1);
    sm100::mbar_init(&kbar[0], 1);
    sm100::mbar_init(&kbar[1], 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) {
    sm100::tmem_alloc(tslot, 256);
    sm100::tmem_relinquish();
  }
  // everything above reads only parameters (published by an earlier step):
  // it overlaps the previous kernel's tail
  APPO_PDL_ENTRY();
  constexpr int CPT = GT * UPC_F / THR;  // 2 cells per thread
  float hreg[CPT], b3[CPT][3], g3[CPT][3];
  uint8_t dn[CPT];
  int ci[CPT], cj[CPT], cl[CPT];
  bool cv[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int e = tid + c * THR;
    cl[c] = e / UPC_F;
    ci[c] = i0 + cl[c];
    cj[c] = j0 + e % UPC_F;
    cv[c] = ci[c] < a.n_traj;
  }
  auto prefetch = [&](int t) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if (!cv[c]) continue;
      const int64_t row = (t < a.T) ? (int64_t)ci[c] * a.T + t : (int64_t)B + ci[c];
      const float* gir = a.gi + row * kGates + cj[c];
      g3[c][0] = __ldg(gir);
      g3[c][1] = __ldg(gir + kHidden);
      g3[c][2] = __ldg(gir + 2 * kHidden);
      dn[c] = (t < a.T) ? a.done[(int64_t)ci[c] * a.T + t] : 0;
    }
  };
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    hreg[c] = cv[c] ? a.hbuf[(int64_t)ci[c] * kHidden + cj[c]] : 0.0f;
#pragma unroll
    for (int g = 0; g < 3; ++g) b3[c][g] = a.bhh[g * kHidden + cj[c]];
    if (cv[c]) a.hbuf_bf[(int64_t)ci[c] * kHidden + cj[c]] = f2bf_(hreg[c]);
  }
  prefetch(0);
  fence_proxy_async_global();
  sm100::tc_fence_before();
  grid_barrier(bar, base + NCTA_F);  // the group's h0 (bf16) complete
  sm100::tc_fence_after();
  const uint32_t tmem = *tslot;
  constexpr uint32_t idesc = sm100::make_idesc_bf16(GQ * GT, G_NB, 0, 0);
  unsigned epoch = 1;
  uint32_t phase = 0;

  for (int t = 0; t <= a.T; ++t) {
    FSTAMP(0);
    const size_t nxt = (size_t)((t + 1) & 1) * a.n_traj * kHidden;
    // the group's h_t: K block kb of quarter q = columns q*128 + kb*64, rows i0..i0+31
    if (warp == 1) {
      fence_proxy_async_global();
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        sm100::mbar_arrive_expect_tx_warp(&kbar[kb], GQ * GT * 128);
#pragma unroll
        for (int q = 0; q < GQ; ++q)
          sm100::tma_load_3d_warp(tA + kb * G_KB + q * GT * 128, &a.hmap, &kbar[kb],
                                  q * GKQ + kb * 64, i0, t & 1);
      }
    }
    if (warp == 0) {
      const uint32_t a0 = sm100::smem_u32(tA), b0 = sm100::smem_u32(tB);
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        sm100::mbar_wait(&kbar[kb], t & 1);
        sm100::tc_fence_after();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = sm100::make_sdesc(a0 + kb * G_KB + k * 32, 16, 1024);
          const uint64_t bd = sm100::make_sdesc(b0 + kb * G_NB * 128 + k * 32, 16, 1024);
          sm100::umma_f16_warp(tmem, ad, bd, idesc, (kb | k) ? 1u : 0u);
        }
      }
      sm100::umma_commit_warp(mbar);
      FSTAMP(1);
    }
    sm100::mbar_wait(mbar, phase);
    phase ^= 1;
    FSTAMP(2);
    sm100::tc_fence_after();
    if (warp < GQ) {  // TMEM lanes 32q.. = quarter q's rows; its diagonal block: columns 48q..
      uint32_t r[NG];
#pragma unroll
      for (int cb = 0; cb < NG; cb += 16)
        sm100::tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + NG * warp + cb,
                         *reinterpret_cast<uint32_t(*)[16]>(r + cb));
      sm100::tmem_ld_wait();
      float4* dst = reinterpret_cast<float4*>(gq + (warp * GT + lane) * GQS);
#pragma unroll
      for (int q = 0; q < NG / 4; ++q)
        dst[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                             __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
    }
    sm100::tc_fence_before();
    __syncthreads();
    FSTAMP(3);
    float ghv[CPT][3];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int u = cj[c] - j0;
#pragma unroll
      for (int g = 0; g < 3; ++g) {
        const int n = g * UPC_F + u;
        ghv[c][g] = ((gq[(0 * GT + cl[c]) * GQS + n] + gq[(1 * GT + cl[c]) * GQS + n]) +
                     (gq[(2 * GT + cl[c]) * GQS + n] + gq[(3 * GT + cl[c]) * GQS + n])) +
                    b3[c][g];
      }
    }
    float cvv[CPT][6];  // r, z, n, ghn, h_prev, h
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if (!cv[c]) continue;
      const float rr = sig_(g3[c][0] + ghv[c][0]);
      const float z = sig_(g3[c][1] + ghv[c][1]);
      const float n = tanh_(g3[c][2] + rr * ghv[c][2]);
      const float hp = hreg[c];
      const float h = (1.0f - z) * n + z * hp;
      cvv[c][0] = rr;
      cvv[c][1] = z;
      cvv[c][2] = n;
      cvv[c][3] = ghv[c][2];
      cvv[c][4] = hp;
      cvv[c][5] = h;
      if (t < a.T) {
        const float hn = dn[c] ? 0.0f : h;
        hreg[c] = hn;
        a.hbuf_bf[nxt + (int64_t)ci[c] * kHidden + cj[c]] = f2bf_(hn);
      }
    }
    FSTAMP(4);
    if (t < a.T) {
      fence_proxy_async_global();
      FSTAMP(5);
      grid_arrive(bar);
    }
    FSTAMP(6);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if (!cv[c]) continue;
      const int i = ci[c], j = cj[c];
      const int64_t row = (t < a.T) ? (int64_t)i * a.T + t : (int64_t)B + i;
      a.core[row * kHidden + j] = cvv[c][5];
      a.core_bf[row * kHidden + j] = f2bf_(cvv[c][5]);
      float* gs = a.gates + row * 4 * kHidden;
      gs[j] = cvv[c][0];
      gs[kHidden + j] = cvv[c][1];
      gs[2 * kHidden + j] = cvv[c][2];
      gs[3 * kHidden + j] = cvv[c][3];
      a.hin[row * kHidden + j] = cvv[c][4];
      a.hbf[row * kHidden + j] = f2bf_(cvv[c][4]);
    }
    FSTAMP(7);
    if (t < a.T) {
      prefetch(t + 1);
      grid_wait(bar, base + ++epoch * NCTA_F);
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, 256);
  }
}

// ---- trajectory-group BPTT: 32 trajectories x 16 units per CTA -------------
// Same split as the forward: the per-step exchange dgh_t is staged per group
// (32 x 1536 bf16 = 96 KB instead of 192 KB per CTA), 64 CTAs as before.
// dnext[i][j] = dh*z + sum_g dgh_t[i][g] W_hh[g][j] as one M=128 chain: rows
// (K quarter q of 384 gates, trajectory), N = (quarter, 16 units) = 64.
constexpr int UPC_GB = 16;                        // units per CTA
constexpr int NCTA_GB = kHidden / UPC_GB;         // 32 CTAs per group
constexpr int GKB_Q = kGates / GQ;                // 384 gates per K quarter = 6 K blocks
constexpr int G_BA = 6 * G_KB;                    // A: 96 KB
constexpr int G_BN = GQ * UPC_GB;                 // 64 B rows
constexpr int G_BB = 6 * G_BN * 128;              // B: 48 KB
constexpr int MMS = UPC_GB + 4;  // padded partial-sum rows (conflict-free float4 stores)
constexpr int G_BWD_SMEM = 1024 + G_BA + G_BB + GQ * GT * MMS * 4 + 64;

struct GBwdArgs {
  CUtensorMap xmap;     // 3-D map over dghx {1536, n_traj, 2}, box {64, 32, 1}, SW128
  int n_traj, T;
  const float* dcore;
  const uint8_t* done;
  const float* gates;
  const float* hin;
  const uint16_t* whh;
  uint16_t* dghx;
  uint16_t* dgi;
  uint16_t* dgh;
  float* gbih;
  float* gbhh;
  unsigned* bar;        // [groups] step counters
  unsigned base[4];     // counter values at launch, per group
  unsigned* pair;       // [NCTA_GB] bias-gradient combine counters (self-resetting)
  float* bpart;         // [groups][512][4] per-group bias partial sums
  long long* prof;
};

__global__ void __launch_bounds__(THR, 1) gru_g_bwd_kernel(const __grid_constant__ GBwdArgs a) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* tA = sm;
  uint8_t* tB = sm + G_BA;
  float* mm = reinterpret_cast<float*>(tB + G_BB);          // [GQ][GT][16] partial sums
  uint64_t* mbar = reinterpret_cast<uint64_t*>(mm + GQ * GT * MMS);
  uint64_t* kbar = mbar + 1;  // [3] one per two K blocks (32 KB)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(kbar + 3);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = blockIdx.x / NCTA_GB, uc = blockIdx.x % NCTA_GB;
  const int j0 = uc * UPC_GB, i0 = grp * GT;
  unsigned* bar = a.bar + grp;
  const unsigned base = a.base[grp];
  const int ngrp = gridDim.x / NCTA_GB;

  // resident B: row q*16 + u, K = k' in the quarter: W_hh[q*384 + k'][j0 + u]
  for (int e = tid; e < G_BN * (GKB_Q / 8); e += THR) {
    const int n = e / (GKB_Q / 8), c8 = e % (GKB_Q / 8);  // chunk of 8 gates
    const int q = n / UPC_GB, u = n % UPC_GB;
    uint32_t w[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int g = q * GKB_Q + c8 * 8 + 2 * p;
      w[p] = (uint32_t)a.whh[(int64_t)g * kHidden + j0 + u] |
             ((uint32_t)a.whh[(int64_t)(g + 1) * kHidden + j0 + u] << 16);
    }
    *reinterpret_cast<uint4*>(tB + sw128(G_BN, n, c8 >> 3, c8 & 7)) =
        make_uint4(w[0], w[1], w[2], w[3]);
  }
  if (tid == 0) {
    sm100::mbar_init(mbar, 1);
    for (int k = 0; k < 3; ++k) sm100::mbar_init(&kbar[k], 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) {
    sm100::tmem_alloc(tslot, 64);
    sm100::tmem_relinquish();
  }
  // the prologue above reads only parameters: it overlaps the previous kernel
  APPO_PDL_ENTRY();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tslot;
  constexpr uint32_t idesc = sm100::make_idesc_bf16(GQ * GT, G_BN, 0, 0);
  unsigned epoch = 0;
  uint32_t phase = 0, kphase = 0;

  constexpr int CPT = GT * UPC_GB / THR;  // 2 cells per thread
  int ci[CPT], cj[CPT], cl[CPT];
  bool cv[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int e = tid + c * THR;
    cl[c] = e / UPC_GB;
    ci[c] = i0 + cl[c];
    cj[c] = j0 + e % UPC_GB;
    cv[c] = ci[c] < a.n_traj;
  }
  float pf[CPT][7];    // dcore, r, z, n, ghn, h_in, keep
  float ddr[CPT];      // dh*z of the later step
  float bsum[CPT][4];  // per-cell sums over t of dgr, dgz, dan, dgn (bias gradients)
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    ddr[c] = 0.0f;
    bsum[c][0] = bsum[c][1] = bsum[c][2] = bsum[c][3] = 0.0f;
  }
  auto prefetch = [&](int t) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if (!cv[c]) continue;
      const int j = cj[c];
      const int64_t s = (int64_t)ci[c] * a.T + t;
      const float* gs = a.gates + s * 4 * kHidden;
      pf[c][0] = __ldg(a.dcore + s * kHidden + j);
      pf[c][1] = __ldg(gs + j);
      pf[c][2] = __ldg(gs + kHidden + j);
      pf[c][3] = __ldg(gs + 2 * kHidden + j);
      pf[c][4] = __ldg(gs + 3 * kHidden + j);
      pf[c][5] = __ldg(a.hin + s * kHidden + j);
      pf[c][6] = a.done[s] ? 0.0f : 1.0f;
    }
  };
  prefetch(a.T - 1);

  for (int t = a.T - 1; t >= 0; --t) {
    if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[t * 4 + 0] = clock64();
    uint16_t* xb = a.dghx + (size_t)(t & 1) * a.n_traj * kGates;
    uint16_t dq[CPT][4];  // dgr, dgz, dgn, dan (bf16) of this step's cells
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if (!cv[c]) continue;
      const int i = ci[c], u = cj[c] - j0, j = cj[c];
      const float dnext =
          (t == a.T - 1)
              ? 0.0f
              : ddr[c] + ((mm[(0 * GT + cl[c]) * MMS + u] + mm[(1 * GT + cl[c]) * MMS + u]) +
                          (mm[(2 * GT + cl[c]) * MMS + u] + mm[(3 * GT + cl[c]) * MMS + u]));
      const float dh = pf[c][0] + pf[c][6] * dnext;
      const float r = pf[c][1], z = pf[c][2], n = pf[c][3], ghn = pf[c][4], hp = pf[c][5];
      const float dnn = dh * (1.0f - z);
      const float dz = dh * (hp - n);
      const float dan = dnn * (1.0f - n * n);
      const float fgr = dan * ghn * r * (1.0f - r);
      const float fgz = dz * z * (1.0f - z);
      const float fgn = dan * r;
      bsum[c][0] += fgr;
      bsum[c][1] += fgz;
      bsum[c][2] += dan;
      bsum[c][3] += fgn;
      const uint16_t dgr = f2bf_(fgr);
      const uint16_t dgz = f2bf_(fgz);
      const uint16_t dgn = f2bf_(fgn);
      dq[c][0] = dgr;
      dq[c][1] = dgz;
      dq[c][2] = dgn;
      dq[c][3] = f2bf_(dan);
      if (t > 0) {  // the exchange: the only store other CTAs wait for
        uint16_t* xr = xb + (int64_t)i * kGates;
        xr[j] = dgr;
        xr[kHidden + j] = dgz;
        xr[2 * kHidden + j] = dgn;
      }
      ddr[c] = dh * z;
    }
    if (t > 0) {
      fence_proxy_async_global();  // dgh_t stores -> visible to the TMA reads
      grid_arrive(bar);
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {  // gradient rows for the weight GEMMs: after the arrive
      if (!cv[c]) continue;
      const int j = cj[c];
      const int64_t s = (int64_t)ci[c] * a.T + t;
      uint16_t* gi_row = a.dgi + s * kGates;
      uint16_t* gh_row = a.dgh + s * kGates;
      gi_row[j] = dq[c][0];
      gi_row[kHidden + j] = dq[c][1];
      gi_row[2 * kHidden + j] = dq[c][3];
      gh_row[j] = dq[c][0];
      gh_row[kHidden + j] = dq[c][1];
      gh_row[2 * kHidden + j] = dq[c][2];
    }
    if (t == 0) break;  // d(h0) is not needed
    prefetch(t - 1);    // independent of the exchange: overlaps barrier + MMA
    if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[t * 4 + 1] = clock64();
    grid_wait(bar, base + ++epoch * NCTA_GB);
    if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[t * 4 + 2] = clock64();
    // the group's dgh_t: K block kb of quarter q = gates q*384 + kb*64, rows i0..i0+31
    if (warp == 1) {
      fence_proxy_async_global();
#pragma unroll
      for (int g = 0; g < 3; ++g) {
        sm100::mbar_arrive_expect_tx_warp(&kbar[g], 2 * GQ * GT * 128);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)
#pragma unroll
          for (int q = 0; q < GQ; ++q) {
            const int kb = 2 * g + kk;
            sm100::tma_load_3d_warp(tA + kb * G_KB + q * GT * 128, &a.xmap, &kbar[g],
                                    q * GKB_Q + kb * 64, i0, t & 1);
          }
      }
    }
    if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[t * 4 + 3] = clock64();
    if (warp == 0) {
      const uint32_t a0 = sm100::smem_u32(tA), b0 = sm100::smem_u32(tB);
      for (int g = 0; g < 3; ++g) {
        sm100::mbar_wait(&kbar[g], kphase);
        sm100::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // K16 steps of this group's two K blocks
          const int kb = 2 * g + (kk >> 2), k = kk & 3;
          const uint64_t ad = sm100::make_sdesc(a0 + kb * G_KB + k * 32, 16, 1024);
          const uint64_t bd = sm100::make_sdesc(b0 + kb * G_BN * 128 + k * 32, 16, 1024);
          sm100::umma_f16_warp(tmem, ad, bd, idesc, (g | kk) ? 1u : 0u);
        }
      }
      sm100::umma_commit_warp(mbar);
    }
    kphase ^= 1;
    sm100::mbar_wait(mbar, phase);
    phase ^= 1;
    sm100::tc_fence_after();
    if (warp < GQ) {  // quarter q = warp: TMEM lanes 32q.., diagonal columns 16q..16q+15
      uint32_t r[16];
      sm100::tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + UPC_GB * warp, r);
      sm100::tmem_ld_wait();
      float4* dst = reinterpret_cast<float4*>(mm + (warp * GT + lane) * MMS);
#pragma unroll
      for (int u = 0; u < UPC_GB / 4; ++u)
        dst[u] = make_float4(__uint_as_float(r[4 * u]), __uint_as_float(r[4 * u + 1]),
                             __uint_as_float(r[4 * u + 2]), __uint_as_float(r[4 * u + 3]));
    }
    sm100::tc_fence_before();
    __syncthreads();
  }
  // bias gradients of the CTA's gate columns: fixed-order sum over the group's
  // trajectories, then over the groups (the last CTA of a unit block adds the
  // groups' partials in group order -- deterministic)
  float* red = reinterpret_cast<float*>(tA);  // [32][16][4]
  __syncthreads();
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int e = tid + c * THR;
#pragma unroll
    for (int k = 0; k < 4; ++k) red[e * 4 + k] = cv[c] ? bsum[c][k] : 0.0f;
  }
  __syncthreads();
  __shared__ bool last;
  if (tid < UPC_GB * 4) {
    const int u = tid >> 2, k = tid & 3;
    float t = 0.0f;
    for (int i = 0; i < GT; ++i) t += red[(i * UPC_GB + u) * 4 + k];
    a.bpart[((size_t)grp * kHidden + j0 + u) * 4 + k] = t;
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    last = atomicAdd(a.pair + uc, 1u) == (unsigned)ngrp - 1;
  }
  __syncthreads();
  if (last && tid < UPC_GB * 4) {
    __threadfence();
    const int u = tid >> 2, k = tid & 3, j = j0 + u;
    float t = 0.0f;
    for (int g = 0; g < ngrp; ++g) t += __ldcg(a.bpart + ((size_t)g * kHidden + j) * 4 + k);
    if (k == 0) {
      a.gbih[j] = t;
      a.gbhh[j] = t;
    } else if (k == 1) {
      a.gbih[kHidden + j] = t;
      a.gbhh[kHidden + j] = t;
    } else if (k == 2) {
      a.gbih[2 * kHidden + j] = t;
    } else {
      a.gbhh[2 * kHidden + j] = t;
    }
  }
  if (last && tid == 0) a.pair[uc] = 0;  // re-arm for the next launch
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, 64);
  }
}

// Phase profiling of block 0 (env APPO_GRU_PROF=1; diagnostics only): clock64
// stamps per step, averaged and printed to stderr after a synchronize.
long long* prof_buffer(Ctx* c) {
  static long long* buf = nullptr;
  if (!getenv("APPO_GRU_PROF")) return nullptr;
  if (!buf && cudaMalloc(&buf, sizeof(long long) * 8 * 64) != cudaSuccess) return nullptr;
  cudaMemsetAsync(buf, 0, sizeof(long long) * 8 * 64, c->stream);
  return buf;
}
// forward stamps: 8 per step; prints the mean cycles of each phase
void prof_report8(Ctx* c, long long* d, int steps, const char* what) {
  long long h[8 * 64];
  cudaStreamSynchronize(c->stream);
  cudaMemcpy(h, d, sizeof(long long) * 8 * steps, cudaMemcpyDeviceToHost);
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int n = 0;
  for (int t = 0; t + 1 < steps; ++t) {
    const long long* a = h + 8 * t;
    if (!a[0] || !a[7] || !h[8 * (t + 1)]) continue;
    for (int k = 0; k < 7; ++k) acc[k] += a[k + 1] - a[k];
    acc[7] += h[8 * (t + 1)] - a[7];
    ++n;
  }
  fprintf(stderr, "[gru prof] %s (cycles/step, %d steps):", what, n);
  for (int k = 0; k < 8; ++k) fprintf(stderr, " %.0f", acc[k] / (n ? n : 1));
  fprintf(stderr, "\n");
}
void prof_report(Ctx* c, long long* d, int steps, const char* what) {
  long long h[4 * 64];
  cudaStreamSynchronize(c->stream);
  cudaMemcpy(h, d, sizeof(long long) * 4 * steps, cudaMemcpyDeviceToHost);
  double acc[4] = {0, 0, 0, 0};
  int n = 0;
  for (int t = 0; t + 1 < steps; ++t) {
    const long long* a = h + 4 * t;
    const long long* b = h + 4 * (t + 1);
    if (!a[0] || !b[0] || !a[1] || !a[3]) continue;
    // forward order: stamps 0..3 then next step's 0; backward steps run downwards
    const long long* nxt = strstr(what, "bwd") ? h + 4 * (t > 0 ? t - 1 : 0) : b;
    (void)nxt;
    acc[0] += a[1] - a[0];
    acc[1] += a[2] - a[1];
    acc[2] += a[3] - a[2];
    acc[3] += (strstr(what, "bwd") ? (t > 0 ? h[4 * (t - 1)] - a[3] : 0) : b[0] - a[3]);
    ++n;
  }
  fprintf(stderr, "[gru prof] %s (cycles/step, %d steps): %.0f %.0f %.0f %.0f\n", what, n,
          acc[0] / n, acc[1] / n, acc[2] / n, acc[3] / n);
}

}  // namespace

// module anchor for preload_library_kernels (slotq.cu)
const void* kanchor_gru() { return reinterpret_cast<const void*>(&gru_g_fwd_kernel); }

int gru_seq_supported(int n_traj) { return n_traj >= 1 && n_traj <= MAXTRAJ; }

namespace {
int gru_ws(Ctx* c) {
  if (c->d_gru_sync) return APPO_OK;
  APPO_CUDA_TRY(cudaMalloc(&c->d_gru_sync, sizeof(unsigned) * 64));
  APPO_CUDA_TRY(cudaMalloc(&c->d_gru_part, sizeof(float) * 4 * kHidden * 4));
  APPO_CUDA_TRY(cudaMemsetAsync(c->d_gru_sync, 0, sizeof(unsigned) * 64, c->stream));
  return APPO_OK;
}
// Cooperative launch (all CTAs co-resident for the step barriers) with
// programmatic stream serialisation when the context uses it
int launch_coop(Ctx* c, const void* kernel, int grid, int smem, void* arg) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THR);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = c->pdl ? 2 : 1;
  void* args[] = {arg};
  APPO_CUDA_TRY(cudaLaunchKernelExC(&cfg, kernel, args));
  return APPO_OK;
}
}  // namespace

int k_gru_seq_fwd(Ctx* c, int n_traj, int T, const float* gi, const uint16_t* whh,
                  const float* bhh, const uint8_t* done, float* hbuf, uint16_t* hbuf_bf,
                  float* core, uint16_t* core_bf, float* gates, float* hin, uint16_t* hbf) {
  APPO_TRY(gru_ws(c));
  APPO_TRY(ensure_smem_attr((const void*)gru_g_fwd_kernel, G_FWD_SMEM, c->device));
  const int ng = (n_traj + GT - 1) / GT;
  unsigned* gbar = c->d_gru_sync;
  GFwdArgs a{};
  for (int g = 0; g < ng; ++g) {  // this launch advances each group's counter by (T+1) NCTA_F
    a.base[g] = c->gru_epochs[g];
    c->gru_epochs[g] += (unsigned)(T + 1) * NCTA_F;
  }
  int st = make_tmap_bf16_3d(&a.hmap, hbuf_bf, kHidden, n_traj, 2, kHidden * 2,
                             (uint64_t)n_traj * kHidden * 2, 64, GT, 1);
  if (st) return st;
  a.n_traj = n_traj; a.T = T; a.gi = gi; a.whh = whh; a.bhh = bhh; a.done = done;
  a.hbuf = hbuf; a.hbuf_bf = hbuf_bf; a.core = core; a.core_bf = core_bf; a.gates = gates;
  a.hin = hin; a.hbf = hbf; a.bar = gbar; a.prof = prof_buffer(c);
  cudaEvent_t ev = timing_begin(c, "gru_seq_fwd_kernel");
  APPO_TRY(launch_coop(c, (const void*)gru_g_fwd_kernel, NCTA_F * ng, G_FWD_SMEM, &a));
  c->next_flops = 2.0 * n_traj * (double)kGates * kHidden * (T + 1);
  timing_end(c, "gru_seq_fwd_kernel", ev);
  c->launches++;
  if (a.prof)
    prof_report8(c, a.prof, T + 1,
                 "fwd: tma+mma issue | mma wait | tmem->smem | cell+xchg store | proxy fence | "
                 "arrive | outputs | prefetch+barrier wait");
  return APPO_OK;
}

int k_gru_seq_bwd(Ctx* c, int n_traj, int T, const float* dcore, const uint8_t* done,
                  const float* gates, const float* hin, const uint16_t* whh, uint16_t* dghx,
                  uint16_t* dgi, uint16_t* dgh, float* gbih, float* gbhh) {
  APPO_TRY(gru_ws(c));
  APPO_TRY(ensure_smem_attr((const void*)gru_g_bwd_kernel, G_BWD_SMEM, c->device));
  const int ng = (n_traj + GT - 1) / GT;
  unsigned* gbar = c->d_gru_sync + 4;
  GBwdArgs a{};
  for (int g = 0; g < ng; ++g) {  // T-1 step barriers of NCTA_GB arrivals
    a.base[g] = c->gru_epochs[4 + g];
    c->gru_epochs[4 + g] += (unsigned)(T > 1 ? T - 1 : 0) * NCTA_GB;
  }
  int st = make_tmap_bf16_3d(&a.xmap, dghx, kGates, n_traj, 2, kGates * 2,
                             (uint64_t)n_traj * kGates * 2, 64, GT, 1);
  if (st) return st;
  a.n_traj = n_traj; a.T = T; a.dcore = dcore; a.done = done; a.gates = gates; a.hin = hin;
  a.whh = whh; a.dghx = dghx; a.dgi = dgi; a.dgh = dgh; a.gbih = gbih; a.gbhh = gbhh;
  a.bar = gbar; a.pair = c->d_gru_sync + 32; a.bpart = c->d_gru_part; a.prof = prof_buffer(c);
  cudaEvent_t ev = timing_begin(c, "gru_seq_bwd_kernel");
  APPO_TRY(launch_coop(c, (const void*)gru_g_bwd_kernel, NCTA_GB * ng, G_BWD_SMEM, &a));
  c->next_flops = 2.0 * n_traj * (double)kGates * kHidden * (T - 1);
  timing_end(c, "gru_seq_bwd_kernel", ev);
  c->launches++;
  if (a.prof) prof_report(c, a.prof, T, "bwd: cell | barrier | stage | mma");
  return APPO_OK;
}

}  // namespace appo_b200
