// Persistent GRU recurrence for the learner: the T-step forward unroll (+ the
// bootstrap step) and the BPTT reverse sweep each run as ONE cooperative
// kernel; the per-step recurrent product runs on tcgen05.
//
//   forward : 32 CTAs x 16 hidden units.  D[i][g] = sum_k h_t[i][k] W_hh[g][k]
//             over the CTA's 48 gate rows (r, z, n of its units): UMMA M=64
//             (trajectories) x N=48 x K=512, B = W slice resident in smem
//             (bf16, SW128 K-major), A = h_t staged from global each step.
//             The epilogue applies the cell (PyTorch r,z,n; oracle gru_fwd)
//             for the CTA's units; the only cross-CTA traffic is h_{t+1}
//             (64 x 512 bf16, L2-resident) behind one grid barrier per step.
//   backward: 64 CTAs x 8 units.  Gate gradients for own units (oracle
//             orc_learner_step BPTT) are published as dgh_t (64 x 1536 bf16);
//             after the barrier dnext[i][j] = dh*z + sum_g dgh_t[i][g] W_hh[g][j]
//             as UMMA M=64 x N=8 x K=1536 with W_hh[:, own]^T resident and all
//             of dgh_t staged at once (three 64 KB K chunks).
// Staging uses cp.async (16 B, L2-only) straight into the swizzled tile, so a
// step costs one L2 round trip + one UMMA chain + one barrier.  Per-cell state
// (h, b_hh, prefetched next-step inputs, dh*z) lives in registers because a
// thread owns the same (trajectory, unit) cells every step.
// TMEM layout for M=64 (cta_group::1): row m lives in lane (m % 16) + 32*(m/16)
// (CuTe "half subpartitions" atom, mma_traits_sm100.hpp), so warp w's lanes
// 0..15 hold rows 16w..16w+15.
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

constexpr int MAXTRAJ = 64;                // UMMA M
constexpr int THR = 256;
constexpr int KB_BYTES_A = MAXTRAJ * 128;  // one 64-wide K block of a 64-row A tile
constexpr int A_TILE = 8 * KB_BYTES_A;     // 64 x 512 bf16 = 64 KB

constexpr int UPC_F = 16;                  // forward: units per CTA
constexpr int NCTA_F = kHidden / UPC_F;    // 32
constexpr int NG = 3 * UPC_F;              // 48 gate rows per CTA (forward N)
constexpr int B_FWD = 8 * NG * 128;        // 48 x 512 bf16 = 48 KB

constexpr int UPC_B = 8;                   // backward: units per CTA (UMMA N)
constexpr int NCTA_B = kHidden / UPC_B;    // 64
constexpr int B_BWD = 24 * UPC_B * 128;    // 8 x 1536 bf16 = 24 KB

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

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// byte offset of 16-byte chunk c (8 bf16) of row r, K block kb in a K-major
// SW128 tile whose K blocks hold `rows` rows each
__device__ __forceinline__ uint32_t sw128(int rows, int r, int kb, int c) {
  return (uint32_t)(kb * rows * 128 + r * 128 + ((c ^ (r & 7)) << 4));
}

// Grid-wide barrier on a monotonically increasing counter (zeroed by the host
// before the launch); all CTAs are co-resident (cooperative launch).
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
    } while (v < target);
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
    } while (v < target);
  }
  __syncthreads();
}

// Issue cp.async copies of rows [n_rows] x 512 bf16 (global row stride ld
// elements, from column col0) into a 64-row SW128 K-major tile; rows >=
// n_rows are zero-filled.  Caller commits / waits.
__device__ __forceinline__ void stage_async(uint8_t* tile, const uint16_t* src, int n_rows,
                                            int64_t ld, int col0) {
  constexpr int CH = MAXTRAJ * 64;  // 16-byte chunks in 64 x 512
  const uint32_t base = sm100::smem_u32(tile);
#pragma unroll 4
  for (int e = threadIdx.x; e < CH; e += THR) {
    const int r = e >> 6, c = e & 63;
    const bool ok = r < n_rows;
    const uint16_t* g = src + (int64_t)(ok ? r : 0) * ld + col0 + c * 8;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                     base + sw128(MAXTRAJ, r, c >> 3, c & 7)),
                 "l"(g), "r"(ok ? 16 : 0)
                 : "memory");
  }
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

struct FwdArgs {
  CUtensorMap hmap;      // 3-D map over hbuf_bf {512, n_traj, 2}, box {64, 64, 1}, SW128
  int n_traj, T;
  const float* gi;       // [R][1536] (x W_ih^T + b_ih), rows s = i*T+t, boot rows B+i
  const uint16_t* whh;   // bf16 [1536][512] (published copy of the master)
  const float* bhh;      // [1536]
  const uint8_t* done;   // [B]
  float* hbuf;           // [n_traj][512] fp32 h0 on entry
  uint16_t* hbuf_bf;     // [2][n_traj][512] bf16 ping-pong h_t (exchange)
  float* core;           // [R][512]
  uint16_t* core_bf;     // [R][512]
  float* gates;          // [R][4][512]
  float* hin;            // [R][512]
  uint16_t* hbf;         // [R][512]
  unsigned* bar;
  long long* prof;       // optional phase timestamps (APPO_GRU_PROF): [steps][4]
};

// per-step phase stamps of block 0 (APPO_GRU_PROF=1 diagnostics), 8 per step
#define FSTAMP(k)                                                     \
  do {                                                                \
    if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[t * 8 + (k)] = clock64(); \
  } while (0)
__global__ void __launch_bounds__(THR, 1) gru_seq_fwd_kernel(const __grid_constant__ FwdArgs a) {
  APPO_PDL_ENTRY();
  extern __shared__ uint8_t smraw[];
  // 1024-B aligned base.  Generic (integer round trip) addressing is kept on
  // purpose: the LDS/STS form measured slower (GRU forward 138 -> 163 us, same
  // box A/B, scripts/gpu_ab.sh)
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* tA = sm;
  uint8_t* tB = sm + A_TILE;
  // h_t . W_hh[own gates]^T as one M=128 chain over the two K halves: rows =
  // (trajectory, half), N = (gate row, half); the diagonal blocks are the two
  // partial sums (half the MMA instructions of an M=64 chain)
  float* gh = reinterpret_cast<float*>(tB + B_FWD);              // [64][NG] K half 0
  float* gh2 = gh + MAXTRAJ * NG;                                 // [64][NG] K half 1
  uint64_t* mbar = reinterpret_cast<uint64_t*>(gh2 + MAXTRAJ * NG);
  uint64_t* kbar = mbar + 1;  // [8] one per staged K block of h_t
  uint32_t* tslot = reinterpret_cast<uint32_t*>(kbar + 8);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int j0 = blockIdx.x * UPC_F;
  const int B = a.n_traj * a.T;

  // resident B operand (2 NG rows x 256): row n + NG h = gate row n = g*16 + u
  // (g in r,z,n) -> W_hh row g*512 + j0 + u, columns h*256 ..
  for (int e = tid; e < 2 * NG * 32; e += THR) {
    const int nn = e >> 5, c = e & 31;  // 16-byte chunk c of the half
    const int n = nn % NG, h = nn / NG;
    const int grow = (n / UPC_F) * kHidden + j0 + (n % UPC_F);
    *reinterpret_cast<uint4*>(tB + sw128(2 * NG, nn, c >> 3, c & 7)) =
        reinterpret_cast<const uint4*>(a.whh + (int64_t)grow * kHidden)[h * 32 + c];
  }
  if (tid == 0) {
    sm100::mbar_init(mbar, 1);
    for (int k = 0; k < 8; ++k) sm100::mbar_init(&kbar[k], 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) {
    sm100::tmem_alloc(tslot, 128);
    sm100::tmem_relinquish();
  }
  // Per-thread cells (trajectory i, own unit u) are fixed across steps.
  constexpr int CPT = MAXTRAJ * UPC_F / THR;  // 4
  const int n_cells = a.n_traj * UPC_F;
  float hreg[CPT], b3[CPT][3], g3[CPT][3];
  uint8_t dn[CPT];
  auto prefetch = [&](int t) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int e = tid + c * THR;
      if (e < n_cells) {
        const int i = e / UPC_F, j = j0 + e % UPC_F;
        const int64_t row = (t < a.T) ? (int64_t)i * a.T + t : (int64_t)B + i;
        const float* gir = a.gi + row * kGates;
        g3[c][0] = __ldg(gir + j);
        g3[c][1] = __ldg(gir + kHidden + j);
        g3[c][2] = __ldg(gir + 2 * kHidden + j);
        dn[c] = (t < a.T) ? a.done[(int64_t)i * a.T + t] : 0;
      }
    }
  };
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int e = tid + c * THR;
    if (e < n_cells) {
      const int i = e / UPC_F, j = j0 + e % UPC_F;
      hreg[c] = a.hbuf[(int64_t)i * kHidden + j];
      a.hbuf_bf[(int64_t)i * kHidden + j] = f2bf_(hreg[c]);  // first h_t, own columns
      b3[c][0] = a.bhh[j];
      b3[c][1] = a.bhh[kHidden + j];
      b3[c][2] = a.bhh[2 * kHidden + j];
    }
  }
  prefetch(0);
  fence_proxy_async_global();  // h0 stores -> visible to the TMA (async proxy) reads
  sm100::tc_fence_before();
  grid_barrier(a.bar, gridDim.x);  // h0 bf16 complete everywhere
  sm100::tc_fence_after();
  const uint32_t tmem = *tslot;
  constexpr uint32_t idesc = sm100::make_idesc_bf16(2 * MAXTRAJ, 2 * NG, 0, 0);
  unsigned epoch = 1;
  uint32_t phase = 0;

  for (int t = 0; t <= a.T; ++t) {
    FSTAMP(0);
    const size_t nxt = (size_t)((t + 1) & 1) * a.n_traj * kHidden;
    // h_t (written by every CTA before the barrier) -> smem by TMA, one K block
    // per mbarrier so the MMAs start on the first block while the rest land
    if (warp == 1) {
      fence_proxy_async_global();
#pragma unroll
      for (int q = 0; q < 8; ++q) {  // K block kb = q >> 1 of half q & 1 (h_t columns 64 q')
        const int kb = q >> 1, h = q & 1, col = (h * 4 + kb) * 64;
        sm100::mbar_arrive_expect_tx_warp(&kbar[q], KB_BYTES_A);
        sm100::tma_load_3d_warp(tA + kb * 2 * KB_BYTES_A + h * KB_BYTES_A, &a.hmap, &kbar[q], col,
                                0, t & 1);
      }
    }
    if (warp == 0) {  // whole warp: elect.sync inside (no per-MMA waterfall)
      const uint32_t a0 = sm100::smem_u32(tA), b0 = sm100::smem_u32(tB);
#pragma unroll
      for (int kb = 0; kb < 4; ++kb) {
        sm100::mbar_wait(&kbar[2 * kb], t & 1);
        sm100::mbar_wait(&kbar[2 * kb + 1], t & 1);
        sm100::tc_fence_after();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = sm100::make_sdesc(a0 + kb * 2 * KB_BYTES_A + k * 32, 16, 1024);
          const uint64_t bd = sm100::make_sdesc(b0 + kb * 2 * NG * 128 + k * 32, 16, 1024);
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
    if (warp < 4) {  // M=128 accumulator: TMEM lane = row = trajectory + 64 * half
      uint32_t r[NG];
      const int row = 32 * warp + lane;
      float* dst = warp < 2 ? gh + row * NG : gh2 + (row - MAXTRAJ) * NG;
      const int c0 = warp < 2 ? 0 : NG;  // diagonal block of the row's K half
      // all three column blocks in flight, one wait
#pragma unroll
      for (int cb = 0; cb < NG; cb += 16)
        sm100::tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0 + cb,
                         *reinterpret_cast<uint32_t(*)[16]>(r + cb));
      sm100::tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < NG; ++q) dst[q] = __uint_as_float(r[q]);
    }
    sm100::tc_fence_before();
    __syncthreads();
    FSTAMP(3);
    // the cell; only the exchange (next h, bf16) is stored before the barrier
    // arrive -- the rest of the step's outputs are stored while it completes
    float cv[CPT][6];  // r, z, n, ghn, h_prev, h
    // every cell's gate pre-activations first: the exchange stores below may
    // not be reordered above these (generic addressing), so loading them per
    // cell would serialise the cells
    float ghv[CPT][3];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int e = tid + c * THR;
      const int i = (e < n_cells ? e : 0) / UPC_F, u = e % UPC_F;
#pragma unroll
      for (int g = 0; g < 3; ++g)
        ghv[c][g] = (gh[i * NG + g * UPC_F + u] + gh2[i * NG + g * UPC_F + u]) + b3[c][g];
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int e = tid + c * THR;
      if (e >= n_cells) continue;
      const int i = e / UPC_F, u = e % UPC_F, j = j0 + u;
      const float ghr = ghv[c][0];
      const float ghz = ghv[c][1];
      const float ghn = ghv[c][2];
      const float rr = sig_(g3[c][0] + ghr);
      const float z = sig_(g3[c][1] + ghz);
      const float n = tanh_(g3[c][2] + rr * ghn);
      const float hp = hreg[c];
      const float h = (1.0f - z) * n + z * hp;
      cv[c][0] = rr;
      cv[c][1] = z;
      cv[c][2] = n;
      cv[c][3] = ghn;
      cv[c][4] = hp;
      cv[c][5] = h;
      if (t < a.T) {
        const float hn = dn[c] ? 0.0f : h;
        hreg[c] = hn;
        a.hbuf_bf[nxt + (int64_t)i * kHidden + j] = f2bf_(hn);
      }
    }
    FSTAMP(4);
    if (t < a.T) {
      fence_proxy_async_global();
      FSTAMP(5);
      grid_arrive(a.bar);
    }
    FSTAMP(6);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int e = tid + c * THR;
      if (e >= n_cells) continue;
      const int i = e / UPC_F, j = j0 + e % UPC_F;
      const int64_t row = (t < a.T) ? (int64_t)i * a.T + t : (int64_t)B + i;
      a.core[row * kHidden + j] = cv[c][5];
      a.core_bf[row * kHidden + j] = f2bf_(cv[c][5]);
      float* gs = a.gates + row * 4 * kHidden;
      gs[j] = cv[c][0];
      gs[kHidden + j] = cv[c][1];
      gs[2 * kHidden + j] = cv[c][2];
      gs[3 * kHidden + j] = cv[c][3];
      a.hin[row * kHidden + j] = cv[c][4];
      a.hbf[row * kHidden + j] = f2bf_(cv[c][4]);
    }
    FSTAMP(7);
    if (t < a.T) {
      prefetch(t + 1);  // independent of the exchange: overlaps the barrier
      grid_wait(a.bar, ++epoch * gridDim.x);
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, 128);
  }
}

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
constexpr int G_FWD_SMEM = 1024 + G_A + G_B + GQ * GT * NG * 4 + 64;

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
  long long* prof;
};

__global__ void __launch_bounds__(THR, 1) gru_g_fwd_kernel(const __grid_constant__ GFwdArgs a) {
  APPO_PDL_ENTRY();
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* tA = sm;
  uint8_t* tB = sm + G_A;
  float* gq = reinterpret_cast<float*>(tB + G_B);                 // [GQ][GT][NG] partial sums
  uint64_t* mbar = reinterpret_cast<uint64_t*>(gq + GQ * GT * NG);
  uint64_t* kbar = mbar + 1;  // [2] one per K block (all four quarters of it)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(kbar + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = blockIdx.x / NCTA_F, uc = blockIdx.x % NCTA_F;
  const int j0 = uc * UPC_F, i0 = grp * GT;
  const int B = a.n_traj * a.T;
  unsigned* bar = a.bar + grp;

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
  grid_barrier(bar, NCTA_F);  // the group's h0 (bf16) complete
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
      float* dst = gq + (warp * GT + lane) * NG;
#pragma unroll
      for (int q = 0; q < NG; ++q) dst[q] = __uint_as_float(r[q]);
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
        ghv[c][g] = ((gq[(0 * GT + cl[c]) * NG + n] + gq[(1 * GT + cl[c]) * NG + n]) +
                     (gq[(2 * GT + cl[c]) * NG + n] + gq[(3 * GT + cl[c]) * NG + n])) +
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
      grid_wait(bar, ++epoch * NCTA_F);
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, 256);
  }
}

struct BwdArgs {
  CUtensorMap xmap;     // 3-D map over dghx {1536, n_traj, 2}, box {64, 64, 1}, SW128
  int n_traj, T;
  const float* dcore;   // [B][512]
  const uint8_t* done;  // [B]
  const float* gates;   // [R][4][512]
  const float* hin;     // [R][512]
  const uint16_t* whh;  // bf16 [1536][512]
  uint16_t* dghx;       // [2][n_traj][1536] bf16 exchange
  uint16_t* dgi;        // [B][1536]
  uint16_t* dgh;        // [B][1536]
  float* gbih;          // [1536] bias gradients (sums over all B rows)
  float* gbhh;          // [1536]
  unsigned* bar;
  long long* prof;      // optional phase timestamps (APPO_GRU_PROF): [steps][4]
  int mc;               // 1: launched in CTA pairs, dgh_t staged by TMA multicast
};

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
constexpr int G_BWD_SMEM = 1024 + G_BA + G_BB + GQ * GT * UPC_GB * 4 + 64;

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
  unsigned* pair;       // [NCTA_GB] bias-gradient combine counters (self-resetting)
  float* bpart;         // [groups][512][4] per-group bias partial sums
  long long* prof;
};

__global__ void __launch_bounds__(THR, 1) gru_g_bwd_kernel(const __grid_constant__ GBwdArgs a) {
  APPO_PDL_ENTRY();
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* tA = sm;
  uint8_t* tB = sm + G_BA;
  float* mm = reinterpret_cast<float*>(tB + G_BB);          // [GQ][GT][16] partial sums
  uint64_t* mbar = reinterpret_cast<uint64_t*>(mm + GQ * GT * UPC_GB);
  uint64_t* kbar = mbar + 1;  // [3] one per two K blocks (32 KB)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(kbar + 3);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = blockIdx.x / NCTA_GB, uc = blockIdx.x % NCTA_GB;
  const int j0 = uc * UPC_GB, i0 = grp * GT;
  unsigned* bar = a.bar + grp;
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
              : ddr[c] + ((mm[(0 * GT + cl[c]) * UPC_GB + u] + mm[(1 * GT + cl[c]) * UPC_GB + u]) +
                          (mm[(2 * GT + cl[c]) * UPC_GB + u] + mm[(3 * GT + cl[c]) * UPC_GB + u]));
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
    grid_wait(bar, ++epoch * NCTA_GB);
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
      float* dst = mm + (warp * GT + lane) * UPC_GB;
#pragma unroll
      for (int u = 0; u < UPC_GB; ++u) dst[u] = __uint_as_float(r[u]);
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

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__global__ void __launch_bounds__(THR, 1) gru_seq_bwd_kernel(const __grid_constant__ BwdArgs a) {
  APPO_PDL_ENTRY();
  extern __shared__ uint8_t smraw[];
  // 1024-B aligned base.  Generic (integer round trip) addressing is kept on
  // purpose: the LDS/STS form measured slower (GRU forward 138 -> 163 us, same
  // box A/B, scripts/gpu_ab.sh)
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* tA = sm;                                      // 3 x 64 KB: all of dgh_t
  uint8_t* tB = sm + 3 * A_TILE;
  // dgh_t . W_hh[:, own] as two K halves: one M=128 MMA chain whose rows are
  // (trajectory, half) and whose N = (unit, half); the diagonal blocks are the
  // two partial sums (half the MMA instructions of an M=64, N=8 chain)
  float* mm = reinterpret_cast<float*>(tB + B_BWD);      // [64][8] K half 0
  float* mm2 = mm + MAXTRAJ * UPC_B;                     // [64][8] K half 1
  uint64_t* mbar = reinterpret_cast<uint64_t*>(mm2 + MAXTRAJ * UPC_B);
  uint64_t* kbar = mbar + 1;  // [6] one per 4 staged K blocks (32 KB) of dgh_t
  uint32_t* tslot = reinterpret_cast<uint32_t*>(kbar + 6);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int j0 = blockIdx.x * UPC_B;

  // resident B (K-major, 16 rows x 768): row n = u + 8 h, K = k':
  // B[n][k'] = W_hh[h * 768 + k'][j0 + u]
  for (int e = tid; e < 2 * UPC_B * (kGates / 16); e += THR) {
    const int n = e / (kGates / 16), c8 = e % (kGates / 16);  // chunk of 8 gates
    const int u = n & (UPC_B - 1), h = n / UPC_B;
    uint32_t w[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int g = h * (kGates / 2) + c8 * 8 + 2 * p;
      w[p] = (uint32_t)a.whh[(int64_t)g * kHidden + j0 + u] |
             ((uint32_t)a.whh[(int64_t)(g + 1) * kHidden + j0 + u] << 16);
    }
    *reinterpret_cast<uint4*>(tB + sw128(2 * UPC_B, n, c8 >> 3, c8 & 7)) =
        make_uint4(w[0], w[1], w[2], w[3]);
  }
  if (tid == 0) {
    sm100::mbar_init(mbar, 1);
    for (int k = 0; k < 6; ++k) sm100::mbar_init(&kbar[k], 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) {
    sm100::tmem_alloc(tslot, 32);
    sm100::tmem_relinquish();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tslot;
  constexpr uint32_t idesc = sm100::make_idesc_bf16(2 * MAXTRAJ, 2 * UPC_B, 0, 0);
  unsigned epoch = 0;
  uint32_t phase = 0, kphase = 0;

  constexpr int CPT = MAXTRAJ * UPC_B / THR;  // 2 cells per thread
  const int n_cells = a.n_traj * UPC_B;
  float pf[CPT][7];  // dcore, r, z, n, ghn, h_in, keep
  float ddr[CPT];    // dh*z of the later step
  float bsum[CPT][4];  // per-cell sums over t of dgr, dgz, dan, dgn (bias gradients)
#pragma unroll
  for (int c = 0; c < CPT; ++c) bsum[c][0] = bsum[c][1] = bsum[c][2] = bsum[c][3] = 0.0f;
  auto prefetch = [&](int t) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int e = tid + c * THR;
      if (e < n_cells) {
        const int i = e / UPC_B, j = j0 + e % UPC_B;
        const int64_t s = (int64_t)i * a.T + t;
        const float* gs = a.gates + s * 4 * kHidden;
        pf[c][0] = __ldg(a.dcore + s * kHidden + j);
        pf[c][1] = __ldg(gs + j);
        pf[c][2] = __ldg(gs + kHidden + j);
        pf[c][3] = __ldg(gs + 2 * kHidden + j);
        pf[c][4] = __ldg(gs + 3 * kHidden + j);
        pf[c][5] = __ldg(a.hin + s * kHidden + j);
        pf[c][6] = a.done[s] ? 0.0f : 1.0f;
      }
    }
  };
  prefetch(a.T - 1);

  for (int t = a.T - 1; t >= 0; --t) {
    if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[t * 4 + 0] = clock64();
    uint16_t* xb = a.dghx + (size_t)(t & 1) * a.n_traj * kGates;
    uint16_t dq[CPT][4];  // dgr, dgz, dgn, dan (bf16) of this step's cells
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int e = tid + c * THR;
      if (e >= n_cells) continue;
      const int i = e / UPC_B, u = e % UPC_B, j = j0 + u;
      const int64_t s = (int64_t)i * a.T + t;
      const float dnext =
          (t == a.T - 1) ? 0.0f : ddr[c] + (mm[i * UPC_B + u] + mm2[i * UPC_B + u]);
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
      grid_arrive(a.bar);
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {  // gradient rows for the weight GEMMs: after the arrive
      const int e = tid + c * THR;
      if (e >= n_cells) continue;
      const int i = e / UPC_B, j = j0 + e % UPC_B;
      const int64_t s = (int64_t)i * a.T + t;
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
    grid_wait(a.bar, ++epoch * gridDim.x);
    if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[t * 4 + 2] = clock64();
    // dnext = dh*z + dgh_t . W_hh[:, own]: dgh_t (24 K blocks of 8 KB) by TMA in
    // six 32 KB groups; the MMAs of a group start as soon as it lands
    if (warp == 1) {
      fence_proxy_async_global();
      if (a.mc) {
        // CTA pair: each CTA fetches every other 32 KB group once for both
        // (multicast into the same smem offsets, completing both CTAs' kbar[g]);
        // the peer finished reading its tA (previous step's MMAs) before the barrier
        const uint32_t rank = cluster_rank();
#pragma unroll
        for (int g = 0; g < 6; ++g) sm100::mbar_arrive_expect_tx_warp(&kbar[g], 4 * KB_BYTES_A);
        if (lane == 0) {
#pragma unroll
          for (int g = 0; g < 6; ++g) {
            if ((uint32_t)(g & 1) != rank) continue;
#pragma unroll
            for (int q = 0; q < 4; ++q)  // K block 2g + (q >> 1) of half q & 1
              sm100::tma_load_3d_mc(tA + (2 * g + (q >> 1)) * 2 * KB_BYTES_A + (q & 1) * KB_BYTES_A,
                                    &a.xmap, &kbar[g], (q & 1) * (kGates / 2) + (2 * g + (q >> 1)) * 64,
                                    0, t & 1, (uint16_t)0x3);
          }
        }
        __syncwarp();
      } else {
#pragma unroll
        for (int g = 0; g < 6; ++g) {
          sm100::mbar_arrive_expect_tx_warp(&kbar[g], 4 * KB_BYTES_A);
#pragma unroll
          for (int q = 0; q < 4; ++q)  // K block 2g + (q >> 1) of half q & 1: rows 64 (q & 1)..
            sm100::tma_load_3d_warp(tA + (2 * g + (q >> 1)) * 2 * KB_BYTES_A + (q & 1) * KB_BYTES_A,
                                    &a.xmap, &kbar[g],
                                    (q & 1) * (kGates / 2) + (2 * g + (q >> 1)) * 64, 0, t & 1);
        }
      }
    }
    if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[t * 4 + 3] = clock64();
    if (warp == 0) {  // whole warp: elect.sync inside (no per-MMA waterfall)
      const uint32_t a0 = sm100::smem_u32(tA), b0 = sm100::smem_u32(tB);
      for (int g = 0; g < 6; ++g) {
        sm100::mbar_wait(&kbar[g], kphase);
        sm100::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // K16 steps of this group's two 128-row K blocks
          const int kg = 8 * g + kk;        // K16 step in the 768-wide half
          const uint64_t ad =
              sm100::make_sdesc(a0 + (kg >> 2) * 2 * KB_BYTES_A + (kg & 3) * 32, 16, 1024);
          const uint64_t bd =
              sm100::make_sdesc(b0 + (kg >> 2) * 2 * UPC_B * 128 + (kg & 3) * 32, 16, 1024);
          sm100::umma_f16_warp(tmem, ad, bd, idesc, kg > 0 ? 1u : 0u);
        }
      }
      sm100::umma_commit_warp(mbar);
    }
    kphase ^= 1;
    sm100::mbar_wait(mbar, phase);
    phase ^= 1;
    sm100::tc_fence_after();
    if (warp < 4) {  // M=128 accumulator: TMEM lane = row = trajectory + 64 * half
      uint32_t r[16];
      sm100::tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16), r);
      sm100::tmem_ld_wait();
      const int row = 32 * warp + lane;
      float* dst = warp < 2 ? mm + row * UPC_B : mm2 + (row - MAXTRAJ) * UPC_B;
      const int c0 = warp < 2 ? 0 : UPC_B;  // diagonal block of the row's K half
#pragma unroll
      for (int u = 0; u < UPC_B; ++u) dst[u] = __uint_as_float(r[c0 + u]);
    }
    sm100::tc_fence_before();
    __syncthreads();
  }
  // bias gradients of the CTA's gate columns: fixed-order sum over trajectories
  // (the A staging tile is free now: every MMA has completed)
  float* red = reinterpret_cast<float*>(tA);  // [64][8][4]
  __syncthreads();
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int e = tid + c * THR;
    if (e < n_cells)
#pragma unroll
      for (int k = 0; k < 4; ++k) red[e * 4 + k] = bsum[c][k];
  }
  __syncthreads();
  if (tid < UPC_B * 4) {
    const int u = tid >> 2, k = tid & 3;
    float t = 0.0f;
    for (int i = 0; i < a.n_traj; ++i) t += red[(i * UPC_B + u) * 4 + k];
    const int j = j0 + u;
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
  sm100::tc_fence_before();
  __syncthreads();
  if (a.mc) sm100::cluster_sync();  // no CTA leaves while its pair may still multicast into it
  if (warp == 0) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, 32);
  }
}

// ---- forward recurrence in ONE 16-CTA cluster -------------------------------
// CTA c owns units 32c..32c+31 (gate rows g*32+u: UMMA N = 96, W_hh slice
// resident, SW128).  h_t is exchanged without any grid barrier: every CTA
// writes its 64 x 32 bf16 slice to global and multicasts it by TMA (SW64 box =
// exactly its K block of the A operand) into the h buffer of all 16 CTAs,
// double-buffered by step parity; per-slice mbarriers (complete_tx) tell the
// MMA warp which K blocks have landed.  A CTA multicasts h_{t+1} only after its
// MMA(t), which needed every CTA's h_t -- so buffer (t+1)&1 (last read by the
// MMAs of step t-1) is free everywhere, and the per-buffer barriers are re-armed
// right after MMA(t-1) completes, before any byte of step t+1 can arrive.
// Cells are read straight from TMEM (16x256b: all 32 lanes busy), 4 per thread.
constexpr int CL_CTAS = 16;
constexpr int CL_UPC = kHidden / CL_CTAS;      // 32 units per CTA
constexpr int CL_NG = 3 * CL_UPC;              // 96 gate rows
constexpr int CL_THR = 512;
constexpr int CL_B = 8 * CL_NG * 128;          // W slice: 8 K blocks x 96 rows x 128 B = 96 KB
constexpr int CL_KB = 4096;                    // one SW64 K block of h: 64 rows x 64 B
constexpr int CL_A = CL_CTAS * CL_KB;          // 64 KB
constexpr int CL_SMEM = 1024 + CL_B + 2 * CL_A + (2 * CL_CTAS + 1) * 8 + 16;

struct ClFwdArgs {
  CUtensorMap xmap;      // 3-D map over xbuf {512, n_traj, 2}, box {32, 64, 1}, SW64
  int n_traj, T;
  const float* gi;       // [R][1536]
  const uint16_t* whh;   // bf16 [1536][512]
  const float* bhh;      // [1536]
  const uint8_t* done;   // [B]
  const float* h0;       // [n_traj][512]
  uint16_t* xbuf;        // [2][n_traj][512] bf16 exchange
  float* core;
  uint16_t* core_bf;
  float* gates;
  float* hin;
  uint16_t* hbf;
  long long* prof;
};

__global__ void __cluster_dims__(CL_CTAS, 1, 1) __launch_bounds__(CL_THR, 1)
    gru_cl_fwd_kernel(const __grid_constant__ ClFwdArgs a) {
  APPO_PDL_ENTRY();
  extern __shared__ uint8_t smraw[];
  // 1024-B aligned base.  Generic (integer round trip) addressing is kept on
  // purpose: the LDS/STS form measured slower (GRU forward 138 -> 163 us, same
  // box A/B, scripts/gpu_ab.sh)
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* tB = sm;                 // W slice (SW128 K-major)
  uint8_t* tA = sm + CL_B;          // [2][16 K blocks][64 rows][64 B] (SW64 K-major)
  uint64_t* kbar = reinterpret_cast<uint64_t*>(tA + 2 * CL_A);  // [2][16]
  uint64_t* mbar = kbar + 2 * CL_CTAS;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = blockIdx.x;  // == rank in the (single) cluster
  const int j0 = cta * CL_UPC;
  const int B = a.n_traj * a.T;

  // resident B operand: row n = g*32 + u -> W_hh row g*512 + j0 + u
  for (int e = tid; e < CL_NG * 64; e += CL_THR) {
    const int n = e >> 6, c = e & 63;
    const int grow = (n / CL_UPC) * kHidden + j0 + (n % CL_UPC);
    *reinterpret_cast<uint4*>(tB + sw128(CL_NG, n, c >> 3, c & 7)) =
        reinterpret_cast<const uint4*>(a.whh + (int64_t)grow * kHidden)[c];
  }
  if (tid == 0) {
    for (int k = 0; k < 2 * CL_CTAS; ++k) sm100::mbar_init(&kbar[k], 1);
    sm100::mbar_init(mbar, 1);
    sm100::fence_barrier_init();
    // arm the slice barriers of steps 0 and 1
    for (int k = 0; k < 2 * CL_CTAS; ++k) sm100::mbar_arrive_expect_tx(&kbar[k], CL_KB);
  }
  if (warp == 0) {
    sm100::tmem_alloc(tslot, 128);
    sm100::tmem_relinquish();
  }
  // TMEM readout: warp w -> lane quarter sp = w % 4 (rows 16sp..16sp+15), unit
  // group ug = w / 4; the gate pre-activations go through shared memory (the
  // consumed h buffer) so that cells map to threads as (row, unit) with
  // consecutive units per warp: every global store is a coalesced 128-B row.
  const int sp = warp & 3, ug = warp >> 2;
  const int ti0 = 16 * sp + (lane >> 2), tu0 = 8 * ug + 2 * (lane & 3);
  int ci[4], cj[4];
  bool cv[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int e = tid + c * CL_THR;
    ci[c] = e / CL_UPC;
    cj[c] = j0 + e % CL_UPC;
    cv[c] = ci[c] < a.n_traj;
  }
  float hreg[4], b3[4][3], g3[4][3];
  uint8_t dn[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    hreg[c] = cv[c] ? a.h0[(int64_t)ci[c] * kHidden + cj[c]] : 0.0f;
#pragma unroll
    for (int g = 0; g < 3; ++g) b3[c][g] = a.bhh[g * kHidden + cj[c]];
    if (cv[c]) a.xbuf[(int64_t)ci[c] * kHidden + cj[c]] = f2bf_(hreg[c]);
  }
  auto prefetch = [&](int t) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (!cv[c]) continue;
      const int64_t row = (t < a.T) ? (int64_t)ci[c] * a.T + t : (int64_t)B + ci[c];
      const float* gir = a.gi + row * kGates + cj[c];
      g3[c][0] = __ldg(gir);
      g3[c][1] = __ldg(gir + kHidden);
      g3[c][2] = __ldg(gir + 2 * kHidden);
      dn[c] = (t < a.T) ? a.done[(int64_t)ci[c] * a.T + t] : 0;
    }
  };
  prefetch(0);
  fence_proxy_async_global();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::cluster_sync();  // every CTA's barriers armed and h0 slice in global
  sm100::tc_fence_after();
  const uint32_t tmem = *tslot;
  if (tid == 0)
    sm100::tma_load_3d_mc(tA + cta * CL_KB, &a.xmap, &kbar[cta], j0, 0, 0, 0xFFFF);
  constexpr uint32_t idesc = sm100::make_idesc_bf16(MAXTRAJ, CL_NG, 0, 0);
  uint32_t phase = 0;

  for (int t = 0; t <= a.T; ++t) {
    const int buf = t & 1;
    const uint32_t kpar = (t >> 1) & 1;
    if (warp == 0) {  // MMAs per landed K block (whole warp, elect inside)
      const uint32_t a0 = sm100::smem_u32(tA + buf * CL_A), b0 = sm100::smem_u32(tB);
      if (a.prof && cta == 0 && lane == 0) a.prof[t * 4 + 0] = clock64();
#pragma unroll 1
      for (int kb = 0; kb < CL_CTAS; ++kb) {
        sm100::mbar_wait(&kbar[buf * CL_CTAS + kb], kpar);
        if (a.prof && cta == 0 && lane == 0 && kb == CL_CTAS - 1) a.prof[t * 4 + 1] = clock64();
        sm100::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const uint64_t ad = sm100::make_sdesc_sw64(a0 + kb * CL_KB + kk * 32, 512);
          const uint64_t bd = sm100::make_sdesc(
              b0 + (kb >> 1) * CL_NG * 128 + ((kb & 1) * 2 + kk) * 32, 16, 1024);
          sm100::umma_f16_warp(tmem, ad, bd, idesc, (kb | kk) ? 1u : 0u);
        }
      }
      sm100::umma_commit_warp(mbar);
    }
    sm100::mbar_wait(mbar, phase);
    phase ^= 1;
    if (a.prof && cta == 0 && tid == 0) a.prof[t * 4 + 2] = clock64();
    sm100::tc_fence_after();
    if (tid == 0 && t + 2 <= a.T)  // buffer `buf` is consumed: arm it for step t+2
      for (int kb = 0; kb < CL_CTAS; ++kb)
        sm100::mbar_arrive_expect_tx(&kbar[buf * CL_CTAS + kb], CL_KB);
    {
      uint32_t r3[3][4];
      const uint32_t ta = tmem + ((uint32_t)(32 * sp) << 16) + 8 * ug;
#pragma unroll
      for (int g = 0; g < 3; ++g) sm100::tmem_ld_16x256b(ta + g * CL_UPC, r3[g]);
      sm100::tmem_ld_wait();
      float* gh = reinterpret_cast<float*>(tA + buf * CL_A);  // [64][96], buffer consumed
#pragma unroll
      for (int g = 0; g < 3; ++g)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          gh[(ti0 + (c >> 1) * 8) * CL_NG + g * CL_UPC + tu0 + (c & 1)] = __uint_as_float(r3[g][c]);
    }
    sm100::tc_fence_before();
    __syncthreads();
    const float* gh = reinterpret_cast<const float*>(tA + buf * CL_A);
    const size_t nxt = (size_t)((t + 1) & 1) * a.n_traj * kHidden;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (!cv[c]) continue;
      const int i = ci[c], j = cj[c], u = j - j0;
      const int64_t row = (t < a.T) ? (int64_t)i * a.T + t : (int64_t)B + i;
      const float ghr = gh[i * CL_NG + u] + b3[c][0];
      const float ghz = gh[i * CL_NG + CL_UPC + u] + b3[c][1];
      const float ghn = gh[i * CL_NG + 2 * CL_UPC + u] + b3[c][2];
      const float rr = sig_(g3[c][0] + ghr);
      const float z = sig_(g3[c][1] + ghz);
      const float n = tanh_(g3[c][2] + rr * ghn);
      const float hp = hreg[c];
      const float h = (1.0f - z) * n + z * hp;
      a.core[row * kHidden + j] = h;
      a.core_bf[row * kHidden + j] = f2bf_(h);
      float* gs = a.gates + row * 4 * kHidden;
      gs[j] = rr;
      gs[kHidden + j] = z;
      gs[2 * kHidden + j] = n;
      gs[3 * kHidden + j] = ghn;
      a.hin[row * kHidden + j] = hp;
      a.hbf[row * kHidden + j] = f2bf_(hp);
      if (t < a.T) {
        const float hn = dn[c] ? 0.0f : h;
        hreg[c] = hn;
        a.xbuf[nxt + (int64_t)i * kHidden + j] = f2bf_(hn);
      }
    }
    if (a.prof && cta == 0 && tid == 0) a.prof[t * 4 + 3] = clock64();
    if (t < a.T) {
      prefetch(t + 1);
      fence_proxy_async_global();  // h_{t+1} slice -> visible to the TMA read
      fence_async_smem();          // staging reads of the consumed buffer before any TMA refill
      sm100::tc_fence_before();
      __syncthreads();             // slice complete; TMEM reads of step t done
      if (tid == 0)
        sm100::tma_load_3d_mc(tA + ((t + 1) & 1) * CL_A + cta * CL_KB, &a.xmap,
                              &kbar[((t + 1) & 1) * CL_CTAS + cta], j0, 0, (t + 1) & 1, 0xFFFF);
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, 128);
  }
  sm100::cluster_sync();  // no CTA leaves while a peer may still multicast into it
}

constexpr int FWD_SMEM = 1024 + A_TILE + B_FWD + 2 * MAXTRAJ * NG * 4 + 128;
constexpr int BWD_SMEM = 1024 + 3 * A_TILE + B_BWD + 2 * MAXTRAJ * UPC_B * 4 + 128;
static_assert(BWD_SMEM <= 227 * 1024, "backward GRU smem");

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
const void* kanchor_gru() { return reinterpret_cast<const void*>(&gru_seq_fwd_kernel); }

int gru_seq_supported(int n_traj) { return n_traj >= 1 && n_traj <= MAXTRAJ; }

namespace {
// trajectory-group kernels unless APPO_GRU_LEGACY=1 (the 64-trajectory kernels,
// kept for A/B measurement)
bool gru_grouped() {
  static const bool g = !(getenv("APPO_GRU_LEGACY") && getenv("APPO_GRU_LEGACY")[0] == '1');
  return g;
}
int gru_ws(Ctx* c) {
  if (c->d_gru_sync) return APPO_OK;
  APPO_CUDA_TRY(cudaMalloc(&c->d_gru_sync, sizeof(unsigned) * 64));
  APPO_CUDA_TRY(cudaMalloc(&c->d_gru_part, sizeof(float) * 4 * kHidden * 4));
  APPO_CUDA_TRY(cudaMemsetAsync(c->d_gru_sync, 0, sizeof(unsigned) * 64, c->stream));
  return APPO_OK;
}
}  // namespace

int k_gru_seq_fwd(Ctx* c, int n_traj, int T, const float* gi, const uint16_t* whh,
                  const float* bhh, const uint8_t* done, float* hbuf, uint16_t* hbuf_bf,
                  float* core, uint16_t* core_bf, float* gates, float* hin, uint16_t* hbf,
                  unsigned* bar) {
  // one 16-CTA cluster (TMA-multicast exchange, no grid barrier) when it can be
  // scheduled; the cooperative 32-CTA kernel otherwise
  // opt-in (APPO_GRU_CLUSTER=1): measured slower than the cooperative kernel at
  // n_traj = 64 (16 CTAs carry twice the cell work per SM: ~8.8k vs 8.1k cycles
  // per step), kept for smaller / different GRU shapes
  static int cl_state = getenv("APPO_GRU_CLUSTER") ? 0 : -1;  // 0 untried, 1 ok, -1 off
  if (cl_state >= 0) {
    if (cl_state == 0) {
      if (ensure_smem_attr((const void*)gru_cl_fwd_kernel, CL_SMEM, c->device) != APPO_OK ||
          cudaFuncSetAttribute(gru_cl_fwd_kernel,
                               cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
        cudaGetLastError();
        cl_state = -1;
      } else {
        cl_state = 1;
      }
    }
    if (cl_state == 1) {
      ClFwdArgs a{};
      int st = make_tmap_bf16_3d(&a.xmap, hbuf_bf, kHidden, n_traj, 2, kHidden * 2,
                                 (uint64_t)n_traj * kHidden * 2, 32, MAXTRAJ, 1, 64);
      if (st) return st;
      a.n_traj = n_traj; a.T = T; a.gi = gi; a.whh = whh; a.bhh = bhh; a.done = done;
      a.h0 = hbuf; a.xbuf = hbuf_bf; a.core = core; a.core_bf = core_bf; a.gates = gates;
      a.hin = hin; a.hbf = hbf;
      a.prof = prof_buffer(c);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(CL_CTAS);
      cfg.blockDim = dim3(CL_THR);
      cfg.dynamicSmemBytes = CL_SMEM;
      cfg.stream = c->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CL_CTAS;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaEvent_t ev = timing_begin(c, "gru_seq_fwd_kernel");
      cudaError_t e = cudaLaunchKernelEx(&cfg, gru_cl_fwd_kernel, a);
      c->next_flops = 2.0 * n_traj * (double)kGates * kHidden * (T + 1);
      timing_end(c, "gru_seq_fwd_kernel", ev);
      if (e == cudaSuccess) {
        c->launches++;
        if (a.prof) prof_report(c, a.prof, T + 1, "cluster fwd: data-wait | mma | cells | (next)");
        return APPO_OK;
      }
      cudaGetLastError();
      cl_state = -1;  // fall back for good
    }
  }
  if (gru_grouped()) {
    APPO_TRY(gru_ws(c));
    APPO_TRY(ensure_smem_attr((const void*)gru_g_fwd_kernel, G_FWD_SMEM, c->device));
    const int ng = (n_traj + GT - 1) / GT;
    unsigned* gbar = c->d_gru_sync;
    APPO_CUDA_TRY(cudaMemsetAsync(gbar, 0, sizeof(unsigned) * ng, c->stream));
    GFwdArgs a{};
    int st = make_tmap_bf16_3d(&a.hmap, hbuf_bf, kHidden, n_traj, 2, kHidden * 2,
                               (uint64_t)n_traj * kHidden * 2, 64, GT, 1);
    if (st) return st;
    a.n_traj = n_traj; a.T = T; a.gi = gi; a.whh = whh; a.bhh = bhh; a.done = done;
    a.hbuf = hbuf; a.hbuf_bf = hbuf_bf; a.core = core; a.core_bf = core_bf; a.gates = gates;
    a.hin = hin; a.hbf = hbf; a.bar = gbar; a.prof = prof_buffer(c);
    void* args[] = {&a};
    cudaEvent_t ev = timing_begin(c, "gru_seq_fwd_kernel");
    APPO_CUDA_TRY(cudaLaunchCooperativeKernel((void*)gru_g_fwd_kernel, dim3(NCTA_F * ng),
                                              dim3(THR), args, G_FWD_SMEM, c->stream));
    c->next_flops = 2.0 * n_traj * (double)kGates * kHidden * (T + 1);
    timing_end(c, "gru_seq_fwd_kernel", ev);
    c->launches++;
    if (a.prof)
      prof_report8(c, a.prof, T + 1,
                   "grouped fwd: tma+mma issue | mma wait | tmem->smem | cell+xchg store | "
                   "proxy fence | arrive | outputs | prefetch+barrier wait");
    return APPO_OK;
  }
  APPO_TRY(ensure_smem_attr((const void*)gru_seq_fwd_kernel, FWD_SMEM, c->device));
  APPO_CUDA_TRY(cudaMemsetAsync(bar, 0, sizeof(unsigned), c->stream));
  long long* prof = prof_buffer(c);
  FwdArgs a{};
  int st = make_tmap_bf16_3d(&a.hmap, hbuf_bf, kHidden, n_traj, 2, kHidden * 2,
                             (uint64_t)n_traj * kHidden * 2, 64, MAXTRAJ, 1);
  if (st) return st;
  a.n_traj = n_traj; a.T = T; a.gi = gi; a.whh = whh; a.bhh = bhh; a.done = done; a.hbuf = hbuf;
  a.hbuf_bf = hbuf_bf; a.core = core; a.core_bf = core_bf; a.gates = gates; a.hin = hin;
  a.hbf = hbf; a.bar = bar; a.prof = prof;
  void* args[] = {&a};
  cudaEvent_t ev = timing_begin(c, "gru_seq_fwd_kernel");
  APPO_CUDA_TRY(cudaLaunchCooperativeKernel((void*)gru_seq_fwd_kernel, dim3(NCTA_F), dim3(THR),
                                            args, FWD_SMEM, c->stream));
  c->next_flops = 2.0 * n_traj * (double)kGates * kHidden * (T + 1);
  timing_end(c, "gru_seq_fwd_kernel", ev);
  c->launches++;
  if (prof)
    prof_report8(c, prof, T + 1,
                 "fwd: tma+mma issue | mma wait | tmem->smem | cell+xchg store | proxy fence | "
                 "arrive | outputs | prefetch+barrier wait");
  return APPO_OK;
}

int k_gru_seq_bwd(Ctx* c, int n_traj, int T, const float* dcore, const uint8_t* done,
                  const float* gates, const float* hin, const uint16_t* whh, uint16_t* dghx,
                  uint16_t* dgi, uint16_t* dgh, float* gbih, float* gbhh, unsigned* bar) {
  if (gru_grouped()) {
    APPO_TRY(gru_ws(c));
    APPO_TRY(ensure_smem_attr((const void*)gru_g_bwd_kernel, G_BWD_SMEM, c->device));
    const int ng = (n_traj + GT - 1) / GT;
    unsigned* gbar = c->d_gru_sync + 4;
    APPO_CUDA_TRY(cudaMemsetAsync(gbar, 0, sizeof(unsigned) * ng, c->stream));
    GBwdArgs a{};
    int st = make_tmap_bf16_3d(&a.xmap, dghx, kGates, n_traj, 2, kGates * 2,
                               (uint64_t)n_traj * kGates * 2, 64, GT, 1);
    if (st) return st;
    a.n_traj = n_traj; a.T = T; a.dcore = dcore; a.done = done; a.gates = gates; a.hin = hin;
    a.whh = whh; a.dghx = dghx; a.dgi = dgi; a.dgh = dgh; a.gbih = gbih; a.gbhh = gbhh;
    a.bar = gbar; a.pair = c->d_gru_sync + 32; a.bpart = c->d_gru_part; a.prof = prof_buffer(c);
    void* args[] = {&a};
    cudaEvent_t ev = timing_begin(c, "gru_seq_bwd_kernel");
    APPO_CUDA_TRY(cudaLaunchCooperativeKernel((void*)gru_g_bwd_kernel, dim3(NCTA_GB * ng),
                                              dim3(THR), args, G_BWD_SMEM, c->stream));
    c->next_flops = 2.0 * n_traj * (double)kGates * kHidden * (T - 1);
    timing_end(c, "gru_seq_bwd_kernel", ev);
    c->launches++;
    if (a.prof) prof_report(c, a.prof, T, "grouped bwd: cell | barrier | stage | mma");
    return APPO_OK;
  }
  APPO_TRY(ensure_smem_attr((const void*)gru_seq_bwd_kernel, BWD_SMEM, c->device));
  APPO_CUDA_TRY(cudaMemsetAsync(bar, 0, sizeof(unsigned), c->stream));
  long long* prof = prof_buffer(c);
  BwdArgs a{};
  int st = make_tmap_bf16_3d(&a.xmap, dghx, kGates, n_traj, 2, kGates * 2,
                             (uint64_t)n_traj * kGates * 2, 64, MAXTRAJ, 1);
  if (st) return st;
  a.n_traj = n_traj; a.T = T; a.dcore = dcore; a.done = done; a.gates = gates; a.hin = hin;
  a.whh = whh; a.dghx = dghx; a.dgi = dgi; a.dgh = dgh; a.gbih = gbih; a.gbhh = gbhh;
  a.bar = bar; a.prof = prof;
  void* args[] = {&a};
  cudaEvent_t ev = timing_begin(c, "gru_seq_bwd_kernel");
  // opt-in (APPO_GRU_MC=1): CTA pairs with multicast staging of dgh_t (half
  // the L2 reads of the exchange) -- measured slower (191 vs 177 us: the pair
  // couples two CTAs' step latencies), so the default is the plain launch
  static int mc_ok = getenv("APPO_GRU_MC") && getenv("APPO_GRU_MC")[0] == '1' ? 1 : 0;
  cudaError_t le = cudaErrorUnknown;
  if (mc_ok) {
    a.mc = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(NCTA_B);
    cfg.blockDim = dim3(THR);
    cfg.dynamicSmemBytes = BWD_SMEM;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    le = cudaLaunchKernelEx(&cfg, gru_seq_bwd_kernel, a);
    if (le != cudaSuccess) {
      (void)cudaGetLastError();
      mc_ok = 0;
    }
  }
  if (!mc_ok) {
    a.mc = 0;
    APPO_CUDA_TRY(cudaLaunchCooperativeKernel((void*)gru_seq_bwd_kernel, dim3(NCTA_B), dim3(THR),
                                              args, BWD_SMEM, c->stream));
  }
  c->next_flops = 2.0 * n_traj * (double)kGates * kHidden * (T - 1);
  timing_end(c, "gru_seq_bwd_kernel", ev);
  c->launches++;
  if (prof) prof_report(c, prof, T, "bwd: cell | barrier | stage | mma");
  return APPO_OK;
}

}  // namespace appo_b200
