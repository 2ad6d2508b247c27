// Persistent GRU recurrence for the learner: the T-step forward unroll (+ the
// bootstrap step) and the BPTT reverse sweep each run as ONE cooperative
// kernel; the per-step recurrent product runs on tcgen05.
//
// Partition: 32 CTAs x 16 hidden units.  A CTA owns units j in [16c, 16c+16)
// for all (<= 64) trajectories:
//   forward : D[i][g] = sum_k h_t[i][k] W_hh[g][k], g over the CTA's 48 gate
//             rows (r, z, n of its 16 units).  UMMA M=64 (trajectories) x N=48
//             x K=512; B = W slice resident in smem (bf16, SW128 K-major), A =
//             h_t staged from global each step.  The epilogue applies the cell
//             (PyTorch r,z,n convention; oracle gru_fwd) for its units, so the
//             only cross-CTA traffic is h_{t+1} (64 x 512 bf16, L2-resident).
//   backward: gate gradients for own units (oracle orc_learner_step BPTT),
//             published as dgh_t (64 x 1536 bf16); after a grid barrier
//             dnext[i][j] = dh*z + sum_g dgh_t[i][g] W_hh[g][j] as UMMA M=64 x
//             N=16 x K=1536 with W_hh[:, own units]^T resident (K-major) and
//             dgh_t staged in three 512-wide K chunks (double-buffered).
// TMEM layout for M=64 (cta_group::1): row m lives in lane (m % 16) + 32*(m/16)
// (CuTe "half subpartitions" atom, mma_traits_sm100.hpp), so warp w's lanes
// 0..15 hold rows 16w..16w+15.
#include <cuda_bf16.h>

#include "model.cuh"
#include "model_kernels.cuh"
#include "sm100.cuh"

namespace appo_b200 {
namespace {

constexpr int UPC = 16;                    // hidden units per CTA
constexpr int NCTA = kHidden / UPC;        // 32
constexpr int MAXTRAJ = 64;                // UMMA M
constexpr int THR = 256;
constexpr int NG = 3 * UPC;                // 48 gate rows per CTA (forward N)
constexpr int KB_BYTES_A = MAXTRAJ * 128;  // one 64-wide K block of the A tile
constexpr int A_FWD = 8 * KB_BYTES_A;      // 64 x 512 bf16 = 64 KB
constexpr int B_FWD = 8 * NG * 128;        // 48 x 512 bf16 = 48 KB
constexpr int A_CH = 8 * KB_BYTES_A;       // backward K chunk 64 x 512 bf16 = 64 KB
constexpr int B_BWD = 24 * UPC * 128;      // 16 x 1536 bf16 = 48 KB

__device__ __forceinline__ uint16_t f2bf_(float f) {
  __nv_bfloat16 h = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t*>(&h);
}
__device__ __forceinline__ float bf2f_(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }
__device__ __forceinline__ float sig_(float x) { return 1.0f / (1.0f + expf(-x)); }

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
__device__ __forceinline__ void grid_barrier(unsigned* counter, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(counter, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// Stage rows [n_rows] x 512 bf16 (global row stride ld elements, starting at
// column col0) into a 64-row SW128 K-major tile; rows >= n_rows are zero.
__device__ __forceinline__ void stage_a(uint8_t* tile, const uint16_t* src, int n_rows, int64_t ld,
                                        int col0) {
  constexpr int CH = MAXTRAJ * 64;  // 16-byte chunks in 64 x 512
  for (int base = threadIdx.x; base < CH; base += THR * 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = base + u * THR;
      const int r = e >> 6, c = e & 63;
      v[u] = (e < CH && r < n_rows)
                 ? __ldcg(reinterpret_cast<const uint4*>(src + (int64_t)r * ld + col0) + c)
                 : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = base + u * THR;
      if (e < CH) {
        const int r = e >> 6, c = e & 63;
        *reinterpret_cast<uint4*>(tile + sw128(MAXTRAJ, r, c >> 3, c & 7)) = v[u];
      }
    }
  }
}

struct FwdArgs {
  int n_traj, T;
  const float* gi;       // [R][1536] (x W_ih^T + b_ih), rows s = i*T+t, boot rows B+i
  const uint16_t* whh;   // bf16 [1536][512] (published copy of the master)
  const float* bhh;      // [1536]
  const uint8_t* done;   // [B]
  float* hbuf;           // [2][n_traj][512] fp32 ping-pong (hbuf[0] = h0 on entry)
  uint16_t* hbuf_bf;     // [2][n_traj][512] bf16 ping-pong
  float* core;           // [R][512]
  uint16_t* core_bf;     // [R][512]
  float* gates;          // [R][4][512]
  float* hin;            // [R][512]
  uint16_t* hbf;         // [R][512]
  unsigned* bar;
};

__global__ void __launch_bounds__(THR, 1) gru_seq_fwd_kernel(FwdArgs a) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* tA = sm;
  uint8_t* tB = sm + A_FWD;
  float* gh = reinterpret_cast<float*>(tB + B_FWD);              // [64][NG]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(gh + MAXTRAJ * NG);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int j0 = blockIdx.x * UPC;
  const int B = a.n_traj * a.T;

  // resident B operand: gate row n = g*16 + u (g in r,z,n) -> W_hh row g*512 + j0 + u
  for (int e = tid; e < NG * 64; e += THR) {
    const int n = e >> 6, c = e & 63;
    const int grow = (n / UPC) * kHidden + j0 + (n % UPC);
    *reinterpret_cast<uint4*>(tB + sw128(NG, n, c >> 3, c & 7)) =
        reinterpret_cast<const uint4*>(a.whh + (int64_t)grow * kHidden)[c];
  }
  if (tid == 0) {
    sm100::mbar_init(mbar, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) {
    sm100::tmem_alloc(tslot, 64);
    sm100::tmem_relinquish();
  }
  // first h_t (bf16) from the fp32 h0, own columns only
  for (int e = tid; e < a.n_traj * UPC; e += THR) {
    const int64_t o = (int64_t)(e / UPC) * kHidden + j0 + (e % UPC);
    a.hbuf_bf[o] = f2bf_(a.hbuf[o]);
  }
  sm100::tc_fence_before();
  grid_barrier(a.bar, gridDim.x);  // h0 bf16 complete everywhere
  sm100::tc_fence_after();
  const uint32_t tmem = *tslot;
  constexpr uint32_t idesc = sm100::make_idesc_bf16(MAXTRAJ, NG, 0, 0);
  unsigned epoch = 1;
  uint32_t phase = 0;

  for (int t = 0; t <= a.T; ++t) {
    const size_t cur = (size_t)(t & 1) * a.n_traj * kHidden;
    const size_t nxt = (size_t)((t + 1) & 1) * a.n_traj * kHidden;
    stage_a(tA, a.hbuf_bf + cur, a.n_traj, kHidden, 0);
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      sm100::tc_fence_after();
      const uint32_t a0 = sm100::smem_u32(tA), b0 = sm100::smem_u32(tB);
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const uint64_t ad = sm100::make_sdesc(a0 + (k >> 2) * KB_BYTES_A + (k & 3) * 32, 16, 1024);
        const uint64_t bd = sm100::make_sdesc(b0 + (k >> 2) * NG * 128 + (k & 3) * 32, 16, 1024);
        sm100::umma_f16(tmem, ad, bd, idesc, k > 0 ? 1u : 0u);
      }
      sm100::umma_commit(mbar);
    }
    sm100::mbar_wait(mbar, phase);
    phase ^= 1;
    sm100::tc_fence_after();
    if (warp < 4) {
      uint32_t r[16];
#pragma unroll
      for (int cb = 0; cb < NG; cb += 16) {
        sm100::tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + cb, r);
        sm100::tmem_ld_wait();
        if (lane < 16) {
          const int i = 16 * warp + lane;
#pragma unroll
          for (int q = 0; q < 16; ++q) gh[i * NG + cb + q] = __uint_as_float(r[q]);
        }
      }
    }
    sm100::tc_fence_before();
    __syncthreads();
    // cells: 64 traj x 16 units, 4 per thread
    for (int e = tid; e < a.n_traj * UPC; e += THR) {
      const int i = e / UPC, u = e % UPC, j = j0 + u;
      const int64_t row = (t < a.T) ? (int64_t)i * a.T + t : (int64_t)B + i;
      const float* gir = a.gi + row * kGates;
      const float ghr = gh[i * NG + u] + a.bhh[j];
      const float ghz = gh[i * NG + UPC + u] + a.bhh[kHidden + j];
      const float ghn = gh[i * NG + 2 * UPC + u] + a.bhh[2 * kHidden + j];
      const float rr = sig_(gir[j] + ghr);
      const float z = sig_(gir[kHidden + j] + ghz);
      const float n = tanhf(gir[2 * kHidden + j] + rr * ghn);
      const float hp = __ldcg(a.hbuf + cur + (int64_t)i * kHidden + j);
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
        const float hn = a.done[(int64_t)i * a.T + t] ? 0.0f : h;
        a.hbuf[nxt + (int64_t)i * kHidden + j] = hn;
        a.hbuf_bf[nxt + (int64_t)i * kHidden + j] = f2bf_(hn);
      }
    }
    if (t < a.T) grid_barrier(a.bar, ++epoch * gridDim.x);
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, 64);
  }
}

struct BwdArgs {
  int n_traj, T;
  const float* dcore;   // [B][512]
  const uint8_t* done;  // [B]
  const float* gates;   // [R][4][512]
  const float* hin;     // [R][512]
  const uint16_t* whh;  // bf16 [1536][512]
  uint16_t* dghx;       // [2][n_traj][1536] bf16 exchange
  uint16_t* dgi;        // [B][1536]
  uint16_t* dgh;        // [B][1536]
  unsigned* bar;
};

__global__ void __launch_bounds__(THR, 1) gru_seq_bwd_kernel(BwdArgs a) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* tA[2] = {sm, sm + A_CH};
  uint8_t* tB = sm + 2 * A_CH;
  float* dn = reinterpret_cast<float*>(tB + B_BWD);     // [64][16] dnext (own units)
  float* dd = dn + MAXTRAJ * UPC;                       // [64][16] dh * z
  uint64_t* mbar = reinterpret_cast<uint64_t*>(dd + MAXTRAJ * UPC);  // [2] per A buffer
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int j0 = blockIdx.x * UPC;

  // resident B: row n = own unit u, K = gate g: B[u][g] = W_hh[g][j0 + u] (K-major)
  for (int e = tid; e < UPC * (kGates / 8); e += THR) {
    const int u = e / (kGates / 8), c8 = e % (kGates / 8);  // chunk of 8 gates
    uint32_t w[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int g = c8 * 8 + 2 * p;
      w[p] = (uint32_t)a.whh[(int64_t)g * kHidden + j0 + u] |
             ((uint32_t)a.whh[(int64_t)(g + 1) * kHidden + j0 + u] << 16);
    }
    *reinterpret_cast<uint4*>(tB + sw128(UPC, u, c8 >> 3, c8 & 7)) =
        make_uint4(w[0], w[1], w[2], w[3]);
  }
  for (int e = tid; e < MAXTRAJ * UPC; e += THR) dn[e] = 0.0f;
  if (tid == 0) {
    sm100::mbar_init(&mbar[0], 1);
    sm100::mbar_init(&mbar[1], 1);
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
  constexpr uint32_t idesc = sm100::make_idesc_bf16(MAXTRAJ, UPC, 0, 0);
  unsigned epoch = 0;
  uint32_t ph[2] = {0, 0};

  for (int t = a.T - 1; t >= 0; --t) {
    uint16_t* xb = a.dghx + (size_t)(t & 1) * a.n_traj * kGates;
    // gate gradients for own units
    for (int e = tid; e < a.n_traj * UPC; e += THR) {
      const int i = e / UPC, u = e % UPC, j = j0 + u;
      const int64_t s = (int64_t)i * a.T + t;
      const float keep = a.done[s] ? 0.0f : 1.0f;
      const float dh = a.dcore[s * kHidden + j] + keep * dn[i * UPC + u];
      const float* gs = a.gates + s * 4 * kHidden;
      const float r = gs[j], z = gs[kHidden + j], n = gs[2 * kHidden + j];
      const float ghn = gs[3 * kHidden + j];
      const float hp = a.hin[s * kHidden + j];
      const float dnn = dh * (1.0f - z);
      const float dz = dh * (hp - n);
      const float dan = dnn * (1.0f - n * n);
      const uint16_t dgr = f2bf_(dan * ghn * r * (1.0f - r));
      const uint16_t dgz = f2bf_(dz * z * (1.0f - z));
      const uint16_t dgn = f2bf_(dan * r);
      uint16_t* gi_row = a.dgi + s * kGates;
      uint16_t* gh_row = a.dgh + s * kGates;
      gi_row[j] = dgr;
      gi_row[kHidden + j] = dgz;
      gi_row[2 * kHidden + j] = f2bf_(dan);
      gh_row[j] = dgr;
      gh_row[kHidden + j] = dgz;
      gh_row[2 * kHidden + j] = dgn;
      uint16_t* xr = xb + (int64_t)i * kGates;
      xr[j] = dgr;
      xr[kHidden + j] = dgz;
      xr[2 * kHidden + j] = dgn;
      dd[i * UPC + u] = dh * z;
    }
    if (t == 0) break;  // d(h0) is not needed
    grid_barrier(a.bar, ++epoch * gridDim.x);
    // dnext = dd + dgh_t . W_hh[:, own]: three K chunks of 512, double-buffered A
    for (int ch = 0; ch < 3; ++ch) {
      const int buf = ch & 1;
      if (ch >= 2) {  // buffer reuse: wait for the MMAs of chunk ch-2
        sm100::mbar_wait(&mbar[buf], ph[buf]);
        ph[buf] ^= 1;
      }
      stage_a(tA[buf], xb, a.n_traj, kGates, ch * 512);
      fence_async_smem();
      __syncthreads();
      if (tid == 0) {
        sm100::tc_fence_after();
        const uint32_t a0 = sm100::smem_u32(tA[buf]), b0 = sm100::smem_u32(tB);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int kg = ch * 32 + k;  // global K16 step over 1536
          const uint64_t ad =
              sm100::make_sdesc(a0 + (k >> 2) * KB_BYTES_A + (k & 3) * 32, 16, 1024);
          const uint64_t bd =
              sm100::make_sdesc(b0 + (kg >> 2) * UPC * 128 + (kg & 3) * 32, 16, 1024);
          sm100::umma_f16(tmem, ad, bd, idesc, kg > 0 ? 1u : 0u);
        }
        sm100::umma_commit(&mbar[buf]);
      }
    }
    // chunks 1 (buf 1) and 2 (buf 0) still outstanding; MMAs complete in order
    sm100::mbar_wait(&mbar[1], ph[1]);
    ph[1] ^= 1;
    sm100::mbar_wait(&mbar[0], ph[0]);
    ph[0] ^= 1;
    sm100::tc_fence_after();
    if (warp < 4) {
      uint32_t r[16];
      sm100::tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16), r);
      sm100::tmem_ld_wait();
      if (lane < 16) {
        const int i = 16 * warp + lane;
#pragma unroll
        for (int u = 0; u < UPC; ++u) dn[i * UPC + u] = dd[i * UPC + u] + __uint_as_float(r[u]);
      }
    }
    sm100::tc_fence_before();
    __syncthreads();
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, 32);
  }
}

constexpr int FWD_SMEM = 1024 + A_FWD + B_FWD + MAXTRAJ * NG * 4 + 64;
constexpr int BWD_SMEM = 1024 + 2 * A_CH + B_BWD + 2 * MAXTRAJ * UPC * 4 + 64;

}  // namespace

int gru_seq_supported(int n_traj) { return n_traj >= 1 && n_traj <= MAXTRAJ; }

int k_gru_seq_fwd(Ctx* c, int n_traj, int T, const float* gi, const uint16_t* whh,
                  const float* bhh, const uint8_t* done, float* hbuf, uint16_t* hbuf_bf,
                  float* core, uint16_t* core_bf, float* gates, float* hin, uint16_t* hbf,
                  unsigned* bar) {
  static bool attr = false;
  if (!attr) {
    APPO_CUDA_TRY(cudaFuncSetAttribute(gru_seq_fwd_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, FWD_SMEM));
    attr = true;
  }
  APPO_CUDA_TRY(cudaMemsetAsync(bar, 0, sizeof(unsigned), c->stream));
  FwdArgs a{n_traj, T, gi, whh, bhh, done, hbuf, hbuf_bf, core, core_bf, gates, hin, hbf, bar};
  void* args[] = {&a};
  cudaEvent_t ev = timing_begin(c, "gru_seq_fwd_kernel");
  APPO_CUDA_TRY(cudaLaunchCooperativeKernel((void*)gru_seq_fwd_kernel, dim3(NCTA), dim3(THR), args,
                                            FWD_SMEM, c->stream));
  c->next_flops = 2.0 * n_traj * (double)kGates * kHidden * (T + 1);
  timing_end(c, "gru_seq_fwd_kernel", ev);
  c->launches++;
  return APPO_OK;
}

int k_gru_seq_bwd(Ctx* c, int n_traj, int T, const float* dcore, const uint8_t* done,
                  const float* gates, const float* hin, const uint16_t* whh, uint16_t* dghx,
                  uint16_t* dgi, uint16_t* dgh, unsigned* bar) {
  static bool attr = false;
  if (!attr) {
    APPO_CUDA_TRY(cudaFuncSetAttribute(gru_seq_bwd_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, BWD_SMEM));
    attr = true;
  }
  APPO_CUDA_TRY(cudaMemsetAsync(bar, 0, sizeof(unsigned), c->stream));
  BwdArgs a{n_traj, T, dcore, done, gates, hin, whh, dghx, dgi, dgh, bar};
  void* args[] = {&a};
  cudaEvent_t ev = timing_begin(c, "gru_seq_bwd_kernel");
  APPO_CUDA_TRY(cudaLaunchCooperativeKernel((void*)gru_seq_bwd_kernel, dim3(NCTA), dim3(THR), args,
                                            BWD_SMEM, c->stream));
  c->next_flops = 2.0 * n_traj * (double)kGates * kHidden * (T - 1);
  timing_end(c, "gru_seq_bwd_kernel", ev);
  c->launches++;
  return APPO_OK;
}

}  // namespace appo_b200
