// conv2 forward (k4 s2, 32 -> 64 channels, bf16 NHWC a1 -> ELU -> bf16 NHWC a2)
// as a space-to-depth taps GEMM on tcgen05 (sm_100a), the conv1.cu idea for a
// bf16 input: no conversion at all, the A operand is the TMA'd activation.
//
// After space-to-depth by 2, Z[py][px] = (a1[2py + e][2px + pj][ci]) for
// e, pj in {0, 1} (128 values) and conv2 is a k2 s1 convolution
//   out[y][x] = sum_{a,b} Z[y+a][x+b] . W_ab,  W_ab[co][(e,pj,ci)] = W2[co][2a+e][2b+pj][ci].
// In the pixel-pair view of a1 (one 128-byte row = pixels 2px, 2px+1 of one
// input row), the two K atoms e = 0, 1 of Z are the even and the odd input
// rows.  Each image is staged by TMA as two planes (even rows, odd rows; an
// element stride of 2 along the rows) of pixel-pair rows r = py*16 + px, so for
// the tile rows m = y*16 + x the operand "Z shifted down a rows" is plane e from
// row 16a on: a descriptor start offset (the SW128 pattern follows the absolute
// address, conv1.cu).  The column taps b are the two halves of an N = 128 B
// operand (rows 2co + b), summed in the epilogue with a one-lane shuffle.  One
// 128-row tile per image (Ho x 16 <= 128): 2 row taps x 2 atoms x 4 K16 steps.
//
//   warp 0      TMA: both planes of an image per stage (ring of C2_NSTG)
//   warp 1      TMEM owner + MMA issuer (16 x M128 N128 K16 per image)
//   warps 2..9  epilogue: TMEM -> + bias, ELU -> bf16 rows of a2 (2 warps per
//               TMEM lane quarter, 32 output channels each)
//
// Replaces: the reference has no convolutional encoder (SURVEY.md §8 a2,
// SPEC.md:273-274); convnet_simple's conv2 of the model contract (DESIGN.md
// §2), parity-checked against the fp64 oracle like the engine path it replaces.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "appo_common.cuh"
#include "gemm.cuh"
#include "sm100.cuh"

namespace appo_b200 {
namespace {

constexpr int C2_EPI_WARPS = 8;
constexpr int C2_THREADS = 32 * (2 + C2_EPI_WARPS);
constexpr int C2_NSTG = 3;                   // images in flight
constexpr int C2_NACC = 2;                   // TMEM accumulators of 128 columns
constexpr int C2_PROWS = 152;                // plane rows: (Ho+1) x 16 pairs + the a = 1 overrun (<= 144)
constexpr int C2_PLANE = C2_PROWS * 128;     // 19 KB (1024-aligned)
constexpr int C2_STAGE = 2 * C2_PLANE;
constexpr int C2_BBYTES = 4 * 128 * 128;     // (a, e) blocks of 128 rows (2co + b)
constexpr int C2_SMEM = 1024 + C2_NSTG * C2_STAGE + C2_BBYTES + 256;

struct C2Params {
  int n_img, Ho, Wo;         // output geometry (Ho * 16 <= 128, Wo + 1 <= 16)
  int plane_rows;            // (Ho + 1) * 16 rows written by the TMA per plane
  const uint16_t* w;         // bf16 [64][4][4][32] (O, kh, kw, I)
  const float* bias;
  uint16_t* out;             // bf16 [n_img][Ho][Wo][64]
};

__device__ __forceinline__ uint64_t c2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 c2_unpack(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ uint64_t c2_add2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t c2_fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ float c2_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t c2_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void c2_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__global__ void __launch_bounds__(C2_THREADS, 1)
    conv2_s2d_kernel(const __grid_constant__ CUtensorMap map_a1,
                     const __grid_constant__ CUtensorMap map_w, const __grid_constant__ C2Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stg = smem;                              // C2_NSTG x (even plane, odd plane)
  uint8_t* bsm = stg + C2_NSTG * C2_STAGE;          // resident weights
  uint64_t* bars = reinterpret_cast<uint64_t*>(bsm + C2_BBYTES);
  uint64_t* full = bars;
  uint64_t* empty = full + C2_NSTG;
  uint64_t* acc_full = empty + C2_NSTG;
  uint64_t* acc_empty = acc_full + C2_NACC;
  uint64_t* bfull = acc_empty + C2_NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    sm100::tma_prefetch(&map_a1);
    sm100::tma_prefetch(&map_w);
    sm100::mbar_init(bfull, 1);
    for (int s = 0; s < C2_NSTG; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < C2_NACC; ++s) {
      sm100::mbar_init(&acc_full[s], 1);
      sm100::mbar_init(&acc_empty[s], C2_EPI_WARPS);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 0) {
    // B block (a, e): row n = 2co + b holds W2[co][2a+e][2b .. 2b+1][0..31]
    // (128 B): one box {64, 2 (b), 1 (kh), 64 (co)} of the weights per block.
    // A published copy (an earlier step): loaded before the PDL wait.
    __syncwarp();
    sm100::mbar_arrive_expect_tx_warp(bfull, C2_BBYTES);
#pragma unroll
    for (int blk = 0; blk < 4; ++blk)
      sm100::tma_load_4d_warp(bsm + blk * 16384, &map_w, bfull, 0, 0, blk, 0);
  }
  if (warp == 1) {
    sm100::tmem_alloc(tmem_slot, C2_NACC * 128);
    sm100::tmem_relinquish();
  }
  // plane rows past the TMA box (read only for dropped output rows): finite zeros
  for (int e = threadIdx.x; e < C2_NSTG * 2 * (C2_PROWS - p.plane_rows) * 8; e += C2_THREADS) {
    const int pl = e / ((C2_PROWS - p.plane_rows) * 8), rest = e % ((C2_PROWS - p.plane_rows) * 8);
    reinterpret_cast<uint4*>(stg + pl * C2_PLANE + p.plane_rows * 128)[rest] = make_uint4(0, 0, 0, 0);
  }
  APPO_PDL_ENTRY();  // a1 and the published weights come from earlier kernels
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---- TMA: even rows (coordinate 0) and odd rows (1), element stride 2 ----
    int j = 0;
    for (int img = blockIdx.x; img < p.n_img; img += gridDim.x, ++j) {
      const int s = j % C2_NSTG;
      sm100::mbar_wait(&empty[s], ((j / C2_NSTG) & 1) ^ 1);
      sm100::mbar_arrive_expect_tx_warp(&full[s], 2u * p.plane_rows * 128);
      sm100::tma_load_4d_warp(stg + s * C2_STAGE, &map_a1, &full[s], 0, 0, 0, img);
      sm100::tma_load_4d_warp(stg + s * C2_STAGE + C2_PLANE, &map_a1, &full[s], 0, 0, 1, img);
    }
  } else if (warp == 1) {
    // ---- MMA: row taps a (plane offset 16a rows) x atoms e x 4 K16 steps ----
    constexpr uint32_t idesc = sm100::make_idesc_bf16(128, 128, 0, 0);
    const uint32_t s0 = sm100::smem_u32(stg), b0 = sm100::smem_u32(bsm);
    sm100::mbar_wait(bfull, 0);
    int j = 0, acc = 0;
    uint32_t accph = 0;
    for (int img = blockIdx.x; img < p.n_img; img += gridDim.x, ++j) {
      const int s = j % C2_NSTG;
      sm100::mbar_wait(&full[s], (j / C2_NSTG) & 1);
      sm100::mbar_wait(&acc_empty[acc], accph ^ 1);
      sm100::tc_fence_after();
      const uint32_t d = tmem_base + acc * 128;
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t ad =
                sm100::make_sdesc(s0 + s * C2_STAGE + e * C2_PLANE + a * 16 * 128 + ks * 32, 16, 1024);
            const uint64_t bd = sm100::make_sdesc(b0 + (2 * a + e) * 16384 + ks * 32, 16, 1024);
            sm100::umma_f16_warp(d, ad, bd, idesc, (a | e | ks) ? 1u : 0u);
          }
      sm100::umma_commit_warp(&empty[s]);
      sm100::umma_commit_warp(&acc_full[acc]);
      if (++acc == C2_NACC) { acc = 0; accph ^= 1; }
    }
  } else {
    // ---- epilogue: quarter q = TMEM lanes 32q.. (rows m = y*16 + x), 32 channels ----
    const int ew = warp - 2, q = warp & 3, part = ew >> 2;
    constexpr float kLog2e = 1.4426950408889634f;
    uint64_t b2[16], b2l[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float x0 = __ldg(p.bias + part * 32 + 2 * k), x1 = __ldg(p.bias + part * 32 + 2 * k + 1);
      b2[k] = c2_pack(x0, x1);
      b2l[k] = c2_pack(x0 * kLog2e, x1 * kLog2e);
    }
    const uint64_t l2e2 = c2_pack(kLog2e, kLog2e), mone2 = c2_pack(-1.0f, -1.0f);
    const int m = 32 * q + lane, y = m >> 4, x = m & 15;
    const bool row_ok = (32 * q) < p.Ho * 16;  // warp-uniform: any valid row in this quarter
    int acc = 0;
    uint32_t accph = 0;
    for (int img = blockIdx.x; img < p.n_img; img += gridDim.x) {
      sm100::mbar_wait(&acc_full[acc], accph);
      sm100::tc_fence_after();
      if (row_ok) {
        uint16_t* dst = p.out + (((size_t)img * p.Ho + y) * p.Wo + x) * 64 + part * 32;
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // 16 channels (32 TMEM columns) at a time
          uint32_t r[32];
          c2_ld32(tmem_base + ((uint32_t)(32 * q) << 16) + acc * 128 + part * 64 + h * 32, r);
          sm100::tmem_ld_wait();
          uint32_t w[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            // column tap b = 0 at pixel x plus b = 1 taken from pixel x + 1
            const uint64_t v = c2_add2(
                c2_pack(__uint_as_float(r[4 * k]), __uint_as_float(r[4 * k + 2])),
                c2_pack(__shfl_down_sync(0xffffffffu, __uint_as_float(r[4 * k + 1]), 1),
                        __shfl_down_sync(0xffffffffu, __uint_as_float(r[4 * k + 3]), 1)));
            const float2 xv = c2_unpack(c2_add2(v, b2[h * 8 + k]));
            const float2 tl = c2_unpack(c2_fma2(v, l2e2, b2l[h * 8 + k]));
            const float2 ev = c2_unpack(
                c2_add2(c2_pack(c2_ex2(fminf(tl.x, 0.0f)), c2_ex2(fminf(tl.y, 0.0f))), mone2));
            w[k] = c2_bf16x2(fmaxf(xv.x, ev.x), fmaxf(xv.y, ev.y));  // ELU
          }
          if (y < p.Ho && x < p.Wo) {
            uint4* o = reinterpret_cast<uint4*>(dst + h * 16);
            o[0] = make_uint4(w[0], w[1], w[2], w[3]);
            o[1] = make_uint4(w[4], w[5], w[6], w[7]);
          }
        }
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&acc_empty[acc]);
      if (++acc == C2_NACC) { acc = 0; accph ^= 1; }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem_base, C2_NACC * 128);
  }
}

// ---- conv2 input gradient (sub-pixel classes) with the shifted-view trick --
// dz1[2py+e][2px+pj][ci] = ELU'(a1) * sum_{a,b} dz2[py-a][px-b] . W2[:, 2a+e, 2b+pj, ci]:
// rows m = py*16 + px (py < 8: the coarse row py = 8 only meets dz2 rows >= Ho,
// its outputs are zero), N = (class 2e+pj, ci) = 128, K = (tap 2a+b, co) = 256.
// dz2 is staged ONCE per image with a zero border (TMA box from (-1, -1): 9 x 16
// rows of 128 B), tap (a, b) = plane rows from 17 - 16a - b on (a column wrap
// lands on the next row's x = -1 border, which is zero); the ELU' operand a1 is
// staged as four class planes (element stride 2 in x and y) whose row m is the
// output pixel of TMEM row m; the bias gradient is summed from the stored bf16
// values into 2^-32 fixed-point atomics (deterministic), as the engine path.
constexpr int D2_EPI_WARPS = 8;
constexpr int D2_THREADS = 32 * (2 + D2_EPI_WARPS);
constexpr int D2_NSTG = 2;                        // images in flight (3 measured no faster)
constexpr int D2_ZROWS = 152;                      // dz2 plane rows (144 + zero overrun)
constexpr int D2_ZBYTES = D2_ZROWS * 128;
constexpr int D2_ABYTES = 4 * 128 * 64;            // a1 class planes: 4 x 128 rows x 64 B
constexpr int D2_STAGE = D2_ZBYTES + D2_ABYTES;
constexpr int D2_BBYTES = 4 * 128 * 128;           // taps x 128 rows (class, ci)
constexpr int D2_OBYTES = D2_EPI_WARPS * 2 * 2048;  // output staging: warp x class x 32 px x 64 B
constexpr int D2_SMEM = 1024 + D2_NSTG * D2_STAGE + D2_BBYTES + D2_OBYTES + 256;

struct D2Params {
  int n_img, Hi, Wi;              // a1 / dz1 geometry (17 x 31)
  const uint16_t* wt;             // [4 cls][32 ci][4 taps][64 co] (publish_derived)
  uint16_t* dz;                   // dz1 [n_img][Hi][Wi][32]
  unsigned long long* bacc;       // [16][32] fixed-point bias accumulators
  unsigned* bcnt;
  float* bout;
};

// two stores in flight per warp (one per class buffer): before refilling class
// pj's buffer, at most one group (the other class's latest) may still read smem
__device__ __forceinline__ void tma_store_wait_read_warp(int) {
  sm100::tma_store_wait_read<1>();
  __syncwarp();
}

__device__ __forceinline__ float d2_reduce16(float (&v)[16], int lane) {
#pragma unroll
  for (int k = 8; k >= 1; k >>= 1) {
    const bool up = (lane & k) != 0;
#pragma unroll
    for (int j = 0; j < k; ++j) {
      const float send = up ? v[j] : v[j + k];
      const float keep = up ? v[j + k] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, k);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

__global__ void __launch_bounds__(D2_THREADS, 1)
    conv2_dgrad_kernel(const __grid_constant__ CUtensorMap map_dz2,
                       const __grid_constant__ CUtensorMap map_a1,
                       const __grid_constant__ CUtensorMap map_out,
                       const __grid_constant__ CUtensorMap map_wt, const __grid_constant__ D2Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stg = smem;
  uint8_t* bsm = stg + D2_NSTG * D2_STAGE;
  uint8_t* osm = bsm + D2_BBYTES;                    // per-warp output staging (TMA stores)
  uint64_t* bars = reinterpret_cast<uint64_t*>(osm + D2_OBYTES);
  uint64_t* full = bars;
  uint64_t* empty = full + D2_NSTG;
  uint64_t* acc_full = empty + D2_NSTG;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* bfull = acc_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
  __shared__ unsigned last_cta;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    sm100::tma_prefetch(&map_dz2);
    sm100::tma_prefetch(&map_a1);
    sm100::tma_prefetch(&map_out);
    sm100::tma_prefetch(&map_wt);
    for (int s = 0; s < D2_NSTG; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1 + D2_EPI_WARPS);  // MMA commit + epilogue (a1 planes)
    }
    sm100::mbar_init(bfull, 1);
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&acc_full[s], 1);
      sm100::mbar_init(&acc_empty[s], D2_EPI_WARPS);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 0) {
    // resident B by TMA: wt rows (class, ci) x K (tap, co), one SW128 box per
    // tap; derived from a published copy (an earlier step): before the PDL wait
    __syncwarp();
    sm100::mbar_arrive_expect_tx_warp(bfull, D2_BBYTES);
#pragma unroll
    for (int tap = 0; tap < 4; ++tap)
      sm100::tma_load_3d_warp(bsm + tap * 16384, &map_wt, bfull, tap * 64, 0, 0);
  }
  if (warp == 1) {
    sm100::tmem_alloc(tmem_slot, 256);
    sm100::tmem_relinquish();
  }
  for (int e = threadIdx.x; e < D2_NSTG * (D2_ZROWS - 144) * 8; e += D2_THREADS) {
    const int st = e / ((D2_ZROWS - 144) * 8), r = e % ((D2_ZROWS - 144) * 8);
    reinterpret_cast<uint4*>(stg + st * D2_STAGE + 144 * 128)[r] = make_uint4(0, 0, 0, 0);
  }
  APPO_PDL_ENTRY();  // dz2 and the derived weights come from earlier kernels
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    int j = 0;
    for (int img = blockIdx.x; img < p.n_img; img += gridDim.x, ++j) {
      const int s = j % D2_NSTG;
      sm100::mbar_wait(&empty[s], ((j / D2_NSTG) & 1) ^ 1);
      uint8_t* base = stg + s * D2_STAGE;
      sm100::mbar_arrive_expect_tx_warp(&full[s], 144 * 128 + D2_ABYTES);
      sm100::tma_load_4d_warp(base, &map_dz2, &full[s], 0, -1, -1, img);
#pragma unroll
      for (int cls = 0; cls < 4; ++cls)
        sm100::tma_load_4d_warp(base + D2_ZBYTES + cls * 8192, &map_a1, &full[s], 0, cls & 1,
                                cls >> 1, img);
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = sm100::make_idesc_bf16(128, 128, 0, 0);
    const uint32_t s0 = sm100::smem_u32(stg), b0 = sm100::smem_u32(bsm);
    sm100::mbar_wait(bfull, 0);
    int j = 0, acc = 0;
    uint32_t accph = 0;
    for (int img = blockIdx.x; img < p.n_img; img += gridDim.x, ++j) {
      const int s = j % D2_NSTG;
      sm100::mbar_wait(&full[s], (j / D2_NSTG) & 1);
      sm100::mbar_wait(&acc_empty[acc], accph ^ 1);
      sm100::tc_fence_after();
      const uint32_t d = tmem_base + acc * 128;
#pragma unroll
      for (int tap = 0; tap < 4; ++tap) {
        const int a = tap >> 1, b = tap & 1;
        const uint32_t arow = (uint32_t)(17 - 16 * a - b);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t ad = sm100::make_sdesc(s0 + s * D2_STAGE + arow * 128 + ks * 32, 16, 1024);
          const uint64_t bd = sm100::make_sdesc(b0 + tap * 16384 + ks * 32, 16, 1024);
          sm100::umma_f16_warp(d, ad, bd, idesc, (tap | ks) ? 1u : 0u);
        }
      }
      sm100::umma_commit_warp(&empty[s]);
      sm100::umma_commit_warp(&acc_full[acc]);
      if (++acc == 2) { acc = 0; accph ^= 1; }
    }
  } else {
    // epilogue: quarter q (rows m = 32q + lane), row parity e = part: classes 2e, 2e+1
    const int ew = warp - 2, q = warp & 3, e = ew >> 2;
    const int m = 32 * q + lane, py = m >> 4, px = m & 15;
    float bs[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) bs[k] = 0.0f;
    int j = 0, acc = 0;
    uint32_t accph = 0;
    for (int img = blockIdx.x; img < p.n_img; img += gridDim.x, ++j) {
      const int s = j % D2_NSTG;
      sm100::mbar_wait(&full[s], (j / D2_NSTG) & 1);  // a1 planes of this image
      sm100::mbar_wait(&acc_full[acc], accph);
      sm100::tc_fence_after();
      const int Y = 2 * py + e;
#pragma unroll
      for (int pj = 0; pj < 2; ++pj) {
        const int cls = 2 * e + pj, X = 2 * px + pj;
        uint32_t r[32];
        c2_ld32(tmem_base + ((uint32_t)(32 * q) << 16) + acc * 128 + cls * 32, r);
        // ELU' operand: a1 class plane row m (64 B)
        const uint4* ap = reinterpret_cast<const uint4*>(stg + s * D2_STAGE + D2_ZBYTES + cls * 8192 + m * 64);
        uint4 av[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) av[c] = ap[c];
        sm100::tmem_ld_wait();
        const bool ok = Y < p.Hi && X < p.Wi;
        uint32_t o[16];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t ww[4] = {av[c].x, av[c].y, av[c].z, av[c].w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float a0 = __uint_as_float(ww[t] << 16), a1v = __uint_as_float(ww[t] & 0xFFFF0000u);
            const float v0 = __uint_as_float(r[8 * c + 2 * t]) * (a0 > 0.0f ? 1.0f : a0 + 1.0f);
            const float v1 = __uint_as_float(r[8 * c + 2 * t + 1]) * (a1v > 0.0f ? 1.0f : a1v + 1.0f);
            o[4 * c + t] = c2_bf16x2(v0, v1);
          }
        }
        // stage the warp's 32 output pixels (box order: coarse row, px; 64 B each)
        // and write them with one TMA store (the strided pixels of a class; X = Wi
        // is clipped): per-lane stores at a 128-byte stride were LSU-bound
        uint8_t* ob = osm + (ew * 2 + pj) * 2048;
        tma_store_wait_read_warp(pj);  // this buffer's previous store has read it
        uint4* sdst = reinterpret_cast<uint4*>(ob + lane * 64);
#pragma unroll
        for (int c = 0; c < 4; ++c) sdst[c] = make_uint4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        sm100::tma_store_4d_warp(&map_out, ob, 0, pj, 4 * q + e, img);
        if (ok) {
#pragma unroll
          for (int k = 0; k < 16; ++k) {  // the stored (rounded) values feed the bias gradient
            bs[2 * k] += __uint_as_float(o[k] << 16);
            bs[2 * k + 1] += __uint_as_float(o[k] & 0xFFFF0000u);
          }
        }
      }
      {  // input row 16 (coarse row 8) meets only dz2 rows >= Ho: its zeros are
         // stored here (a memset node would end the kernels' PDL overlap)
        uint4* zr = reinterpret_cast<uint4*>(p.dz + ((size_t)img * p.Hi + 16) * p.Wi * 32);
        for (int i = ew * 32 + lane; i < p.Wi * 4; i += 8 * 32) zr[i] = make_uint4(0, 0, 0, 0);
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        sm100::mbar_arrive(&acc_empty[acc]);
        sm100::mbar_arrive(&empty[s]);
      }
      if (++acc == 2) { acc = 0; accph ^= 1; }
    }
    sm100::tma_store_wait_all();  // stores read their smem before the CTA exits
    // bias gradient: lanes -> 32 column sums per warp -> fixed-point atomics
    float lo[16], hi[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      lo[k] = bs[k];
      hi[k] = bs[16 + k];
    }
    const float s_lo = d2_reduce16(lo, lane), s_hi = d2_reduce16(hi, lane);  // lane l < 16: column l (+16)
    if (lane < 16) {
      atomicAdd(p.bacc + (size_t)(blockIdx.x % 16) * 32 + lane,
                (unsigned long long)llrint((double)s_lo * 4294967296.0));
      atomicAdd(p.bacc + (size_t)(blockIdx.x % 16) * 32 + 16 + lane,
                (unsigned long long)llrint((double)s_hi * 4294967296.0));
    }
    __threadfence();
    asm volatile("bar.sync 1, %0;" ::"n"(32 * D2_EPI_WARPS) : "memory");  // epilogue warps only
    if (ew == 0 && lane == 0) last_cta = atomicAdd(p.bcnt, 1u) == gridDim.x - 1;
    asm volatile("bar.sync 1, %0;" ::"n"(32 * D2_EPI_WARPS) : "memory");
    if (last_cta) {
      __threadfence();
      const int et = threadIdx.x - 64;
      if (et < 32) {
        unsigned long long v = 0;
        for (int k = 0; k < 16; ++k) v += atomicExch(p.bacc + (size_t)k * 32 + et, 0ull);
        p.bout[et] = (float)((double)(long long)v * (1.0 / 4294967296.0));
      }
      if (et == 0) *p.bcnt = 0;
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem_base, 256);
  }
}

// ---- conv2 weight gradient with the same planes ----------------------------
// dW2[co][2a+e][2b+pj][ci] = sum over pixels k = y*16 + x of P_e[k + 16a + b][(pj, ci)]
// * dz2[k][co], P_e = the even / odd-row pixel-pair planes of conv2_s2d_kernel.
// Per image and (a, e): one chain of 7 K16 pixel steps with A = plane e from row
// 16a on as an MN-major operand whose two M atoms are the column taps b = 0, 1
// (LBO 128 B: one pixel row) and B = the dz2 rows (TMA box {64, 16, 7}: columns
// x >= Wo are zero, so padding pixels add nothing); the four accumulators live in
// TMEM for the CTA's share of images, are written once (per-CTA partials) and
// reduced deterministically by splitk_reduce.
constexpr int W2_NSTG = 3;
constexpr int W2_DBYTES = 16 * 1024;                 // dz2 rows (112 used) x 128 B
constexpr int W2_STAGE = 2 * C2_PLANE + W2_DBYTES;
constexpr int W2_THREADS = 32 * 6;                   // TMA, MMA, 4 epilogue warps
constexpr int W2_SMEM = 1024 + W2_NSTG * W2_STAGE + 256;

struct W2Params {
  int n_img, Ho;
  float* partial;  // [gridDim.x][64 co][512 = (kh, kw, ci)]
};

__global__ void __launch_bounds__(W2_THREADS, 1)
    conv2_wgrad_kernel(const __grid_constant__ CUtensorMap map_a1,
                       const __grid_constant__ CUtensorMap map_dz2, const __grid_constant__ W2Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + W2_NSTG * W2_STAGE);
  uint64_t* full = bars;
  uint64_t* empty = full + W2_NSTG;
  uint64_t* done = empty + W2_NSTG;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int plane_rows = (p.Ho + 1) * 16;
  if (threadIdx.x == 0) {
    sm100::tma_prefetch(&map_a1);
    sm100::tma_prefetch(&map_dz2);
    for (int s = 0; s < W2_NSTG; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    sm100::mbar_init(done, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 1) {
    sm100::tmem_alloc(tmem_slot, 256);
    sm100::tmem_relinquish();
  }
  // plane rows past the TMA box meet dz2 zeros only: finite zeros
  for (int e = threadIdx.x; e < W2_NSTG * 2 * (C2_PROWS - plane_rows) * 8; e += W2_THREADS) {
    const int pl = e / ((C2_PROWS - plane_rows) * 8), r = e % ((C2_PROWS - plane_rows) * 8);
    reinterpret_cast<uint4*>(smem + (pl >> 1) * W2_STAGE + (pl & 1) * C2_PLANE + plane_rows * 128)[r] =
        make_uint4(0, 0, 0, 0);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  APPO_PDL_ENTRY();  // a1 / dz2 come from earlier kernels
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    int j = 0;
    for (int img = blockIdx.x; img < p.n_img; img += gridDim.x, ++j) {
      const int s = j % W2_NSTG;
      sm100::mbar_wait(&empty[s], ((j / W2_NSTG) & 1) ^ 1);
      uint8_t* base = smem + s * W2_STAGE;
      sm100::mbar_arrive_expect_tx_warp(&full[s], 2u * plane_rows * 128 + (uint32_t)p.Ho * 16 * 128);
      sm100::tma_load_4d_warp(base, &map_a1, &full[s], 0, 0, 0, img);
      sm100::tma_load_4d_warp(base + C2_PLANE, &map_a1, &full[s], 0, 0, 1, img);
      sm100::tma_load_4d_warp(base + 2 * C2_PLANE, &map_dz2, &full[s], 0, 0, 0, img);
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = sm100::make_idesc_bf16(128, 64, 1, 1);
    const uint32_t s0 = sm100::smem_u32(smem);
    int j = 0;
    const int ksteps = p.Ho;  // 16-pixel K steps: Ho rows x 16 columns
    for (int img = blockIdx.x; img < p.n_img; img += gridDim.x, ++j) {
      const int s = j % W2_NSTG;
      sm100::mbar_wait(&full[s], (j / W2_NSTG) & 1);
      sm100::tc_fence_after();
      const uint32_t st = s0 + s * W2_STAGE;
#pragma unroll
      for (int blk = 0; blk < 4; ++blk) {  // (a, e) = (blk >> 1, blk & 1)
        const int a = blk >> 1, e = blk & 1;
        for (int ks = 0; ks < ksteps; ++ks) {
          const uint64_t ad = sm100::make_sdesc(st + e * C2_PLANE + (16 * a + 16 * ks) * 128, 128, 1024);
          const uint64_t bd = sm100::make_sdesc(st + 2 * C2_PLANE + ks * 2048, 8192, 1024);
          sm100::umma_f16_warp(tmem_base + blk * 64, ad, bd, idesc, (j | ks) ? 1u : 0u);
        }
      }
      sm100::umma_commit_warp(&empty[s]);
    }
    sm100::umma_commit_warp(done);
  } else {
    // ---- final epilogue: TMEM row m = (b = m >> 6, pj = (m >> 5) & 1, ci = m & 31) ----
    sm100::mbar_wait(done, 0);
    sm100::tc_fence_after();
    const int q = warp & 3, m = 32 * q + lane;
    const int b = m >> 6, pj = (m >> 5) & 1, ci = m & 31;
    float* out = p.partial + (size_t)blockIdx.x * 64 * 512;
#pragma unroll
    for (int blk = 0; blk < 4; ++blk) {
      const int kh = 2 * (blk >> 1) + (blk & 1), kw = 2 * b + pj;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t r[32];
        c2_ld32(tmem_base + ((uint32_t)(32 * q) << 16) + blk * 64 + h * 32, r);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; ++c)
          out[(size_t)(h * 32 + c) * 512 + (kh * 4 + kw) * 32 + ci] = __uint_as_float(r[c]);
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem_base, 256);
  }
}

}  // namespace

const void* kanchor_conv2() { return reinterpret_cast<const void*>(&conv2_s2d_kernel); }

int conv2_s2d_forward(Ctx* c, const uint16_t* a1, int n_img, int Hi, int Wi, int Ho, int Wo,
                      const uint16_t* w2, const Epilogue& e) {
  if (n_img <= 0) return APPO_OK;
  // k4 s2 geometry, one 128-row tile per image, 16-byte aligned rows for TMA
  if (Ho != (Hi - 4) / 2 + 1 || Wo != (Wi - 4) / 2 + 1 || Ho * 16 > 128 || Wo + 1 > 16 ||
      e.flags != (EPI_BIAS | EPI_ELU | EPI_BF16) || e.ldo != 64 || !e.bias ||
      (reinterpret_cast<uintptr_t>(a1) & 15) || (reinterpret_cast<uintptr_t>(e.out) & 15) ||
      (Wi * 64) % 16 || (reinterpret_cast<uintptr_t>(w2) & 15))
    return APPO_ERR_CONTRACT;
  // pixel-pair view of a1 [img][Hi][Wi][32] bf16: {64, Wi/2 pairs, Hi rows, n_img};
  // box {64, 16 pairs, Ho+1 rows at stride 2, 1} (pairs / rows outside -> 0)
  EncodeTiledFnPublic enc = tensor_map_encoder();
  if (!enc) return APPO_ERR_RESOURCE;
  CUtensorMap map;
  cuuint64_t dims[4] = {64, (cuuint64_t)(Wi / 2), (cuuint64_t)Hi, (cuuint64_t)n_img};
  cuuint64_t str[3] = {128, (cuuint64_t)Wi * 64, (cuuint64_t)Hi * Wi * 64};
  cuuint32_t box[4] = {64, 16, (cuuint32_t)(2 * (Ho + 1)), 1};
  cuuint32_t es[4] = {1, 1, 2, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(a1), dims, str, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return APPO_ERR_CONTRACT;
  CUtensorMap wmap;  // W2 [64 co][4 kh][4 kw][32 ci] as {64 (kw pair x ci), 2, 4, 64}
  {
    cuuint64_t dims[4] = {64, 2, 4, 64};
    cuuint64_t str[3] = {128, 256, 1024};
    cuuint32_t box[4] = {64, 2, 1, 64};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&wmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(w2), dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return APPO_ERR_CONTRACT;
  }
  C2Params p{};
  p.n_img = n_img;
  p.Ho = Ho;
  p.Wo = Wo;
  p.plane_rows = (Ho + 1) * 16;
  p.w = w2;
  p.bias = e.bias;
  p.out = reinterpret_cast<uint16_t*>(e.out);
  static int attr_bytes[64] = {};
  const int dev = c->device & 63;
  if (attr_bytes[dev] < C2_SMEM) {
    APPO_CUDA_TRY(cudaFuncSetAttribute(conv2_s2d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       C2_SMEM));
    attr_bytes[dev] = C2_SMEM;
  }
  const int grid = c->num_sms < n_img ? c->num_sms : n_img;
  c->next_name = "conv2_s2d_tcgen05";
  c->next_flops = 2.0 * n_img * Ho * Wo * 64 * 512;
  c->next_bytes = 2.0 * n_img * ((double)Hi * Wi * 32 + (double)Ho * Wo * 64) + 2.0 * 64 * 512;
  APPO_LAUNCH(c, conv2_s2d_kernel, grid, C2_THREADS, C2_SMEM, map, wmap, p);
  return APPO_OK;
}

int conv2_dgrad(Ctx* c, const DgradIn& in) {
  if (!(in.N == 32 && in.Co == 64 && in.k == 4 && in.Hi == 17 && in.Wi == 31 && in.Ho == 7 &&
        in.Wo == 14 && in.bias.out && in.bias.acc && in.bias.counter && in.n_img > 0 &&
        !((reinterpret_cast<uintptr_t>(in.dz_next) | reinterpret_cast<uintptr_t>(in.dz) |
           reinterpret_cast<uintptr_t>(in.aprev)) & 15)))
    return APPO_ERR_CONTRACT;
  EncodeTiledFnPublic enc = tensor_map_encoder();
  if (!enc) return APPO_ERR_RESOURCE;
  CUtensorMap mz, ma;
  {  // dz2 [img][7][14][64], box {64, 16, 9, 1} from (-1, -1): zero border, SW128
    cuuint64_t dims[4] = {64, (cuuint64_t)in.Wo, (cuuint64_t)in.Ho, (cuuint64_t)in.n_img};
    cuuint64_t str[3] = {128, (cuuint64_t)in.Wo * 128, (cuuint64_t)in.Ho * in.Wo * 128};
    cuuint32_t box[4] = {64, 16, 9, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&mz, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(in.dz_next), dims, str,
            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return APPO_ERR_CONTRACT;
  }
  {  // a1 [img][17][31][32] class planes: box {32, 32 (x stride 2), 16 (y stride 2), 1}
    cuuint64_t dims[4] = {32, (cuuint64_t)in.Wi, (cuuint64_t)in.Hi, (cuuint64_t)in.n_img};
    cuuint64_t str[3] = {64, (cuuint64_t)in.Wi * 64, (cuuint64_t)in.Hi * in.Wi * 64};
    cuuint32_t box[4] = {32, 32, 16, 1};
    cuuint32_t es[4] = {1, 2, 2, 1};
    if (enc(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(in.aprev), dims, str,
            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return APPO_ERR_CONTRACT;
  }
  CUtensorMap mo;
  {  // dz1 class boxes (TMA stores): box {32, 32 (x stride 2), 4 (y stride 2), 1}, X = Wi clipped
    cuuint64_t dims[4] = {32, (cuuint64_t)in.Wi, (cuuint64_t)in.Hi, (cuuint64_t)in.n_img};
    cuuint64_t str[3] = {64, (cuuint64_t)in.Wi * 64, (cuuint64_t)in.Hi * in.Wi * 64};
    cuuint32_t box[4] = {32, 32, 4, 1};
    cuuint32_t es[4] = {1, 2, 2, 1};
    if (enc(&mo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, in.dz, dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return APPO_ERR_CONTRACT;
  }
  CUtensorMap mw;  // wt [128 rows (class, ci)][256 (tap, co)], box {64, 128, 1}
  {
    const int st = make_tmap_bf16_3d(&mw, in.wt, 256, 128, 1, 512, 128 * 512, 64, 128, 1);
    if (st) return st;
  }
  D2Params p{};
  p.n_img = in.n_img;
  p.Hi = in.Hi;
  p.Wi = in.Wi;
  p.wt = in.wt;
  p.dz = in.dz;
  p.bacc = in.bias.acc;
  p.bcnt = in.bias.counter;
  p.bout = in.bias.out;
  static int attr_bytes[64] = {};
  const int dev = c->device & 63;
  if (attr_bytes[dev] < D2_SMEM) {
    APPO_CUDA_TRY(cudaFuncSetAttribute(conv2_dgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       D2_SMEM));
    attr_bytes[dev] = D2_SMEM;
  }
  const int grid = c->num_sms < in.n_img ? c->num_sms : in.n_img;
  c->next_name = "conv2_dgrad_s2d_tcgen05";
  c->next_flops = 2.0 * in.n_img * in.Hi * in.Wi * 32.0 * 64 * 4;
  c->next_bytes = 2.0 * in.n_img * ((double)in.Ho * in.Wo * 64 + 2.0 * in.Hi * in.Wi * 32);
  APPO_LAUNCH(c, conv2_dgrad_kernel, grid, D2_THREADS, D2_SMEM, mz, ma, mo, mw, p);
  return APPO_OK;
}

int conv2_wgrad(Ctx* c, const uint16_t* a1, int n_img, int Hi, int Wi, const uint16_t* dz2, int Ho,
                int Wo, float* dw) {
  if (n_img <= 0) return APPO_OK;
  if (Ho != (Hi - 4) / 2 + 1 || Wo != (Wi - 4) / 2 + 1 || Ho * 16 > 128 || Wo + 1 > 16 ||
      ((reinterpret_cast<uintptr_t>(a1) | reinterpret_cast<uintptr_t>(dz2)) & 15) || (Wi * 64) % 16)
    return APPO_ERR_CONTRACT;
  EncodeTiledFnPublic enc = tensor_map_encoder();
  if (!enc) return APPO_ERR_RESOURCE;
  CUtensorMap ma, mz;
  {  // the conv2_s2d_kernel planes: pixel pairs, rows at stride 2
    cuuint64_t dims[4] = {64, (cuuint64_t)(Wi / 2), (cuuint64_t)Hi, (cuuint64_t)n_img};
    cuuint64_t str[3] = {128, (cuuint64_t)Wi * 64, (cuuint64_t)Hi * Wi * 64};
    cuuint32_t box[4] = {64, 16, (cuuint32_t)(2 * (Ho + 1)), 1};
    cuuint32_t es[4] = {1, 1, 2, 1};
    if (enc(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(a1), dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return APPO_ERR_CONTRACT;
  }
  {  // dz2 [img][Ho][Wo][64]: box {64, 16, Ho, 1} (x >= Wo -> 0)
    cuuint64_t dims[4] = {64, (cuuint64_t)Wo, (cuuint64_t)Ho, (cuuint64_t)n_img};
    cuuint64_t str[3] = {128, (cuuint64_t)Wo * 128, (cuuint64_t)Ho * Wo * 128};
    cuuint32_t box[4] = {64, 16, (cuuint32_t)Ho, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&mz, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(dz2), dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return APPO_ERR_CONTRACT;
  }
  const int grid = c->num_sms < n_img ? c->num_sms : n_img;
  float* part = nullptr;
  const int wst = gemm_workspace(c, (size_t)grid * 64 * 512 * sizeof(float), &part);
  if (wst) return wst;
  W2Params p{};
  p.n_img = n_img;
  p.Ho = Ho;
  p.partial = part;
  static int attr_bytes[64] = {};
  const int dev = c->device & 63;
  if (attr_bytes[dev] < W2_SMEM) {
    APPO_CUDA_TRY(cudaFuncSetAttribute(conv2_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       W2_SMEM));
    attr_bytes[dev] = W2_SMEM;
  }
  c->next_name = "conv2_wgrad_s2d_tcgen05";
  c->next_flops = 2.0 * n_img * Ho * Wo * 64.0 * 512;
  c->next_bytes = 2.0 * n_img * ((double)Hi * Wi * 32 + (double)Ho * Wo * 64) + 4.0 * grid * 64 * 512;
  APPO_LAUNCH(c, conv2_wgrad_kernel, grid, W2_THREADS, W2_SMEM, ma, mz, p);
  Epilogue e;
  e.out = dw;
  e.ldo = 512;
  return splitk_reduce(c, 64, 512, grid, part, e);
}

}  // namespace appo_b200
