// conv1 forward (k8 s4, u8 CHW observations -> 32 channels, ELU, bf16 NHWC)
// as a space-to-depth "taps" GEMM on tcgen05 (sm_100a).
//
// A k8 s4 convolution is, after space-to-depth by 4 (Z[py][px][c,i,j] =
// X[c][4py+i][4px+j], C*16 values per s2d pixel), a k2 s1 convolution:
//   out[y][x] = sum_{a,b in {0,1}} Z[y+a][x+b] . W_ab        (W_ab: [32][C*16])
// With the s2d rows of a tile stored ONCE in shared memory as a K-major
// SWIZZLE_128B matrix (one 128-byte row per s2d pixel: its C*16 values, zero
// padded to 64), the operand "Z shifted by (a, b)" is the same smem matrix with
// its descriptor start moved by (32a + b) rows: the four taps are four MMA
// chains (N = 32, C K16 steps each) into ONE TMEM accumulator, and every
// observation byte is converted to fp16 once (the im2col form of gemm.cu's
// AG_U8 path builds every byte 4 times).  (Measured alternative: the column
// taps as the two halves of an N = 64 B operand summed by a lane shuffle in the
// epilogue -- half the MMAs, but the shuffles and the wider TMEM reads made the
// issue-bound epilogue slower: 312 vs 281 us per 16 K images.)  Pipeline
// (warp-specialised, persistent, one CTA per SM):
//   warp 0        TMA: whole image {W, 4*Hs rows, C} per box into a staging ring
//   warp 1        TMEM owner + MMA issuer (4 taps x C K-steps of M128 N32 K16)
//   warps 2..9    converters: staged u8 -> fp16 (1024 + v, exact) s2d windows
//   warps 10..17  epilogue: TMEM -> scale/bias/ELU -> bf16 rows of a1 (2 warps
//                 per TMEM lane quarter, 16 output channels each)
// The 1024 offset is removed through the corrected bias of the published copy
// (k_conv1_half_weights), so A is exact and B is the fp16 weights.
//
// Replaces: the reference has no convolutional encoder (SURVEY.md §8 a2,
// SPEC.md:273-274); this is convnet_simple's conv1 of the model contract
// (DESIGN.md §2), parity-checked against the fp64 oracle (tests/test_model_gpu.py,
// tests/test_parity_prod_gpu.py) exactly like the engine path it replaces.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "appo_common.cuh"
#include "gemm.cuh"
#include "sm100.cuh"

namespace appo_b200 {
namespace {

#ifndef C1_CONV_WARPS_DEF
#define C1_CONV_WARPS_DEF 8
#endif
#ifndef C1_EPI_PARTS_DEF
#define C1_EPI_PARTS_DEF 2
#endif
constexpr int C1_CONV_WARPS = C1_CONV_WARPS_DEF;
constexpr int C1_TMA = 0, C1_MMA = 1;  // warp roles (MMA on warp 0 measured no faster)
constexpr int C1_EPI_PARTS = C1_EPI_PARTS_DEF;  // epilogue warps per TMEM lane quarter
constexpr int C1_EPI_WARPS = 4 * C1_EPI_PARTS;
constexpr int C1_EPI_CO = 32 / C1_EPI_PARTS;    // output channels per epilogue warp
constexpr int C1_THREADS = 32 * (2 + C1_CONV_WARPS + C1_EPI_WARPS);
#ifndef C1_NSTG_DEF
#define C1_NSTG_DEF 3
#endif
#ifndef C1_NA_DEF
#define C1_NA_DEF 4
#endif
constexpr int C1_NSTG = C1_NSTG_DEF;  // staged images in flight
constexpr int C1_NA = C1_NA_DEF;      // s2d A windows (one per 128-row tile)
constexpr int C1_NACC = 4;    // TMEM accumulators (64 columns apart; 32 used)
constexpr int C1_WROWS = 168; // window rows: 5 s2d rows x 32 px + 1 (x-tap overrun), to 8
constexpr int C1_WBYTES = C1_WROWS * 128;  // one window (SW128 rows, 1024-aligned)

struct C1Params {
  int n_img, C, H, W, Ho, Wo, Hs;  // Hs = Ho + 1 s2d rows are read
  int tiles;                       // 128-row tiles per image = ceil(Ho / 4)
  int box_rows;                    // 4 * Hs input rows staged per image
  int stg_bytes;                   // staging slot bytes (C * box_rows * W, 128-aligned)
  int slack;                       // bytes after the ring read by the last tile's padding rows
  // trajectory-slot images: r < n_traj*T is step r % T of slot slot_ids[r / T],
  // later ones the bootstrap observation of slot slot_ids[r - n_traj*T]
  const int32_t* slot_ids;
  int T, n_traj;
  const uint16_t* w;  // fp16 [32][C*64], k = c*64 + kh*8 + kw (published copy)
  const float* bias;  // corrected bias (offset 1024 * sum(W) * scale removed)
  float scale;
  uint16_t* out;      // bf16 [n_img * Ho * Wo][ldo]
  int64_t ldo;
  long long* prof;    // diagnostics (APPO_C1_PROF): CTA 0 per-tile timestamps [64][16]
};
#ifdef C1_PROF_ON  // per-tile timeline of CTA 0 (build with -DC1_PROF_ON, run with APPO_C1_PROF=1)
#define C1_PROF(tile, k)                                                   \
  do {                                                                     \
    if (p.prof && blockIdx.x == 0 && (tile) < 64) p.prof[(tile) * 16 + (k)] = clock64(); \
  } while (0)
#else
#define C1_PROF(tile, k) \
  do {                   \
  } while (0)
#endif

constexpr int C1_BBYTES = 2 * 64 * 128;     // 2 row taps x (2 column taps x 32 channels), SW128 rows
int c1_smem_bytes(int stg_bytes, int slack) {
  return 1024 + C1_NA * C1_WBYTES + C1_BBYTES + C1_NSTG * stg_bytes + slack + 256;
}
// Converters read input rows up to 16 * tiles + 3 of every channel (the last
// tile's rows past the image): slack after the ring so the last slot's reads
// stay inside the allocation (a W-wide row per row past 4 * Hs, + 128)
int c1_slack(int tiles, int box_rows, int W) {
  const int over = 16 * tiles + 4 - box_rows;
  return ((over > 0 ? over : 0) * W + 128 + 127) & ~127;
}

// A K-major SWIZZLE_128B descriptor may start at any 128-byte row of the
// 1024-byte swizzle pattern with base offset 0: the XOR pattern follows the
// absolute shared-memory address (measured: setting the row phase in the
// base-offset field, bits 49-51, gives wrong products), so a row shift of the
// operand is only a start-address change.


// MN-major SWIZZLE_64B descriptor (atoms of 32 bf16 MN elements x 8 K rows of
// 64 B): lbo = stride between MN atoms, sbo = between 8-row K groups
__device__ __forceinline__ uint64_t sdesc_mn_sw64(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  d |= (uint64_t)4 << 61;  // SWIZZLE_64B
  return d;
}

__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// packed fp32 pairs (sm_100 FFMA2 / FADD2): half the epilogue's FP instructions
__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 f2unpack(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
// 32 lanes x 32-bit, 32 consecutive TMEM columns per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
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
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

template <int C>
__global__ void __launch_bounds__(C1_THREADS, 1)
    conv1_s2d_kernel(const __grid_constant__ CUtensorMap map_obs,
                     const __grid_constant__ CUtensorMap map_boot, const __grid_constant__ C1Params p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base derived by pointer arithmetic from smem_raw, so the
  // compiler keeps the shared address space (LDS/STS, not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* awin = smem;                                  // C1_NA s2d windows (SW128 rows)
  uint8_t* bsm = awin + C1_NA * C1_WBYTES;               // 4 taps x 32 rows (SW128)
  uint8_t* stg = bsm + C1_BBYTES;                        // C1_NSTG staged images
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg + C1_NSTG * p.stg_bytes + p.slack);
  uint64_t* stg_full = bars;
  uint64_t* stg_empty = stg_full + C1_NSTG;
  uint64_t* a_full = stg_empty + C1_NSTG;
  uint64_t* a_empty = a_full + C1_NA;
  uint64_t* acc_full = a_empty + C1_NA;
  uint64_t* acc_empty = acc_full + C1_NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + C1_NACC);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    sm100::tma_prefetch(&map_obs);
    if (p.slot_ids) sm100::tma_prefetch(&map_boot);
    for (int s = 0; s < C1_NSTG; ++s) {
      sm100::mbar_init(&stg_full[s], 1);
      sm100::mbar_init(&stg_empty[s], C1_CONV_WARPS);
    }
    for (int s = 0; s < C1_NA; ++s) {
      sm100::mbar_init(&a_full[s], C1_CONV_WARPS);
      sm100::mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < C1_NACC; ++s) {
      sm100::mbar_init(&acc_full[s], 1);
      sm100::mbar_init(&acc_empty[s], C1_EPI_WARPS);
    }
    sm100::fence_barrier_init();
  }
  if (warp == C1_MMA) {
    sm100::tmem_alloc(tmem_slot, C1_NACC * 64);
    sm100::tmem_relinquish();
  }
  // B operand of row tap a: row n = (output channel co = n >> 1, column tap
  // b = n & 1), chunk kc = 2c + h holds 8 fp16 W[co][c][4a + 2h + ii][4b + j]
  // (ii = 0, 1; j = 0..3), the same (ii, j) order as the A chunks
  // (A/B variant) B of tap tau = 2a + b: row co, 32 rows per tap
  for (int e = threadIdx.x; e < 4 * 2 * C * 32; e += C1_THREADS) {
    const int co = e & 31, kc = (e >> 5) % (2 * C), tau = (e >> 5) / (2 * C);
    const int c = kc >> 1, h = kc & 1, a = tau >> 1, b = tau & 1;
    const uint16_t* src = p.w + (size_t)co * (C * 64) + c * 64 + (4 * a + 2 * h) * 8 + 4 * b;
    const uint2 lo = *reinterpret_cast<const uint2*>(src);
    const uint2 hi = *reinterpret_cast<const uint2*>(src + 8);
    *reinterpret_cast<uint4*>(bsm + tau * 4096 + co * 128 + ((kc ^ (co & 7)) << 4)) =
        make_uint4(lo.x, lo.y, hi.x, hi.y);
  }
  // the weights are a published copy (an earlier step): staged before the wait,
  // overlapping the previous kernel; the images come from earlier kernels
  APPO_PDL_ENTRY();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int B = p.n_traj * p.T;

  if (warp == C1_TMA) {
    // ---- TMA producer: one box per image ----
    int j = 0;
    for (int img = blockIdx.x; img < p.n_img; img += gridDim.x, ++j) {
      const int s = j % C1_NSTG;
      sm100::mbar_wait(&stg_empty[s], ((j / C1_NSTG) & 1) ^ 1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      sm100::mbar_arrive_expect_tx_warp(&stg_full[s], (uint32_t)(C * p.box_rows * p.W));
      uint8_t* dst = stg + s * p.stg_bytes;
      if (lane == 0) C1_PROF(j * p.tiles, 0);
      if (!p.slot_ids) {
        sm100::tma_load_4d_warp(dst, &map_obs, &stg_full[s], 0, 0, 0, img);
      } else if (img < B) {
        sm100::tma_load_5d_warp(dst, &map_obs, &stg_full[s], 0, 0, 0, img % p.T,
                                __ldg(p.slot_ids + img / p.T));
      } else {
        sm100::tma_load_4d_warp(dst, &map_boot, &stg_full[s], 0, 0, 0, __ldg(p.slot_ids + img - B));
      }
    }
  } else if (warp == C1_MMA) {
    // ---- MMA issuer: per tile, 2 row taps x C K16 steps into one accumulator ----
    constexpr uint32_t idesc = sm100::make_idesc_f16(128, 32, 0, 0);
    const uint32_t a0 = sm100::smem_u32(awin), b0 = sm100::smem_u32(bsm);
    int a = 0, acc = 0, tile_i = 0;
    uint32_t aph = 0, accph = 0;
    for (int img = blockIdx.x; img < p.n_img; img += gridDim.x) {
      for (int t = 0; t < p.tiles; ++t) {
        sm100::mbar_wait(&a_full[a], aph);
        if (lane == 0) C1_PROF(tile_i, 8);
        sm100::mbar_wait(&acc_empty[acc], accph ^ 1);
        sm100::tc_fence_after();
        if (lane == 0) C1_PROF(tile_i, 3);
        const uint32_t d = tmem_base + acc * 64;
        const uint32_t abase = a0 + a * C1_WBYTES;
#pragma unroll
        for (int tau = 0; tau < 4; ++tau) {
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const uint64_t ad = sm100::make_sdesc(
                abase + (32 * (tau >> 1) + (tau & 1)) * 128 + c * 32, 16, 1024);
            const uint64_t bd = sm100::make_sdesc(b0 + tau * 4096 + c * 32, 16, 1024);
            sm100::umma_f16_warp(d, ad, bd, idesc, (tau | c) ? 1u : 0u);
          }
        }
        sm100::umma_commit_warp(&a_empty[a]);
        sm100::umma_commit_warp(&acc_full[acc]);
        if (lane == 0) C1_PROF(tile_i, 4);
        ++tile_i;
        if (++a == C1_NA) { a = 0; aph ^= 1; }
        if (++acc == C1_NACC) { acc = 0; accph ^= 1; }
      }
    }
  } else if (warp < 2 + C1_CONV_WARPS) {
    // ---- converters: lane = s2d column px (window row pyl*32 + px); unit = (pyl, chunk) ----
    // plain C++ shared-memory accesses (not asm volatile) so the fully unrolled
    // units' loads are issued together: the loop is LDS-latency bound otherwise
    const int cw = warp - 2;
    constexpr int kUnits = 5 * 2 * C;
    constexpr int kPerWarp = (kUnits + C1_CONV_WARPS - 1) / C1_CONV_WARPS;
    // per unit k of this warp: staging offset of its two input rows (tile 0) and
    // its window offset; every unit is converted for every tile (rows past the
    // image read the staging slack and only feed output rows that are dropped)
    uint32_t soff[kPerWarp], doff[kPerWarp];
#pragma unroll
    for (int k = 0; k < kPerWarp; ++k) {
      const int u = min(cw + k * C1_CONV_WARPS, kUnits - 1);
      const int pyl = u / (2 * C), kc = u - pyl * 2 * C;
      soff[k] = (uint32_t)(((kc >> 1) * p.box_rows + 4 * pyl + 2 * (kc & 1)) * p.W + 4 * lane);
      doff[k] = (uint32_t)(lane * 128 + pyl * 4096 + ((kc ^ (lane & 7)) << 4));
    }
    const uint32_t tstep = 16u * p.W;  // staging bytes per tile (4 s2d rows x 4 input rows)
    int j = 0, a = 0;
    uint32_t aph = 0;
    for (int img = blockIdx.x; img < p.n_img; img += gridDim.x, ++j) {
      const int s = j % C1_NSTG;
      sm100::mbar_wait(&stg_full[s], (j / C1_NSTG) & 1);
      const uint8_t* src0 = stg + s * p.stg_bytes;
      for (int t = 0; t < p.tiles; ++t, src0 += tstep) {
        sm100::mbar_wait(&a_empty[a], aph ^ 1);
        if (cw == 0 && lane == 0) C1_PROF(j * p.tiles + t, 1);
        uint8_t* dst0 = awin + a * C1_WBYTES;
        uint32_t lo[kPerWarp], hi[kPerWarp];
#pragma unroll
        for (int k = 0; k < kPerWarp; ++k) {
          lo[k] = *reinterpret_cast<const uint32_t*>(src0 + soff[k]);
          hi[k] = *reinterpret_cast<const uint32_t*>(src0 + soff[k] + p.W);
        }
#pragma unroll
        for (int k = 0; k < kPerWarp; ++k)  // SW128 row: chunk kc at (kc ^ (row & 7))
          *reinterpret_cast<uint4*>(dst0 + doff[k]) =
              make_uint4(__byte_perm(lo[k], 0x64646464u, 0x4140),
                         __byte_perm(lo[k], 0x64646464u, 0x4342),
                         __byte_perm(hi[k], 0x64646464u, 0x4140),
                         __byte_perm(hi[k], 0x64646464u, 0x4342));
        if (cw == 0 && lane == 0) C1_PROF(j * p.tiles + t, 7);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> UMMA
        __syncwarp();
        if (cw == 0 && lane == 0) C1_PROF(j * p.tiles + t, 2);
        if (cw == C1_CONV_WARPS - 1 && lane == 0) C1_PROF(j * p.tiles + t, 9);
        if (lane == 0) sm100::mbar_arrive(&a_full[a]);
        if (++a == C1_NA) { a = 0; aph ^= 1; }
      }
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&stg_empty[s]);
    }
  } else {
    // ---- epilogue: warp quarter q = TMEM lanes (output row 4t + q), 16 output
    // channels = 32 TMEM columns (co, b) ----
    const int ew = warp - (2 + C1_CONV_WARPS);
    const int q = warp & 3, part = ew >> 2;
    constexpr float kLog2e = 1.4426950408889634f;
    uint64_t bias2[C1_EPI_CO / 2], bias2l[C1_EPI_CO / 2];  // bias, bias*log2(e) pairs
#pragma unroll
    for (int k = 0; k < C1_EPI_CO / 2; ++k) {
      const float b0 = __ldg(p.bias + part * C1_EPI_CO + 2 * k);
      const float b1 = __ldg(p.bias + part * C1_EPI_CO + 2 * k + 1);
      bias2[k] = f2pack(b0, b1);
      bias2l[k] = f2pack(b0 * kLog2e, b1 * kLog2e);
    }
    const uint64_t scale2 = f2pack(p.scale, p.scale);
    const uint64_t scale2l = f2pack(p.scale * kLog2e, p.scale * kLog2e);
    const uint64_t mone2 = f2pack(-1.0f, -1.0f);
    int acc = 0, tile_i = 0;
    uint32_t accph = 0;
    for (int img = blockIdx.x; img < p.n_img; img += gridDim.x) {
      // this lane's output pixel (row 4t + q, column lane) of the image, 8 channels
      uint16_t* obase = p.out + ((int64_t)img * p.Ho * p.Wo + (int64_t)q * p.Wo + lane) * p.ldo +
                        part * C1_EPI_CO;
      const int64_t tstride = 4 * (int64_t)p.Wo * p.ldo;
      for (int t = 0; t < p.tiles; ++t, ++tile_i, obase += tstride) {
        sm100::mbar_wait(&acc_full[acc], accph);
        sm100::tc_fence_after();
        if (ew == 0 && lane == 0) C1_PROF(tile_i, 5);
        const int y = 4 * t + q;
        if (y < p.Ho) {  // warp-uniform
          static_assert(C1_EPI_CO == 16, "4-tap variant: 16 channels per epilogue warp");
          uint32_t r[16];
          sm100::tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + acc * 64 + part * 16, r);
          sm100::tmem_ld_wait();
          if (ew == 0 && lane == 0) C1_PROF(tile_i, 11);
          uint32_t w[C1_EPI_CO / 2];
#pragma unroll
          for (int k = 0; k < C1_EPI_CO / 2; ++k) {
            const uint64_t v = f2pack(__uint_as_float(r[2 * k]), __uint_as_float(r[2 * k + 1]));
            const float2 x = f2unpack(ffma2(v, scale2, bias2[k]));
            const float2 tl = f2unpack(ffma2(v, scale2l, bias2l[k]));  // x * log2(e)
            const float2 e = f2unpack(fadd2(f2pack(ex2_ftz(fminf(tl.x, 0.0f)), ex2_ftz(fminf(tl.y, 0.0f))), mone2));
            // ELU = max(x, exp(min(x, 0)) - 1)
            w[k] = pack_bf16x2(fmaxf(x.x, e.x), fmaxf(x.y, e.y));
          }
          if (ew == 0 && lane == 0) C1_PROF(tile_i, 12);
          if (lane < p.Wo) {
            uint4* dst = reinterpret_cast<uint4*>(obase);
#pragma unroll
            for (int k = 0; k < C1_EPI_CO / 8; ++k)
              dst[k] = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
          }
        }
        sm100::tc_fence_before();
        __syncwarp();
        if (ew == 0 && lane == 0) C1_PROF(tile_i, 6);
        if (ew == C1_EPI_WARPS - 1 && lane == 0) C1_PROF(tile_i, 10);
        if (lane == 0) sm100::mbar_arrive(&acc_empty[acc]);
        if (++acc == C1_NACC) { acc = 0; accph ^= 1; }
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == C1_MMA) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem_base, C1_NACC * 64);
  }
}

template <int C>
int c1_launch(Ctx* c, const CUtensorMap& mo, const CUtensorMap& mbt, const C1Params& p) {
  auto kern = conv1_s2d_kernel<C>;
  const int smem = c1_smem_bytes(p.stg_bytes, p.slack);
  static int attr_bytes[64] = {};
  const int dev = c->device & 63;
  if (attr_bytes[dev] < smem) {
    APPO_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_bytes[dev] = smem;
  }
  const int grid = c->num_sms < p.n_img ? c->num_sms : p.n_img;
  C1Params q = p;
#ifdef C1_PROF_ON
  static long long* prof = nullptr;
  const char* pe = getenv("APPO_C1_PROF");
  if (pe && pe[0] == '1' && p.n_img > 4096) {
    if (!prof) cudaMalloc(&prof, sizeof(long long) * 1024);
    cudaMemsetAsync(prof, 0, sizeof(long long) * 1024, c->stream);
    q.prof = prof;
  }
#endif
  c->next_name = "conv1_s2d_tcgen05";
  const double M = (double)p.n_img * p.Ho * p.Wo;
  c->next_flops = 2.0 * M * 32 * C * 64;
  c->next_bytes = (double)p.n_img * C * p.H * p.W + 2.0 * M * 32 + 2.0 * 32 * C * 64;
  APPO_LAUNCH(c, kern, grid, C1_THREADS, smem, mo, mbt, q);
#ifdef C1_PROF_ON
  if (q.prof) {
    long long h[1024];
    cudaStreamSynchronize(c->stream);
    cudaMemcpy(h, prof, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[conv1 prof] CTA0 tile: tma_issue conv_start conv_done | mma_start mma_issued | epi_start epi_done | conv_stores_issued mma_afull conv7_done epi7_done (cycles from first TMA)\n");
    for (int i = 0; i < 64; ++i) {
      fprintf(stderr, "  t%-2d", i);
      for (int k = 0; k < 13; ++k) fprintf(stderr, " %8lld", h[i * 16 + k] ? h[i * 16 + k] - h[0] : -1);
      fprintf(stderr, "\n");
    }
  }
#endif
  return APPO_OK;
}

// ---- conv1 weight gradient in the same space-to-depth form ----------------
// dW[co][c][4a+i][4b+j] = sum_{Y,x} Z[Y][x+b][(c,i,j)] * dz1[Y-a][x][co]: per
// tile of 4 s2d rows Y (128 pixels), ONE MMA chain of 8 K16 pixel steps with
// A = the s2d window as an MN-major SW128 operand whose two 64-row M atoms are
// the column taps b = 0, 1 (atom stride LBO = 128 B = one pixel row: the
// shifted view again) and B = dz1 rows 4t-1 .. 4t+3 (TMA box {32 channels, 32
// x, 5 rows}, MN-major SWIZZLE_64B) whose two 32-wide N atoms are the row taps
// a = 1, 0 (atom stride 2 KB = one dz1 row; N = 64 with no zero padding: the
// MMA time is proportional to N, measured 16 cycles per M128 N32 K16 step).  The accumulator
// [128 x 64] lives in TMEM for the CTA's whole share of images (split-K over
// the CTAs), is written once at the end and reduced deterministically.  Pixels
// outside the image (x = Wo, rows -1 and >= Ho) have dz1 = 0 from the TMA zero
// fill, so window rows past the image contribute nothing.  Operands are bf16 here (dz1 is bf16;
// u8 -> bf16 is exact), so the converters build exact bf16 values.
constexpr int W1_CONV_WARPS = 8;
constexpr int W1_THREADS = 32 * (3 + W1_CONV_WARPS);  // image TMA, MMA, dz1 TMA, converters
#ifndef W1_NSTG_DEF
#define W1_NSTG_DEF 3
#endif
#ifndef W1_NA_DEF
#define W1_NA_DEF 3
#endif
#ifndef W1_ND_DEF
#define W1_ND_DEF 6  // dz1 tiles in flight (3 -> 6: 44 -> 39 us, measured)
#endif
constexpr int W1_NSTG = W1_NSTG_DEF, W1_NA = W1_NA_DEF, W1_ND = W1_ND_DEF;
constexpr int W1_DROWS = 5;                           // dz1 rows per tile (4t-1 .. 4t+3)
constexpr int W1_DBYTES = 32 * 2 * 32 * W1_DROWS;     // dz1 tile {32 ch, 32 x, 5 rows} bf16, SW64

struct W1Params {
  int n_img, C, H, W, Ho, Wo, Hs, tiles, box_rows, stg_bytes, slack;
  const int32_t* slot_ids;
  int T, n_traj;
  float* partial;  // [gridDim.x][32][C*64] per-CTA partial sums
};

int w1_smem_bytes(int stg_bytes, int slack) {
  return 1024 + W1_NA * C1_WBYTES + W1_ND * W1_DBYTES + W1_NSTG * stg_bytes + slack + 256;
}

template <int C>
__global__ void __launch_bounds__(W1_THREADS, 1)
    conv1_s2d_wgrad_kernel(const __grid_constant__ CUtensorMap map_obs,
                           const __grid_constant__ CUtensorMap map_boot,
                           const __grid_constant__ CUtensorMap map_dz, const __grid_constant__ W1Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* awin = smem;                          // W1_NA s2d windows (SW128 rows)
  uint8_t* dtl = awin + W1_NA * C1_WBYTES;       // W1_ND dz1 tiles
  uint8_t* stg = dtl + W1_ND * W1_DBYTES;        // W1_NSTG staged images
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg + W1_NSTG * p.stg_bytes + p.slack);
  uint64_t* stg_full = bars;
  uint64_t* stg_empty = stg_full + W1_NSTG;
  uint64_t* a_full = stg_empty + W1_NSTG;
  uint64_t* a_empty = a_full + W1_NA;
  uint64_t* d_full = a_empty + W1_NA;
  uint64_t* d_empty = d_full + W1_ND;
  uint64_t* acc_done = d_empty + W1_ND;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    sm100::tma_prefetch(&map_obs);
    sm100::tma_prefetch(&map_dz);
    if (p.slot_ids) sm100::tma_prefetch(&map_boot);
    for (int s = 0; s < W1_NSTG; ++s) {
      sm100::mbar_init(&stg_full[s], 1);
      sm100::mbar_init(&stg_empty[s], W1_CONV_WARPS);
    }
    for (int s = 0; s < W1_NA; ++s) {
      sm100::mbar_init(&a_full[s], W1_CONV_WARPS);
      sm100::mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < W1_ND; ++s) {
      sm100::mbar_init(&d_full[s], 1);
      sm100::mbar_init(&d_empty[s], 1);
    }
    sm100::mbar_init(acc_done, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 1) {
    sm100::tmem_alloc(tmem_slot, 128);
    sm100::tmem_relinquish();
  }
  // windows fully zeroed once: rows the converters never write (the x-tap
  // overrun row, K padding) must hold finite values, they meet dz1 = 0
  for (int e = threadIdx.x; e < W1_NA * C1_WBYTES / 16; e += W1_THREADS)
    reinterpret_cast<uint4*>(awin)[e] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  APPO_PDL_ENTRY();  // dz1 comes from the previous kernel
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int B = p.n_traj * p.T;

  if (warp == 0) {
    // ---- image TMA: one box per image ----
    int j = 0;
    for (int img = blockIdx.x; img < p.n_img; img += gridDim.x, ++j) {
      const int s = j % W1_NSTG;
      sm100::mbar_wait(&stg_empty[s], ((j / W1_NSTG) & 1) ^ 1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      sm100::mbar_arrive_expect_tx_warp(&stg_full[s], (uint32_t)(C * p.box_rows * p.W));
      uint8_t* dst = stg + s * p.stg_bytes;
      if (!p.slot_ids) {
        sm100::tma_load_4d_warp(dst, &map_obs, &stg_full[s], 0, 0, 0, img);
      } else if (img < B) {
        sm100::tma_load_5d_warp(dst, &map_obs, &stg_full[s], 0, 0, 0, img % p.T,
                                __ldg(p.slot_ids + img / p.T));
      } else {
        sm100::tma_load_4d_warp(dst, &map_boot, &stg_full[s], 0, 0, 0, __ldg(p.slot_ids + img - B));
      }
    }
  } else if (warp == 2) {
    // ---- dz1 TMA: rows 4t-1 .. 4t+3 of the tile's image (outside the image -> 0) ----
    int d = 0;
    uint32_t dph = 0;
    for (int img = blockIdx.x; img < p.n_img; img += gridDim.x) {
      for (int t = 0; t < p.tiles; ++t) {
        sm100::mbar_wait(&d_empty[d], dph ^ 1);
        sm100::mbar_arrive_expect_tx_warp(&d_full[d], (uint32_t)W1_DBYTES);
        sm100::tma_load_4d_warp(dtl + d * W1_DBYTES, &map_dz, &d_full[d], 0, 0, 4 * t - 1, img);
        if (++d == W1_ND) { d = 0; dph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---- MMA: per tile, 8 K16 pixel steps; M = (b, feature), N = (a = 1, 0; channel) = 64 ----
    constexpr uint32_t idesc = sm100::make_idesc_bf16(128, 64, 1, 1);
    const uint32_t a0 = sm100::smem_u32(awin), d0 = sm100::smem_u32(dtl);
    int a = 0, d = 0;
    uint32_t aph = 0, dph = 0, acc = 0;
    for (int img = blockIdx.x; img < p.n_img; img += gridDim.x) {
      for (int t = 0; t < p.tiles; ++t) {
        sm100::mbar_wait(&a_full[a], aph);
        sm100::mbar_wait(&d_full[d], dph);
        sm100::tc_fence_after();
        const uint32_t wb = a0 + a * C1_WBYTES, db = d0 + d * W1_DBYTES;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          // A: pixels 16ks.. of the tile, M atoms b = 0, 1 one pixel row apart
          // (LBO = 128 B); B: dz1 of the same pixels one row up (a = 1, N atom 0)
          // and of the same row (a = 0, N atom 1, LBO = 2 KB)
          const uint64_t ad = sm100::make_sdesc(wb + 16 * ks * 128, 128, 1024);
          const uint64_t bd = sdesc_mn_sw64(db + 16 * ks * 64, 2048, 512);
          sm100::umma_f16_warp(tmem_base, ad, bd, idesc, (acc | ks) ? 1u : 0u);
        }
        acc = 1;
        sm100::umma_commit_warp(&a_empty[a]);
        sm100::umma_commit_warp(&d_empty[d]);
        if (++a == W1_NA) { a = 0; aph ^= 1; }
        if (++d == W1_ND) { d = 0; dph ^= 1; }
      }
    }
    sm100::umma_commit_warp(acc_done);
  } else {
    // ---- converters: staged u8 -> exact bf16 s2d windows (as conv1_s2d_kernel) ----
    // (4 s2d rows per window: the row taps are in B; window row 128 (read by
    // the b = 1 atom of the tile's last pixel, whose dz1 is 0) stays zero)
    const int cw = warp - 3;
    constexpr int kUnits = 4 * 2 * C;
    constexpr int kPerWarp = (kUnits + W1_CONV_WARPS - 1) / W1_CONV_WARPS;
    uint32_t soff[kPerWarp], doff[kPerWarp];
#pragma unroll
    for (int k = 0; k < kPerWarp; ++k) {
      const int u = min(cw + k * W1_CONV_WARPS, kUnits - 1);
      const int pyl = u / (2 * C), kc = u - pyl * 2 * C;
      soff[k] = (uint32_t)(((kc >> 1) * p.box_rows + 4 * pyl + 2 * (kc & 1)) * p.W + 4 * lane);
      doff[k] = (uint32_t)(lane * 128 + pyl * 4096 + ((kc ^ (lane & 7)) << 4));
    }
    const uint32_t tstep = 16u * p.W;
    const uint64_t big2 = f2pack(8388608.0f, 8388608.0f);
    // exact bf16 of 4 u8 values: 2^23 + v as float, minus 2^23, upper halves
    auto cvt4 = [&](uint32_t w, uint32_t& x0, uint32_t& x1) {
      const float2 v01 = f2unpack(fadd2(
          f2pack(__uint_as_float(__byte_perm(w, 0x4B000000u, 0x7650)),
                 __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7651))), big2 ^ 0x8000000080000000ull));
      const float2 v23 = f2unpack(fadd2(
          f2pack(__uint_as_float(__byte_perm(w, 0x4B000000u, 0x7652)),
                 __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7653))), big2 ^ 0x8000000080000000ull));
      x0 = __byte_perm(__float_as_uint(v01.x), __float_as_uint(v01.y), 0x7632);
      x1 = __byte_perm(__float_as_uint(v23.x), __float_as_uint(v23.y), 0x7632);
    };
    int j = 0, a = 0;
    uint32_t aph = 0;
    for (int img = blockIdx.x; img < p.n_img; img += gridDim.x, ++j) {
      const int s = j % W1_NSTG;
      sm100::mbar_wait(&stg_full[s], (j / W1_NSTG) & 1);
      const uint8_t* src0 = stg + s * p.stg_bytes;
      for (int t = 0; t < p.tiles; ++t, src0 += tstep) {
        sm100::mbar_wait(&a_empty[a], aph ^ 1);
        uint8_t* dst0 = awin + a * C1_WBYTES;
        uint32_t lo[kPerWarp], hi[kPerWarp];
#pragma unroll
        for (int k = 0; k < kPerWarp; ++k) {
          lo[k] = *reinterpret_cast<const uint32_t*>(src0 + soff[k]);
          hi[k] = *reinterpret_cast<const uint32_t*>(src0 + soff[k] + p.W);
        }
#pragma unroll
        for (int k = 0; k < kPerWarp; ++k) {
          uint4 v;
          cvt4(lo[k], v.x, v.y);
          cvt4(hi[k], v.z, v.w);
          *reinterpret_cast<uint4*>(dst0 + doff[k]) = v;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&a_full[a]);
        if (++a == W1_NA) { a = 0; aph ^= 1; }
      }
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&stg_empty[s]);
    }
    // ---- final epilogue (converter warps 0..3 = lane quarters 3, 0, 1, 2):
    //      TMEM row m = (b = m / 64, feature f = m % 64 = c*16 + i*4 + j) ----
    if (cw < 4) {
      sm100::mbar_wait(acc_done, 0);
      sm100::tc_fence_after();
      const int q = warp & 3, m = 32 * q + lane;
      const int b = m >> 6, f = m & 63;
      const int c = f >> 4, i = (f >> 2) & 3, jj = f & 3;
      float* out = p.partial + (size_t)blockIdx.x * 32 * (C * 64);
#pragma unroll
      for (int ta = 0; ta < 2; ++ta) {  // TMEM columns 32 * (1 - ta): row tap ta
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(32 * q) << 16) + (1 - ta) * 32, r);
        sm100::tmem_ld_wait();
        if (f < 16 * C) {
          const int k = c * 64 + (4 * ta + i) * 8 + 4 * b + jj;
#pragma unroll
          for (int co = 0; co < 32; ++co) out[co * (C * 64) + k] = __uint_as_float(r[co]);
        }
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem_base, 128);
  }
}

template <int C>
int w1_launch(Ctx* c, const CUtensorMap& mo, const CUtensorMap& mbt, const CUtensorMap& mdz,
              const W1Params& p, int grid) {
  auto kern = conv1_s2d_wgrad_kernel<C>;
  const int smem = w1_smem_bytes(p.stg_bytes, p.slack);
  static int attr_bytes[64] = {};
  const int dev = c->device & 63;
  if (attr_bytes[dev] < smem) {
    APPO_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_bytes[dev] = smem;
  }
  c->next_name = "conv1_s2d_wgrad_tcgen05";
  const double M = (double)p.n_img * p.Ho * p.Wo;
  c->next_flops = 2.0 * M * 32 * C * 64;
  c->next_bytes = (double)p.n_img * C * p.H * p.W + 2.0 * M * 32 + 4.0 * grid * 32 * C * 64;
  APPO_LAUNCH(c, kern, grid, W1_THREADS, smem, mo, mbt, mdz, p);
  return APPO_OK;
}

}  // namespace

const void* kanchor_conv1() { return reinterpret_cast<const void*>(&conv1_s2d_kernel<3>); }

// Host side: contract of the s2d path (else the caller keeps the engine path).
bool conv1_s2d_supported(const ConvIn& in, int N, const Epilogue& e) {
  if (!in.u8 || in.ksz != 8 || in.s != 4 || N != 32) return false;
  if (e.flags != (EPI_BIAS | EPI_ELU | EPI_BF16) || (e.ldo & 7) || !e.bias) return false;
  if ((reinterpret_cast<uintptr_t>(e.out) & 15)) return false;
  const int Hs = in.Ho + 1, Ws = in.Wo + 1;
  if (Ws > 32 || in.Wi % 16 || 4 * Hs > in.Hi || 4 * Hs > 256 || in.Cin < 1 || in.Cin > 4)
    return false;
  const int tiles = (in.Ho + 3) / 4;
  return c1_smem_bytes((in.Cin * 4 * Hs * in.Wi + 127) & ~127, c1_slack(tiles, 4 * Hs, in.Wi)) <=
         227 * 1024;
}

int conv1_s2d_forward(Ctx* c, const ConvIn& in, const uint16_t* w1h, const Epilogue& e) {
  if (in.n_img <= 0) return APPO_OK;
  APPO_REQUIRE(conv1_s2d_supported(in, 32, e), APPO_ERR_CONTRACT, "conv1_s2d: unsupported shape");
  C1Params p{};
  p.n_img = in.n_img;
  p.C = in.Cin;
  p.H = in.Hi;
  p.W = in.Wi;
  p.Ho = in.Ho;
  p.Wo = in.Wo;
  p.Hs = in.Ho + 1;
  p.tiles = (in.Ho + 3) / 4;
  p.box_rows = 4 * p.Hs;
  p.stg_bytes = (p.C * p.box_rows * p.W + 127) & ~127;
  p.slack = c1_slack(p.tiles, p.box_rows, p.W);
  p.slot_ids = in.slot_ids;
  p.T = in.T;
  p.n_traj = in.n_traj;
  p.w = w1h;
  p.bias = e.bias;
  p.scale = e.scale;
  p.out = reinterpret_cast<uint16_t*>(e.out);
  p.ldo = e.ldo;
  CUtensorMap mo, mbt;
  APPO_REQUIRE(make_u8_image_maps(&mo, &mbt, in, p.box_rows), APPO_ERR_CONTRACT,
               "conv1_s2d: images must be 16-byte aligned for TMA staging");
  switch (p.C) {
    case 1: return c1_launch<1>(c, mo, mbt, p);
    case 2: return c1_launch<2>(c, mo, mbt, p);
    case 3: return c1_launch<3>(c, mo, mbt, p);
    default: return c1_launch<4>(c, mo, mbt, p);
  }
}

int conv1_s2d_wgrad(Ctx* c, const ConvIn& in, const uint16_t* dz1, float* dw, float scale) {
  if (in.n_img <= 0) return APPO_OK;
  const int Hs = in.Ho + 1, Ws = in.Wo + 1;
  if (!in.u8 || in.ksz != 8 || in.s != 4 || Ws > 32 || in.Wi % 16 || 4 * Hs > in.Hi ||
      4 * Hs > 256 || in.Cin < 1 || in.Cin > 3 || (reinterpret_cast<uintptr_t>(dz1) & 15))
    return APPO_ERR_CONTRACT;
  W1Params p{};
  p.n_img = in.n_img;
  p.C = in.Cin;
  p.H = in.Hi;
  p.W = in.Wi;
  p.Ho = in.Ho;
  p.Wo = in.Wo;
  p.Hs = Hs;
  p.tiles = (in.Ho + 3) / 4;
  p.box_rows = 4 * Hs;
  p.stg_bytes = (p.C * p.box_rows * p.W + 127) & ~127;
  p.slack = c1_slack(p.tiles, p.box_rows, p.W);
  p.slot_ids = in.slot_ids;
  p.T = in.T;
  p.n_traj = in.n_traj;
  if (w1_smem_bytes(p.stg_bytes, p.slack) > 227 * 1024) return APPO_ERR_CONTRACT;
  CUtensorMap mo, mbt, mdz;
  if (!make_u8_image_maps(&mo, &mbt, in, p.box_rows)) return APPO_ERR_CONTRACT;
  // dz1 [img][Ho][Wo][32] bf16, box {64 (32 real), 32, 5, 1}: out-of-range -> 0
  const int st = make_tmap_bf16_4d(&mdz, dz1, 32, (uint64_t)in.Wo, (uint64_t)in.Ho,
                                   (uint64_t)in.n_img, 32, 32, W1_DROWS, 1, 64);
  if (st) return st;
  const int grid = c->num_sms < p.n_img ? c->num_sms : p.n_img;
  const int K1 = p.C * 64;
  float* part = nullptr;
  const int wst = gemm_workspace(c, (size_t)grid * 32 * K1 * sizeof(float), &part);
  if (wst) return wst;
  p.partial = part;
  int r;
  switch (p.C) {
    case 1: r = w1_launch<1>(c, mo, mbt, mdz, p, grid); break;
    case 2: r = w1_launch<2>(c, mo, mbt, mdz, p, grid); break;
    default: r = w1_launch<3>(c, mo, mbt, mdz, p, grid); break;
  }
  if (r) return r;
  Epilogue e;
  e.scale = scale;
  e.out = dw;
  e.ldo = K1;
  return splitk_reduce(c, 32, K1, grid, part, e);
}

}  // namespace appo_b200
