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
    conv2_s2d_kernel(const __grid_constant__ CUtensorMap map_a1, const __grid_constant__ C2Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stg = smem;                              // C2_NSTG x (even plane, odd plane)
  uint8_t* bsm = stg + C2_NSTG * C2_STAGE;          // resident weights
  uint64_t* bars = reinterpret_cast<uint64_t*>(bsm + C2_BBYTES);
  uint64_t* full = bars;
  uint64_t* empty = full + C2_NSTG;
  uint64_t* acc_full = empty + C2_NSTG;
  uint64_t* acc_empty = acc_full + C2_NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + C2_NACC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    sm100::tma_prefetch(&map_a1);
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
  // B block (a, e): row n = 2co + b holds W2[co][2a+e][2b .. 2b+1][0..31] (128 B)
  for (int i = threadIdx.x; i < 4 * 128 * 8; i += C2_THREADS) {
    const int blk = i >> 10, n = (i >> 3) & 127, c = i & 7;
    const int a = blk >> 1, e = blk & 1, co = n >> 1, b = n & 1;
    const uint4 v = reinterpret_cast<const uint4*>(
        p.w + ((size_t)(co * 4 + 2 * a + e) * 4 + 2 * b) * 32)[c];
    *reinterpret_cast<uint4*>(bsm + blk * 16384 + n * 128 + ((c ^ (n & 7)) << 4)) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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

}  // namespace

const void* kanchor_conv2() { return reinterpret_cast<const void*>(&conv2_s2d_kernel); }

int conv2_s2d_forward(Ctx* c, const uint16_t* a1, int n_img, int Hi, int Wi, int Ho, int Wo,
                      const uint16_t* w2, const Epilogue& e) {
  if (n_img <= 0) return APPO_OK;
  // k4 s2 geometry, one 128-row tile per image, 16-byte aligned rows for TMA
  if (Ho != (Hi - 4) / 2 + 1 || Wo != (Wi - 4) / 2 + 1 || Ho * 16 > 128 || Wo + 1 > 16 ||
      e.flags != (EPI_BIAS | EPI_ELU | EPI_BF16) || e.ldo != 64 || !e.bias ||
      (reinterpret_cast<uintptr_t>(a1) & 15) || (reinterpret_cast<uintptr_t>(e.out) & 15) ||
      (Wi * 64) % 16)
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
  APPO_LAUNCH(c, conv2_s2d_kernel, grid, C2_THREADS, C2_SMEM, map, p);
  return APPO_OK;
}

}  // namespace appo_b200
