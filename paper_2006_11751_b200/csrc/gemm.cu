// tcgen05 GEMM engine for sm_100a: D = A . B^T, bf16 operands, fp32 accumulate
// in TMEM, fused epilogue.  Every dense contraction of the model (conv layers
// as im2col GEMMs, FC, GRU projections, and all their backward dgrad / wgrad
// products) runs through this kernel.
//
// Design (one CTA per SM or two, persistent over output tiles):
//   warp 0  : TMA producer -- 128B-swizzled boxes of A and B into a 4-stage
//             shared-memory ring guarded by full/empty mbarriers
//   warp 1  : MMA issuer   -- one elected thread issues tcgen05.mma (M=128,
//             N=BN, K=16) into a double-buffered TMEM accumulator and commits
//             to the stage's empty barrier / the accumulator's full barrier
//   warps 2-9: epilogue    -- two warps per TMEM lane quarter (column halves);
//             tcgen05.ld 32 lanes x 16 columns, compile-time scale / bias /
//             ELU / ELU' / bf16 pack, global store; releases the accumulator
// Operands may be K-major or MN-major (UMMA descriptor major bits), so weight
// gradients (reduction over the batch) read activations and output grads in
// the layout the forward / backward produced them -- no transposes.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <string>

#include "gemm.cuh"
#include "sm100.cuh"

namespace appo_b200 {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one swizzle row
constexpr int THREADS = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue
constexpr int A_TILE_BYTES = BM * BK * 2;  // 16 KB

// Implicit-GEMM A operand (convolution forward): row m = output position
// (image r = m / P, p = m % P, y = p / Wo, x = p % Wo), K = receptive field.
struct GatherP {
  const uint8_t* src;  // AG_NHWC: bf16 NHWC activations; AG_U8: first u8 CHW image / slot region
  int64_t img_stride;  // AG_U8: bytes between images (contiguous batches)
  int P, Wo;           // output positions per image, output width
  int Hi, Wi, Cin;     // input geometry (AG_U8: channels C, H, W)
  int ksz, s;          // kernel size, stride
  // AG_U8 images in trajectory slots (layout v2): image r < n_traj*T is step
  // r % T of slot slot_ids[r / T]; later images are the bootstrap observations
  const int32_t* slot_ids;
  uint64_t slot_bytes, obs_off, boot_off;
  int T, n_traj;
  int nq;    // AG_U8: output rows (images x Ho); AG_TAPS: images per M tile
  int tma;   // AG_U8 staging: 1 = tensor-map boxes (mapA / map2), 0 = bulk copies
};
enum AGather : int {
  AG_NONE = 0, AG_NHWC = 1, AG_U8 = 2, AG_DGRAD = 3, AG_U8W = 4, AG_TAPS = 5, AG_TAPSW = 6
};
constexpr int GATHER_THREADS = 128;  // NHWC gather warps (after the epilogue warps)
constexpr int U8_GATHER_THREADS = 256;  // conv1 staging/convert warps: two per tile row
#ifndef APPO_U8_CONV_THREADS
#define APPO_U8_CONV_THREADS 256
#endif
constexpr int U8_CONV_THREADS = APPO_U8_CONV_THREADS;  // conv1 forward converters (128 x 2^k)

// Input gradient of a stride-2 convolution (kernel k <= 4, no padding) by
// sub-pixel decomposition.  Input position (2yy+py, 2xx+px) only receives
// taps kh = py + 2a, kw = px + 2b (a, b in {0, 1}) from dz_next[yy-a][xx-b],
// so for a COARSE position (yy, xx) all four parity classes read the same
// 2x2 neighbourhood: one GEMM with rows = coarse positions, K = (a, b, co)
// and N = (class, ci) computes the four output pixels of the 2x2 block:
//   D[(r,yy,xx)][(cls,ci)] = sum_{a,b,co} dz_next[r][yy-a][xx-b][co] Wt[(cls,ci)][(a,b,co)]
// The A tile is one 4-D TMA box {64 ch, Wb x, Hb y, Ib images} of dz_next at
// (x, y) offset (-b, -a): out-of-range taps are zero-filled by the TMA unit.
struct DgradP {
  int Hcc, Wcc;      // coarse grid (ceil(Hi/2), ceil(Wi/2)); boxes cover its live part
  int Hb, Wb, Ib;    // TMA box (Hb * Wb * Ib == 128 rows)
  int Hi, Wi, Ci;    // produced dz [img][Hi][Wi][Ci]
  int n_img, apt;    // images; 64-channel atoms per tap (Co / 64)
  unsigned long long* bacc;  // fused bias gradient: fixed-point accumulators [16][Ci]
  unsigned* bcnt;            // CTA completion counter
  float* bout;               // bias gradient [Ci]
};

struct KParams {
  CUtensorMap map2;  // AG_U8 / AG_U8W image staging: observation map (4-D contiguous / 5-D slots)
  CUtensorMap map3;  // ... and the bootstrap-observation map (slots)
  int M, N, K;
  int tiles_m, tiles_n, splits, kb_per_split, nkb;
  Epilogue epi;
  float* partial;  // split-K workspace [splits][M][N]
  GatherP g;
  DgradP dg;
  long long* prof;  // optional per-role timestamps of CTA 0 (APPO_GEMM_PROF), [16 units][8]
};
#define GEMM_PROF(slot)                                                      \
  do {                                                                       \
    if (p.prof && blockIdx.x == 0 && (u - (int)blockIdx.x) / (int)gridDim.x < 16) \
      p.prof[((u - blockIdx.x) / gridDim.x) * 16 + (slot)] = clock64();      \
  } while (0)

// Work unit u of the persistent schedule: output tile + K-block range.
struct Unit {
  int tm, tn, z, kb0, kb1;
};
__device__ __forceinline__ Unit decode_unit(const KParams& p, int u) {
  Unit r;
  if (p.tiles_n == 1 && p.splits == 1) {  // (conv / dgrad shapes) no integer divisions
    r.tm = u;
    r.tn = 0;
    r.z = 0;
    r.kb0 = 0;
    r.kb1 = p.nkb;
    return r;
  }
  r.tm = u % p.tiles_m;
  r.tn = (u / p.tiles_m) % p.tiles_n;
  r.z = u / (p.tiles_m * p.tiles_n);
  r.kb0 = r.z * p.kb_per_split;
  r.kb1 = min(r.kb0 + p.kb_per_split, p.nkb);
  return r;
}

// barrier area after the stage ring / resident operands: full[<=8] empty[<=8]
// acc_full[<=8] acc_empty[<=8] tmem slot, then (conv1 staging / resident-B)
// barriers at +BAR_AUX, conv1 staging data at +BAR_BYTES
constexpr int BAR_AUX = 320;
constexpr int BAR_BYTES = 512;

template <int BN>
struct Cfg {
  static constexpr int B_TILE_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_TILE_BYTES + B_TILE_BYTES;
  // TMEM accumulator ring: small tiles keep more tiles in flight (the
  // full -> MMA -> epilogue chain per tile is latency-bound, not MMA-bound)
  static constexpr int NACC = BN <= 32 ? 8 : BN <= 64 ? 4 : 2;
  static constexpr int TMEM_COLS = (NACC * BN <= 32)    ? 32
                                   : (NACC * BN <= 64)  ? 64
                                   : (NACC * BN <= 128) ? 128
                                   : (NACC * BN <= 256) ? 256
                                                        : 512;
  // as many stages as fit in ~192 KB (4..8): the gathered / HBM-streamed
  // operands are latency-bound, bytes in flight per SM set the rate
  static constexpr int STAGES = (196608 / STAGE_BYTES) > 8   ? 8
                                : (196608 / STAGE_BYTES) < 4 ? 4
                                                             : (196608 / STAGE_BYTES);
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + BAR_BYTES;
};

// ELU with the MUFU exponential: |error| <= ~1e-7 absolute, far below the
// bf16 rounding of the stored activation (accurate expm1f costs ~25 instructions
// per element, which made the small-N conv epilogues instruction-bound).
__device__ __forceinline__ float elu_fast(float x) { return x > 0.0f ? x : __expf(x) - 1.0f; }

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float bf16_bits_to_float(uint16_t b) {
  return __uint_as_float(((uint32_t)b) << 16);
}

template <int BN>
__device__ __forceinline__ void epilogue_chunk(const KParams& p, int m, int n0, int z,
                                               const uint32_t (&r)[16]) {
  const Epilogue& e = p.epi;
  if (m >= p.M) return;
  float v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
  if (p.splits > 1) {  // raw partial; the reduce kernel applies the epilogue
    float* dst = p.partial + ((size_t)z * p.M + m) * p.N + n0;
    if (n0 + 16 <= p.N && (p.N & 3) == 0) {
#pragma unroll
      for (int j = 0; j < 16; j += 4)
        *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
      for (int j = 0; j < 16 && n0 + j < p.N; ++j) dst[j] = v[j];
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int n = n0 + j;
    float x = v[j] * e.scale;
    if ((e.flags & EPI_BIAS) && n < p.N) x += e.bias[n];
    if (e.flags & EPI_ELU) x = elu_fast(x);
    if ((e.flags & EPI_DELU) && n < p.N) {
      const float a = bf16_bits_to_float(e.aux[(size_t)m * e.ld_aux + n]);
      x *= (a > 0.0f ? 1.0f : a + 1.0f);
    }
    v[j] = x;
  }
  if (e.flags & EPI_TRANS) {
    for (int j = 0; j < 16 && n0 + j < p.N; ++j) {
      const size_t o = (size_t)(n0 + j) * e.ldo + m;
      if (e.flags & EPI_BF16) {
        reinterpret_cast<__nv_bfloat16*>(e.out)[o] = __float2bfloat16_rn(v[j]);
      } else {
        float* dst = reinterpret_cast<float*>(e.out) + o;
        *dst = (e.flags & EPI_ACCUM) ? *dst + v[j] : v[j];
      }
    }
    return;
  }
  const bool full = (n0 + 16 <= p.N);
  if (e.flags & EPI_BF16) {
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(e.out) + (size_t)m * e.ldo + n0;
    if (full && ((e.ldo & 7) == 0) && ((reinterpret_cast<uintptr_t>(e.out) & 15) == 0)) {
      uint32_t w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
        w[j] = *reinterpret_cast<uint32_t*>(&h);
      }
      reinterpret_cast<uint4*>(dst)[0] = make_uint4(w[0], w[1], w[2], w[3]);
      reinterpret_cast<uint4*>(dst)[1] = make_uint4(w[4], w[5], w[6], w[7]);
    } else {
      for (int j = 0; j < 16 && n0 + j < p.N; ++j) dst[j] = __float2bfloat16_rn(v[j]);
    }
  } else {
    float* dst = reinterpret_cast<float*>(e.out) + (size_t)m * e.ldo + n0;
    if (full && ((e.ldo & 3) == 0) && ((reinterpret_cast<uintptr_t>(e.out) & 15) == 0)) {
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        float4 x = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        if (e.flags & EPI_ACCUM) {
          const float4 o = *reinterpret_cast<float4*>(dst + j);
          x.x += o.x; x.y += o.y; x.z += o.z; x.w += o.w;
        }
        *reinterpret_cast<float4*>(dst + j) = x;
      }
    } else {
      for (int j = 0; j < 16 && n0 + j < p.N; ++j)
        dst[j] = (e.flags & EPI_ACCUM) ? dst[j] + v[j] : v[j];
    }
  }
}

// Compile-time epilogue variants: straight-line code for the fused epilogues
// the model uses; anything else (tails, unaligned, rare flag mixes) takes the
// generic runtime-flag path above.
enum EpiVariant : int {
  EV_GENERIC = 0,
  EV_SPLIT = 1,     // raw fp32 partial (split-K)
  EV_F32 = 2,       // fp32: x*scale (+bias)
  EV_ELU_BF16 = 3,  // bf16: ELU(x*scale + bias)
  EV_DELU_BF16 = 4, // bf16: x * ELU'(aux)
  EV_BF16 = 5,      // bf16: x*scale
  EV_DGRAD = 6,     // bf16: x * ELU'(aux) at the sub-pixel position + bias sums
  EV_DELU_BSUM = 7, // EV_DELU_BF16 + fused bias gradient (Epilogue::bsum_*)
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int EV>
__device__ __forceinline__ void epilogue_dispatch(const KParams& p, int m, int n0, int z,
                                                  const uint32_t (&r)[16],
                                                  float* sv = nullptr) {
  if constexpr (EV == EV_GENERIC) {
    epilogue_chunk<0>(p, m, n0, z, r);
  } else {
    if (m >= p.M) return;
    const Epilogue& e = p.epi;
    if (n0 + 16 > p.N) {  // ragged N tail: generic path
      epilogue_chunk<0>(p, m, n0, z, r);
      return;
    }
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
    if constexpr (EV == EV_SPLIT) {
      float4* dst = reinterpret_cast<float4*>(p.partial + ((size_t)z * p.M + m) * p.N + n0);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      return;
    }
    if constexpr (EV == EV_F32 || EV == EV_ELU_BF16 || EV == EV_BF16) {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] *= e.scale;
    }
    if constexpr (EV == EV_F32 || EV == EV_ELU_BF16) {
      if (e.flags & EPI_BIAS) {
        const float4* b4 = reinterpret_cast<const float4*>(e.bias + n0);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 b = __ldg(b4 + j);
          v[4 * j] += b.x;
          v[4 * j + 1] += b.y;
          v[4 * j + 2] += b.z;
          v[4 * j + 3] += b.w;
        }
      }
    }
    if constexpr (EV == EV_ELU_BF16) {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = elu_fast(v[j]);
    }
    if constexpr (EV == EV_DELU_BF16 || EV == EV_DELU_BSUM) {
      const uint4* a4 = reinterpret_cast<const uint4*>(e.aux + (size_t)m * e.ld_aux + n0);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint4 w = a4[h];
        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float a0 = bf16_bits_to_float((uint16_t)(ww[q] & 0xFFFF));
          const float a1 = bf16_bits_to_float((uint16_t)(ww[q] >> 16));
          v[8 * h + 2 * q] *= (a0 > 0.0f ? 1.0f : a0 + 1.0f);
          v[8 * h + 2 * q + 1] *= (a1 > 0.0f ? 1.0f : a1 + 1.0f);
        }
      }
    }
    if constexpr (EV == EV_F32) {
      float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(e.out) +
                                              (size_t)m * e.ldo + n0);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    } else {
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(e.out) +
                                            (size_t)m * e.ldo + n0);
      uint32_t w[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) w[q] = pack_bf16(v[2 * q], v[2 * q + 1]);
      dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
      dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
      if constexpr (EV == EV_DELU_BSUM) {  // stored (rounded) values feed the bias gradient
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          sv[2 * q] = bf16_bits_to_float((uint16_t)(w[q] & 0xFFFF));
          sv[2 * q + 1] = bf16_bits_to_float((uint16_t)(w[q] >> 16));
        }
      }
    }
  }
}

// A-tile gatherers (warps 10..13, one output row per thread, all 8 chunks of
// the 64-wide K block): NHWC bf16 rows via cp.async straight into the SW128
// layout (completion tracked by the stage's full mbarrier), or u8 pixels
// loaded, converted to bf16 (exact integers; 1/255 folded into the epilogue)
// and stored to shared memory.
// Window origin of output row m (image r, position y, x): computed once per
// tile, the per-chunk offsets come from a per-CTA table (NHWC) or are affine
// in (channel, kh) (u8).
template <int AG>
__device__ __forceinline__ const uint8_t* gather_row_origin(const KParams& p, int m, bool& valid) {
  const GatherP& g = p.g;
  valid = m < p.M;
  const int mm = valid ? m : 0;
  const int r = mm / g.P, pp = mm % g.P;
  const int y = pp / g.Wo, x = pp % g.Wo;
  if constexpr (AG == AG_NHWC)
    return g.src + 2 * ((((int64_t)r * g.Hi + y * g.s) * g.Wi + x * g.s) * g.Cin);
  else
    return g.src + (int64_t)r * g.img_stride + (int64_t)(y * g.s) * g.Wi + x * g.s;
}

template <int AG>
__device__ __forceinline__ void gather_stage(const KParams& p, uint8_t* sA, uint64_t* full,
                                             const uint8_t* origin, bool valid, int kb, int gt,
                                             const int* off_tab) {
  const GatherP& g = p.g;
  if constexpr (AG == AG_NHWC) {
    // two threads per tile row: chunks 4*(gt >> 7) .. +3 of row gt & 127
    const int row = gt & 127, c0 = (gt >> 7) * 4;
    const uint32_t row_base = sm100::smem_u32(sA) + row * 128;
#pragma unroll
    for (int c = c0; c < c0 + 4; ++c) {
      const uint8_t* src = origin + off_tab[kb * 8 + c];
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                       row_base + ((c ^ (row & 7)) << 4)),
                   "l"(src), "r"(valid ? 16 : 0)
                   : "memory");
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                     sm100::smem_u32(full))
                 : "memory");
  } else {
    const uint32_t row_base = sm100::smem_u32(sA) + gt * 128;
    const uint8_t* img = origin + (int64_t)kb * g.Hi * g.Wi;  // channel kb
    uint32_t lo[8], hi[8];
#pragma unroll
    for (int kh = 0; kh < 8; ++kh) {
      const uint8_t* s = img + (int64_t)kh * g.Wi;
      lo[kh] = valid ? __ldg(reinterpret_cast<const uint32_t*>(s)) : 0u;
      hi[kh] = valid ? __ldg(reinterpret_cast<const uint32_t*>(s + 4)) : 0u;
    }
#pragma unroll
    for (int kh = 0; kh < 8; ++kh) {
      // u8 -> exact bf16 without I2F: PRMT places byte k into the float bits of
      // 2^23 + v, one FADD removes 2^23 (exact), and since v has <= 8
      // significant bits the upper 16 bits of the float ARE its bf16 encoding.
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t word = q < 2 ? lo[kh] : hi[kh];
        const int k0 = (q & 1) * 2;
        const float f0 = __uint_as_float(__byte_perm(word, 0x4B000000u, 0x7650 + k0)) - 8388608.0f;
        const float f1 =
            __uint_as_float(__byte_perm(word, 0x4B000000u, 0x7650 + k0 + 1)) - 8388608.0f;
        w[q] = __byte_perm(__float_as_uint(f0), __float_as_uint(f1), 0x7632);
      }
      asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(
                       row_base + ((kh ^ (gt & 7)) << 4)),
                   "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                   : "memory");
    }
    sm100::mbar_arrive(full);
  }
}

// ---- conv1 (u8, k8 s4) implicit GEMM with smem-staged input ------------------
// Tile = 4 consecutive output rows q (q = image * Ho + y) x 32 columns (the
// last one padding for Wo = 31): tile row m = 32 * (q - 4 * tile) + x.  The
// gather warps cp.async the 8 input rows of every (output row, channel) into
// a double-buffered staging area (12 KB, the next tile's while this one is
// converted), then build each channel's [128 rows x 64 (kh, kw)] A block from
// shared memory (u8 -> exact bf16; 1/255 folded into the epilogue scale).
constexpr int U8_ROWS = 4;  // output rows per tile (x 32 columns = BM)
constexpr int U8_NSTG = 4;  // staging ring depth (tiles in flight per CTA)

__device__ __forceinline__ const uint8_t* u8_image(const GatherP& g, int img) {
  if (!g.slot_ids) return g.src + (int64_t)img * g.img_stride;
  const int B = g.n_traj * g.T;
  if (img < B)
    return g.src + (uint64_t)g.slot_ids[img / g.T] * g.slot_bytes + g.obs_off +
           (uint64_t)(img % g.T) * ((uint64_t)g.Hi * g.Wi * g.Cin);
  return g.src + (uint64_t)g.slot_ids[img - B] * g.slot_bytes + g.boot_off;
}

// Staging slot layout: block (output row k, channel c) of U8_BLK bytes holds
// the 8 input rows (8*W contiguous bytes in global memory), copied from the
// 16-byte aligned address at or below them; delta[k] (0 or 8, per image) is
// where they start inside the block.
constexpr int U8_BLK = 8 * 128 + 16;
constexpr int U8_SID_CACHE = 256;  // slot ids cached in shared memory by the staging warp
constexpr int U8_BOX_ROWS = 4 * (U8_ROWS - 1) + 8;  // input rows of U8_ROWS output rows
__host__ __device__ constexpr int u8_stage_bytes(int C) {
  // max of the bulk layout and the two-run tensor-box layout (+16 B overread slack)
  // (rounded to 128 B: tensor-TMA destinations must be 128-byte aligned)
  return ((U8_ROWS * U8_BLK > 2 * U8_BOX_ROWS * 128 ? U8_ROWS * U8_BLK : 2 * U8_BOX_ROWS * 128) * C +
          16 + 127) & ~127;
}

// One staging box (rows row0.. of every channel of image img) from the
// observation maps: contiguous batch (4-D) or trajectory slots (5-D steps /
// 4-D bootstrap observations), slot ids from the shared-memory cache.
__device__ __forceinline__ void u8_box_load(const KParams& p, void* dst, uint64_t* bar, int img,
                                            int row0, const int* sids) {
  const GatherP& g = p.g;
  if (!g.slot_ids) {
    sm100::tma_load_4d_warp(dst, &p.map2, bar, 0, row0, 0, img);
  } else {
    const int B = g.n_traj * g.T;
    const int si = img < B ? img / g.T : img - B;
    const int sid = si < U8_SID_CACHE ? sids[si] : g.slot_ids[si];
    if (img < B)
      sm100::tma_load_5d_warp(dst, &p.map2, bar, 0, row0, 0, img % g.T, sid);
    else
      sm100::tma_load_4d_warp(dst, &p.map3, bar, 0, row0, 0, sid);
  }
}

// conv1 weight gradient staging: K block kb = output rows (2*(kb % KPI),
// +1) of image kb / KPI -> one box {W, 12 rows, C}.
constexpr int U8W_ROWS = 2;                          // output rows per K block (x 32 = 64 pixels)
constexpr int U8W_BOX_ROWS = 4 * (U8W_ROWS - 1) + 8;  // 12 input rows
__device__ __forceinline__ void u8w_stage(const KParams& p, int kb, uint8_t* buf, uint64_t* bar,
                                          const int* sids) {
  const GatherP& g = p.g;
  const int Ho = g.P / g.Wo;
  const int kpi = (Ho + U8W_ROWS - 1) / U8W_ROWS;
  const int img = kb / kpi, y0 = (kb - img * kpi) * U8W_ROWS;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of buf
  sm100::mbar_arrive_expect_tx_warp(bar, g.Cin * U8W_BOX_ROWS * g.Wi);
  u8_box_load(p, buf, bar, img, 4 * y0, sids);
}

// conv1 weight gradient B block (MN-major SW128, one 64-wide atom per channel):
// K row = pixel (ky, x) of the K block, N = (c, kh, kw); exact bf16 of u8.
// Thread gt < 64*C: row gt & 63, channel gt >> 6.
__device__ __forceinline__ void u8w_convert(const GatherP& g, const uint8_t* buf, uint8_t* sB,
                                            int gt) {
  const int row = gt & 63, c = gt >> 6;
  if (c >= g.Cin) return;
  const int ky = row >> 5, x = row & 31;
  const uint32_t src = sm100::smem_u32(buf) + (c * U8W_BOX_ROWS + 4 * ky) * g.Wi + 4 * x;
  const uint32_t row_base = sm100::smem_u32(sB) + c * 8192 + row * 128;
#pragma unroll
  for (int kh = 0; kh < 8; ++kh) {
    uint32_t lo, hi;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(lo) : "r"(src + kh * g.Wi));
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(hi) : "r"(src + kh * g.Wi + 4));
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // exact u8 -> bf16 (2^23 + v trick, see u8_convert history)
      const uint32_t word = q < 2 ? lo : hi;
      const int k0 = (q & 1) * 2;
      const float f0 = __uint_as_float(__byte_perm(word, 0x4B000000u, 0x7650 + k0)) - 8388608.0f;
      const float f1 = __uint_as_float(__byte_perm(word, 0x4B000000u, 0x7650 + k0 + 1)) - 8388608.0f;
      w[q] = __byte_perm(__float_as_uint(f0), __float_as_uint(f1), 0x7632);
    }
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(row_base + ((kh ^ (row & 7)) << 4)),
                 "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                 : "memory");
  }
}

// Tensor-map staging (one TMA box {W, 20 rows, C} per run of consecutive
// output rows of the same image: at most two per tile).  meta[k] = byte
// offset of output row k's first input row (channel 0) in the slot; channel
// planes are U8_BOX_ROWS * W apart.
__device__ __forceinline__ void u8_stage_tma(const KParams& p, int tile,
                                             uint8_t* buf, int* meta, uint64_t* bar, int lane,
                                             const int* sids, long long* pf = nullptr) {
  const GatherP& g = p.g;
  const int Ho = g.P / g.Wo;
  const int q0 = tile * U8_ROWS;
  const int nrow = min(U8_ROWS, g.nq - q0);
  const int img0 = q0 / Ho, y0 = q0 - img0 * Ho;
  const int n0 = min(nrow, Ho - y0);  // rows of the first image
  const int box = g.Cin * U8_BOX_ROWS * g.Wi;
  if (pf && lane == 0) pf[8] = clock64();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < U8_ROWS; ++k)
      meta[k] = k < n0 ? 4 * k * g.Wi : box + 4 * (k - n0) * g.Wi;
  __syncwarp();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of buf
  if (pf && lane == 0) pf[9] = clock64();
  sm100::mbar_arrive_expect_tx_warp(bar, (n0 < nrow ? 2 : 1) * box);
  if (pf && lane == 0) pf[10] = clock64();
  for (int r = 0; r < (n0 < nrow ? 2 : 1); ++r) {
    const int img = r ? img0 + 1 : img0, y = r ? 0 : y0;
    uint8_t* dst = buf + r * box;
    u8_box_load(p, dst, bar, img, 4 * y, sids);
  }
}

// Producer side (whole warp; one elected lane issues): bulk copies of tile
// `tile`'s input rows into a staging slot, completion on its mbarrier.  Image
// addresses are computed for all rows first (independent slot-id loads in
// flight together), the per-row alignment deltas are stored afterwards.
__device__ __forceinline__ void u8_stage_bulk(const GatherP& g, int tile, uint8_t* buf,
                                              int* delta, uint64_t* bar, int lane) {
  const int Ho = g.P / g.Wo;
  const uint32_t bytes = 8u * g.Wi;
  const uint8_t* r0[U8_ROWS];
#pragma unroll
  for (int k = 0; k < U8_ROWS; ++k) {
    const int q = min(tile * U8_ROWS + k, g.nq - 1);  // clamp: padding rows are not copied
    const int img = q / Ho, y = q - img * Ho;
    r0[k] = u8_image(g, img) + (int64_t)(y * 4) * g.Wi;
  }
  uint32_t total = 0;
  int d[U8_ROWS];
  uint32_t cbytes[U8_ROWS];
#pragma unroll
  for (int k = 0; k < U8_ROWS; ++k) {
    const bool ok = tile * U8_ROWS + k < g.nq;
    d[k] = (int)(reinterpret_cast<uintptr_t>(r0[k]) & 15);
    cbytes[k] = ok ? (bytes + d[k] + 15) & ~15u : 0u;
    total += g.Cin * cbytes[k];
  }
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < U8_ROWS; ++k) delta[k] = k * g.Cin * U8_BLK + d[k];  // meta: block + delta
  __syncwarp();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of buf
  sm100::mbar_arrive_expect_tx_warp(bar, total);
#pragma unroll
  for (int k = 0; k < U8_ROWS; ++k) {
    if (!cbytes[k]) continue;
    for (int c = 0; c < g.Cin; ++c)
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n\t}" ::"r"(
              sm100::smem_u32(buf + (k * g.Cin + c) * U8_BLK)),
          "l"(r0[k] - d[k] + (int64_t)c * g.Hi * g.Wi), "r"(cbytes[k]), "r"(sm100::smem_u32(bar))
          : "memory");
  }
}

// Build half a row of channel c's A block from the staged bytes (SW128
// K-major): thread gt handles tile row gt & 127, kernel rows kh = 4*(gt>>7)..+3.
// Values are written as fp16 (1024 + v): one PRMT per pair, exact for v in
// 0..255 (fp16 has unit spacing on [1024, 2048)); the constant 1024 * sum(W)
// is removed through the epilogue bias (k_conv1_half_weights).
// Thread gt's source address (channel 0) in a staged tile: slot base + the row's
// meta offset (read through a shared-space load) + its kernel rows and column.
__device__ __forceinline__ uint32_t u8_src0(const GatherP& g, const uint8_t* buf, const int* meta,
                                            int gt) {
  constexpr int KHT = 8 / (U8_CONV_THREADS / 128);
  const int row = gt & 127, kh0 = (gt >> 7) * KHT;
  int mk;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(mk) : "r"(sm100::smem_u32(meta + (row >> 5))));
  return sm100::smem_u32(buf) + mk + kh0 * g.Wi + 4 * (row & 31);
}

__device__ __forceinline__ void u8_convert(const GatherP& g, uint32_t src0, int plane,
                                           uint8_t* sA, int c, int gt) {
  constexpr int KHT = 8 / (U8_CONV_THREADS / 128);  // kernel rows per thread
  const int row = gt & 127, kh0 = (gt >> 7) * KHT;
  const uint32_t src = src0 + c * plane;
  const uint32_t row_base = sm100::smem_u32(sA) + row * 128;
#pragma unroll
  for (int j = 0; j < KHT; ++j) {
    uint32_t lo, hi;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(lo) : "r"(src + j * g.Wi));
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(hi) : "r"(src + j * g.Wi + 4));
    const uint32_t w0 = __byte_perm(lo, 0x64646464u, 0x4140);
    const uint32_t w1 = __byte_perm(lo, 0x64646464u, 0x4342);
    const uint32_t w2 = __byte_perm(hi, 0x64646464u, 0x4140);
    const uint32_t w3 = __byte_perm(hi, 0x64646464u, 0x4342);
    const int kh = kh0 + j;
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(row_base + ((kh ^ (row & 7)) << 4)),
                 "r"(w0), "r"(w1), "r"(w2), "r"(w3)
                 : "memory");
  }
}

// Output row of tile row m (conv1 epilogue), -1 for padding.
__device__ __forceinline__ int u8_out_row(const GatherP& g, int m) {
  const int q = m >> 5, x = m & 31;
  return (q < g.nq && x < g.Wo) ? q * g.Wo + x : -1;
}

// Sub-pixel dgrad epilogue for 16 columns (class cls, channels ci0..ci0+15)
// of coarse row m: output offset of dz at (2yy+py, 2xx+px), or -1 when the
// position is outside the image / the row is padding.
template <int CI>
__device__ __forceinline__ int64_t dgrad_offset(const KParams& p, int m, int col) {
  const DgradP& g = p.dg;
  const int per = g.Hb * g.Wb;
  const int img = m / per, rem = m % per;  // tile rows: (image, y, x) of the TMA box
  const int yy = rem / g.Wb, xx = rem % g.Wb;
  const int cls = col / CI, ci0 = col % CI;
  const int yi = 2 * yy + (cls >> 1), xi = 2 * xx + (cls & 1);
  if (img >= g.n_img || yy >= g.Hcc || xx >= g.Wcc || yi >= g.Hi || xi >= g.Wi) return -1;
  return (((int64_t)img * g.Hi + yi) * g.Wi + xi) * CI + ci0;
}
// x * ELU'(a_prev) -> bf16 store; bias sums of the stored values.
__device__ __forceinline__ void dgrad_finish(const KParams& p, int64_t off,
                                             const uint32_t (&r)[16], const uint4 (&a)[2],
                                             float (&sv)[16]) {
  uint32_t o[8];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t ww[4] = {a[h].x, a[h].y, a[h].z, a[h].w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float a0 = bf16_bits_to_float((uint16_t)(ww[q] & 0xFFFF));
      const float a1 = bf16_bits_to_float((uint16_t)(ww[q] >> 16));
      const float v0 = __uint_as_float(r[8 * h + 2 * q]) * (a0 > 0.0f ? 1.0f : a0 + 1.0f);
      const float v1 = __uint_as_float(r[8 * h + 2 * q + 1]) * (a1 > 0.0f ? 1.0f : a1 + 1.0f);
      o[4 * h + q] = pack_bf16(v0, v1);
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {  // the stored (rounded) values feed the bias gradient
    sv[2 * j] = bf16_bits_to_float((uint16_t)(o[j] & 0xFFFF));
    sv[2 * j + 1] = bf16_bits_to_float((uint16_t)(o[j] >> 16));
  }
  uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.epi.out) + off);
  dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
  dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
}

// AG_TAPS ring depth: A-only stages of 16 KB next to the resident weights
// (as many bytes in flight as fit: the strided boxes are latency-bound)
constexpr int taps_stages(int bn) { return bn <= 64 ? 8 : 4; }

template <int AG>
constexpr bool has_gather() {
  return AG == AG_NHWC || AG == AG_U8 || AG == AG_U8W;
}
// Epilogue warps: 8 (two per TMEM lane quarter); 16 for the sub-pixel dgrad,
// whose epilogue gathers its ELU' operand from HBM and needs more loads in flight.
template <int EV>
constexpr int epi_warps() {
  return EV == EV_DGRAD ? 16 : 8;
}
template <int AG>
constexpr int gather_threads() {
  return AG == AG_U8 ? U8_CONV_THREADS : has_gather<AG>() ? U8_GATHER_THREADS : 0;
}
template <int EV, int AG>
constexpr int kernel_threads() {
  // conv1 adds U8_NSTG staging warps after the gatherers (input rows -> smem ring)
  return 64 + 32 * epi_warps<EV>() + gather_threads<AG>() +
         ((AG == AG_U8 || AG == AG_U8W) ? 32 * U8_NSTG : 0);
}

// Lane l ends with the sum over all 32 lanes of v[l & 15] (recursive halving,
// 16 shuffles instead of 16 full butterflies).
__device__ __forceinline__ float transpose_reduce16(float (&v)[16], int lane) {
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

template <int BN, bool A_MN, bool B_MN, int EV, int AG = AG_NONE>
__global__ void __launch_bounds__(kernel_threads<EV, AG>(), 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapB, const __grid_constant__ KParams p) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base (generic addressing of the staged epilogue values;
  // the LDS/STS form measured slower for conv1: 133 -> 138 us, scripts/gpu_ab.sh)
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  // stage ring (AG_TAPS: A only, the whole B operand stays resident after it)
  constexpr int NST = AG == AG_TAPS ? taps_stages(BN) : C::STAGES;
  constexpr int SST = AG == AG_TAPS ? A_TILE_BYTES : C::STAGE_BYTES;
  uint8_t* const bres = smem + NST * SST;
  uint8_t* const bar_base = bres + (AG == AG_TAPS ? p.nkb * BN * 128 : 0);
  uint64_t* full = reinterpret_cast<uint64_t*>(bar_base);
  uint64_t* empty = full + NST;
  uint64_t* acc_full = empty + NST;
  uint64_t* acc_empty = acc_full + C::NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + C::NACC);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&mapA);
    sm100::tma_prefetch(&mapB);
    for (int s = 0; s < NST; ++s) {
      sm100::mbar_init(&full[s], 1 + gather_threads<AG>());
      sm100::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < C::NACC; ++s) {
      sm100::mbar_init(&acc_full[s], 1);
      sm100::mbar_init(&acc_empty[s], epi_warps<EV>());
    }
    if (AG == AG_TAPS) sm100::mbar_init(reinterpret_cast<uint64_t*>(bar_base + BAR_AUX), 1);
    if (AG == AG_U8 || AG == AG_U8W) {  // conv1 staging ring: full (tx) / empty (all gatherers)
      uint64_t* sfull = reinterpret_cast<uint64_t*>(bar_base + BAR_AUX);
      for (int s = 0; s < U8_NSTG; ++s) {
        sm100::mbar_init(&sfull[s], 1);
        sm100::mbar_init(&sfull[U8_NSTG + s], gather_threads<AG>());
      }
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) {
    sm100::tmem_alloc(tmem_slot, C::TMEM_COLS);
    sm100::tmem_relinquish();
  }
  if (AG == AG_U8W || (AG == AG_TAPSW && p.M <= 64)) {
    // weight gradients with M <= 64 output channels; A rows 64..127 (the second MN atom,
    // never written by the TMA) must read as zero
    for (int i = threadIdx.x; i < NST * 512; i += blockDim.x) {
      uint4* z = reinterpret_cast<uint4*>(smem + (i >> 9) * SST + 8192) + (i & 511);
      *z = make_uint4(0, 0, 0, 0);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // everything above is local (barriers, TMEM, descriptor prefetch): overlap
  // it with the previous kernel's tail, then wait for its results
  APPO_PDL_ENTRY();

  const int units = p.tiles_m * p.tiles_n * p.splits;

  if (warp == 0) {
    // TMA producer: whole warp, one elected lane issues (sm100.cuh *_warp)
    int stage = 0;
    uint32_t phase = 0;
    if (AG == AG_TAPS) {  // the whole weight operand, once, resident for every tile
      uint64_t* bb = reinterpret_cast<uint64_t*>(bar_base + BAR_AUX);
      sm100::mbar_arrive_expect_tx_warp(bb, (uint32_t)p.nkb * BN * 128);
      for (int kb = 0; kb < p.nkb; ++kb)
        sm100::tma_load_2d_warp(bres + kb * BN * 128, &mapB, bb, kb * BK, 0);
    }
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const Unit un = decode_unit(p, u);
      const int m0 = un.tm * BM, n0 = un.tn * BN;
      for (int kb = un.kb0; kb < un.kb1; ++kb) {
        sm100::mbar_wait(&empty[stage], phase ^ 1);

        uint8_t* sA = smem + stage * SST;
        uint8_t* sB = sA + A_TILE_BYTES;
        if (AG == AG_TAPSW) {
          // weight gradient of a stride-2 NHWC conv (32 input channels): K block =
          // 4 output rows x 16 columns of one image (zero padded); A = dz^T box,
          // B = BN/64 tap pairs of the input window (pixel-pair view, strided)
          // K block kb: images img0.. (p.g.nq per block) or a row block oy0.. of one
          // image (p.g.T blocks per image); A = the dz^T box (one per 64 output
          // channels), B = one window box per 64 K-values (tap, or tap pair when
          // the input has 32 channels)
          const int kpi = p.g.T;
          const int img0 = (kb / kpi) * p.g.nq, oy0 = (kb % kpi) * p.g.P;
          const int natoms = p.M > 64 ? 2 : 1;
          sm100::mbar_arrive_expect_tx_warp(&full[stage], 8192u * (natoms + BN / 64));
          for (int a = 0; a < natoms; ++a)
            sm100::tma_load_4d_warp(sA + a * 8192, &mapA, &full[stage], 64 * a, 0, oy0, img0);
          const int tpr = p.g.Cin == 32 ? p.g.ksz / 2 : p.g.ksz;  // K atoms per kernel row
#pragma unroll
          for (int j = 0; j < BN / 64; ++j) {
            const int tp = un.tn * (BN / 64) + j;
            sm100::tma_load_4d_warp(sB + j * 8192, &p.map2, &full[stage], 0, tp % tpr,
                                    2 * oy0 + tp / tpr, img0);
          }
          if (++stage == NST) {
            stage = 0;
            phase ^= 1;
          }
          continue;
        }
        if (AG == AG_U8W) {
          // dz1^T (MN-major A) box {64 ch (32 real), 32 x, 2 rows} of K block kb;
          // B (col1 rows) is built by the converter warps
          const int Ho = p.g.P / p.g.Wo;
          const int kpi = (Ho + U8W_ROWS - 1) / U8W_ROWS;
          const int img = kb / kpi;
          sm100::mbar_arrive_expect_tx_warp(&full[stage], 8192);
          sm100::tma_load_4d_warp(sA, &mapA, &full[stage], 0, 0, (kb - img * kpi) * U8W_ROWS, img);
          if (++stage == NST) {
            stage = 0;
            phase ^= 1;
          }
          continue;
        }
        if (AG == AG_TAPS) {
          // NHWC convolution, K block = one kernel tap (Cin channels): A = the
          // stride-s sampled input window of the tile's images (4-D box with
          // element strides {1, s, s, 1}), B = the tap's weight slice
          // K block = 64 channels: one tap (Cin 64) or a pair of horizontally
          // adjacent taps (Cin 32, "pixel pair" view of the input: 128 B rows)
          const int tpr = p.g.Cin == 64 ? p.g.ksz : p.g.ksz / 2;  // K blocks per kernel row
          const int kh = kb / tpr, kw = kb % tpr;
          sm100::mbar_arrive_expect_tx_warp(&full[stage], 128u * p.g.P * p.g.nq);
          sm100::tma_load_4d_warp(sA, &mapA, &full[stage], 0, kw, kh, un.tm * p.g.nq);
          if (++stage == NST) {
            stage = 0;
            phase ^= 1;
          }
          continue;
        }
        sm100::mbar_arrive_expect_tx_warp(&full[stage],
                                          has_gather<AG>() ? C::B_TILE_BYTES : C::STAGE_BYTES);
        if (has_gather<AG>()) {
          // A tile produced by the gather warps
        } else if (AG == AG_DGRAD) {
          // coarse rows (img, y, x) of the box; K block = (tap (a, b), channel atom)
          const int tap = kb / p.dg.apt, at = kb % p.dg.apt;
          sm100::tma_load_4d_warp(sA, &mapA, &full[stage], at * 64, -(tap & 1), -(tap >> 1),
                                  un.tm * p.dg.Ib);
        } else if (!A_MN) {
          sm100::tma_load_2d_warp(sA, &mapA, &full[stage], kb * BK, m0);
        } else {
          sm100::tma_load_2d_warp(sA, &mapA, &full[stage], m0, kb * BK);
          sm100::tma_load_2d_warp(sA + 8192, &mapA, &full[stage], m0 + 64, kb * BK);
        }
        if (!B_MN) {
          sm100::tma_load_2d_warp(sB, &mapB, &full[stage], kb * BK, n0);
        } else {
#pragma unroll
          for (int j = 0; j < BN / 64; ++j)
            sm100::tma_load_2d_warp(sB + j * 8192, &mapB, &full[stage], n0 + 64 * j, kb * BK);
        }
        if (++stage == NST) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // MMA issuer: the whole warp runs the loop; elect.sync inside the tcgen05
    // asm picks the issuing lane (no per-instruction waterfall, sm100.cuh)
    if (AG == AG_TAPS) sm100::mbar_wait(reinterpret_cast<uint64_t*>(bar_base + BAR_AUX), 0);
    // conv1 (AG_U8) runs on fp16 operands (exact 1024 + u8, fp16 weights)
    constexpr uint32_t idesc = AG == AG_U8 ? sm100::make_idesc_f16(BM, BN, 0, 0)
                                           : sm100::make_idesc_bf16(BM, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const Unit un = decode_unit(p, u);
      const int kb0 = un.kb0, kb1 = un.kb1;
      sm100::mbar_wait(&acc_empty[acc], acc_phase ^ 1);
      if (lane == 0) GEMM_PROF(3);
      sm100::tc_fence_after();
      const uint32_t tmem_d = tmem_base + acc * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        sm100::mbar_wait(&full[stage], phase);
        if (lane == 0 && kb == kb0) GEMM_PROF(8);
        if (has_gather<AG>()) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        sm100::tc_fence_after();
        const uint32_t a0 = sm100::smem_u32(smem + stage * SST);
        const uint32_t b0 = AG == AG_TAPS ? sm100::smem_u32(bres + kb * BN * 128) : a0 + A_TILE_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint64_t ad = A_MN ? sm100::make_sdesc(a0 + k * 2048, 8192, 1024)
                                   : sm100::make_sdesc(a0 + k * 32, 16, 1024);
          const uint64_t bd = B_MN ? sm100::make_sdesc(b0 + k * 2048, 8192, 1024)
                                   : sm100::make_sdesc(b0 + k * 32, 16, 1024);
          sm100::umma_f16_warp(tmem_d, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
        }
        sm100::umma_commit_warp(&empty[stage]);
        if (++stage == NST) {
          stage = 0;
          phase ^= 1;
        }
      }
      sm100::umma_commit_warp(&acc_full[acc]);
      if (lane == 0) GEMM_PROF(4);
      if (++acc == C::NACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if ((AG == AG_U8 || AG == AG_U8W) &&
             warp >= 2 + epi_warps<EV>() + gather_threads<AG>() / 32) {
    // conv1 staging warps: warp w owns ring slot w and stages the CTA's units
    // j = w, w + U8_NSTG, ... (a TMA issue costs ~1000 cycles of the issuing
    // warp, so the slots are filled in parallel)
    uint64_t* sfull = reinterpret_cast<uint64_t*>(bar_base + BAR_AUX);
    uint8_t* stg = bar_base + BAR_BYTES;
    int* smeta = reinterpret_cast<int*>(stg + U8_NSTG * u8_stage_bytes(p.g.Cin));
    __shared__ int sids[U8_SID_CACHE];
    if (p.g.slot_ids)
      for (int i = lane; i < min(p.g.n_traj, U8_SID_CACHE); i += 32) sids[i] = p.g.slot_ids[i];
    __syncwarp();
    const int slot = warp - (2 + epi_warps<EV>() + gather_threads<AG>() / 32);
    uint32_t sphase = 0;
    if constexpr (AG == AG_U8W) {
      // work items = the CTA's K blocks in order; item j goes to slot j % U8_NSTG
      int j = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const Unit un = decode_unit(p, u);
        for (int kb = un.kb0; kb < un.kb1; ++kb, ++j) {
          if (j % U8_NSTG != slot) continue;
          sm100::mbar_wait(&sfull[U8_NSTG + slot], sphase ^ 1);
          u8w_stage(p, kb, stg + slot * u8_stage_bytes(p.g.Cin), &sfull[slot], sids);
          sphase ^= 1;
        }
      }
    }
    for (int u = blockIdx.x + slot * gridDim.x; AG == AG_U8 && u < units;
         u += U8_NSTG * gridDim.x) {
      const Unit un = decode_unit(p, u);
      sm100::mbar_wait(&sfull[U8_NSTG + slot], sphase ^ 1);
      if (lane == 0) GEMM_PROF(0);
      if (p.g.tma)
        u8_stage_tma(p, un.tm, stg + slot * u8_stage_bytes(p.g.Cin), smeta + slot * U8_ROWS,
                     &sfull[slot], lane, sids,
                     (p.prof && blockIdx.x == 0 && u / (int)gridDim.x < 16)
                         ? p.prof + (u / gridDim.x) * 16 : nullptr);
      else
        u8_stage_bulk(p.g, un.tm, stg + slot * u8_stage_bytes(p.g.Cin), smeta + slot * U8_ROWS,
                      &sfull[slot], lane);
      if (lane == 0) GEMM_PROF(7);
      sphase ^= 1;
    }
  } else if (has_gather<AG>() && warp >= 2 + epi_warps<EV>()) {
    // A gatherers: same (unit, k block) schedule as the TMA producer
    const int gt = threadIdx.x - 32 * (2 + epi_warps<EV>());
    // byte offset of chunk (kb, c) from the window origin (NHWC: (kh, kw, ci) order)
    __shared__ int off_tab[16 * 8];
    if (AG == AG_NHWC) {
      for (int e = gt; e < p.nkb * 8; e += gather_threads<AG>()) {
        const int kk = e * 8;  // (kb*64 + c*8)
        const int tap = kk / p.g.Cin, ci0 = kk % p.g.Cin;
        const int kh = tap / p.g.ksz, kw = tap % p.g.ksz;
        off_tab[e] = 2 * ((kh * p.g.Wi + kw) * p.g.Cin + ci0);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(gather_threads<AG>()));  // gatherers only
    }
    int stage = 0;
    uint32_t phase = 0;
    if constexpr (AG == AG_U8W) {
      // one staged box per K block -> the B (col1) block of that stage
      uint8_t* stg = bar_base + BAR_BYTES;
      uint64_t* sfull = reinterpret_cast<uint64_t*>(bar_base + BAR_AUX);
      uint64_t* sempty = sfull + U8_NSTG;
      int slot = 0;
      uint32_t sphase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const Unit un = decode_unit(p, u);
        for (int kb = un.kb0; kb < un.kb1; ++kb) {
          sm100::mbar_wait(&sfull[slot], sphase);
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          u8w_convert(p.g, stg + slot * u8_stage_bytes(p.g.Cin),
                      smem + stage * SST + A_TILE_BYTES, gt);
          sm100::mbar_arrive(&full[stage]);
          sm100::mbar_arrive(&sempty[slot]);
          if (++stage == NST) {
            stage = 0;
            phase ^= 1;
          }
          if (++slot == U8_NSTG) {
            slot = 0;
            sphase ^= 1;
          }
        }
      }
    }
    if constexpr (AG == AG_U8) {
      // staged input ring (filled by the producer warp): wait slot -> convert
      // the tile channel by channel -> release the slot
      uint8_t* stg = bar_base + BAR_BYTES;
      uint64_t* sfull = reinterpret_cast<uint64_t*>(bar_base + BAR_AUX);
      uint64_t* sempty = sfull + U8_NSTG;
      int* sdelta = reinterpret_cast<int*>(stg + U8_NSTG * u8_stage_bytes(p.g.Cin));
      const int u8_plane = p.g.tma ? U8_BOX_ROWS * p.g.Wi : U8_BLK;
      int slot = 0;
      uint32_t sphase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        sm100::mbar_wait(&sfull[slot], sphase);
        if (gt == 0) GEMM_PROF(1);
        const uint32_t src0 = u8_src0(p.g, stg + slot * u8_stage_bytes(p.g.Cin),
                                      sdelta + slot * U8_ROWS, gt);
        for (int c = 0; c < p.nkb; ++c) {
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          u8_convert(p.g, src0, u8_plane, smem + stage * SST, c, gt);
          sm100::mbar_arrive(&full[stage]);
          if (gt == 0 && c == 0) GEMM_PROF(2);
          if (++stage == NST) {
            stage = 0;
            phase ^= 1;
          }
        }
        sm100::mbar_arrive(&sempty[slot]);
        if (++slot == U8_NSTG) {
          slot = 0;
          sphase ^= 1;
        }
      }
    }
    for (int u = blockIdx.x; AG == AG_NHWC && u < units; u += gridDim.x) {
      const int tm = u % p.tiles_m;
      const int z = u / (p.tiles_m * p.tiles_n);
      const int kb0 = z * p.kb_per_split;
      const int kb1 = min(kb0 + p.kb_per_split, p.nkb);
      bool valid;
      if (gt == 0) GEMM_PROF(0);
      const uint8_t* origin = gather_row_origin<AG>(p, tm * BM + (gt & 127), valid);
      for (int kb = kb0; kb < kb1; ++kb) {
        sm100::mbar_wait(&empty[stage], phase ^ 1);
        if (gt == 0 && kb == kb0) GEMM_PROF(1);
        gather_stage<AG>(p, smem + stage * SST, &full[stage], origin, valid, kb, gt,
                         off_tab);
        if (gt == 0 && kb == kb1 - 1) GEMM_PROF(2);
        if (++stage == NST) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // epilogue warps 2..: TMEM lane quarter (warp % 4), column part (warp - 2) / 4
    constexpr int EPIW = epi_warps<EV>();
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;  // column part
    constexpr int HALF = BN / (EPIW / 4);
    int acc = 0;
    uint32_t acc_phase = 0;
    constexpr int CI = EV == EV_DGRAD ? BN / 4 : 1;  // dgrad: N = 4 classes x CI channels
    constexpr int NCHB = EV == EV_DGRAD ? HALF / 16 : 1;
    float bsum[NCHB];  // dgrad bias sums: lane l < 16 owns column part*HALF + ch*16 + l
#pragma unroll
    for (int j = 0; j < NCHB; ++j) bsum[j] = 0.0f;
    // conv1 forward (N == BN == 32, HALF == 16): this warp's bias columns and
    // the scale, loaded once for every tile
    float u8_bias[16];
    float u8_scale = 1.0f;
    if constexpr (AG == AG_U8 && EV == EV_ELU_BF16) {
      u8_scale = p.epi.scale;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        u8_bias[j] = (p.epi.flags & EPI_BIAS) ? __ldg(p.epi.bias + half * HALF + j) : 0.0f;
    }
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const Unit un = decode_unit(p, u);
      const int tn = un.tn, z = un.z;
      sm100::mbar_wait(&acc_full[acc], acc_phase);
      if (warp == 2 && lane == 0) GEMM_PROF(5);
      sm100::tc_fence_after();
      const int m = un.tm * BM + q * 32 + lane;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      if constexpr (EV == EV_DGRAD) {
        // all ELU' operands of this warp's columns first (independent of the
        // accumulator), then TMEM chunk by chunk
        constexpr int NCH = HALF / 16;
        int64_t off[NCH];
        uint4 av[NCH][2];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          off[ch] = dgrad_offset<CI>(p, m, half * HALF + ch * 16);
          const uint4* a4 = reinterpret_cast<const uint4*>(p.epi.aux + (off[ch] < 0 ? 0 : off[ch]));
          av[ch][0] = off[ch] < 0 ? make_uint4(0, 0, 0, 0) : __ldg(a4);
          av[ch][1] = off[ch] < 0 ? make_uint4(0, 0, 0, 0) : __ldg(a4 + 1);
        }
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          uint32_t r[16];
          sm100::tmem_ld16(tbase + half * HALF + ch * 16, r);
          sm100::tmem_ld_wait();
          float sv[16];
          if (off[ch] >= 0) {
            dgrad_finish(p, off[ch], r, av[ch], sv);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) sv[j] = 0.0f;
          }
          bsum[ch] += transpose_reduce16(sv, lane);
        }
      } else {
#pragma unroll 1
        for (int c = half * HALF; c < (half + 1) * HALF; c += 16) {
          if (tn * BN + c >= p.N) break;  // warp-uniform
          uint32_t r[16];
          sm100::tmem_ld16(tbase + c, r);
          sm100::tmem_ld_wait();
          if constexpr (EV == EV_DELU_BSUM) {
            float sv[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) sv[j] = 0.0f;
            epilogue_dispatch<EV>(p, m, tn * BN + c, z, r, sv);
            const float t = transpose_reduce16(sv, lane);  // lane l < 16: column c + l
            if (lane < 16)
              atomicAdd(p.epi.bsum_acc + (size_t)(blockIdx.x % 16) * p.epi.bsum_mod +
                            (tn * BN + c + lane) % p.epi.bsum_mod,
                        (unsigned long long)llrint((double)t * 4294967296.0));
            continue;
          }
          if constexpr (AG == AG_U8 && EV == EV_ELU_BF16) {
            // conv1: the warp's 16 columns never change (N == BN), so scale and
            // bias stay in registers; x*scale + bias -> ELU -> bf16 row store
            const int mo = u8_out_row(p.g, m);
            if (mo >= 0 && mo < p.M) {
              uint32_t w[8];
#pragma unroll
              for (int q = 0; q < 8; ++q)
                w[q] = pack_bf16(elu_fast(fmaf(__uint_as_float(r[2 * q]), u8_scale, u8_bias[2 * q])),
                                 elu_fast(fmaf(__uint_as_float(r[2 * q + 1]), u8_scale,
                                               u8_bias[2 * q + 1])));
              uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.epi.out) +
                                                    (size_t)mo * p.epi.ldo + c);
              dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
              dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
            }
          } else if constexpr (AG == AG_U8) {  // tile rows -> (output row, x); padding skipped
            const int mo = u8_out_row(p.g, m);
            if (mo >= 0) epilogue_dispatch<EV>(p, mo, tn * BN + c, z, r);
          } else if constexpr (AG == AG_TAPS) {  // tile = nq whole images, rows beyond are padding
            const int rpt = p.g.P * p.g.nq, loc = m - un.tm * BM;
            if (loc < rpt) epilogue_dispatch<EV>(p, un.tm * rpt + loc, tn * BN + c, z, r);
          } else if constexpr (EV == EV_F32 && AG == AG_NONE) {
            // fp32 rows: lane pairs (row m, row m ^ 1) swap half-chunks so each
            // 16-byte store instruction of the warp covers whole 32-byte sectors
            const int n0 = tn * BN + c;
            const bool paired = __all_sync(0xffffffffu, m < p.M) && n0 + 16 <= p.N &&
                                (p.epi.ldo & 7) == 0;
            if (!paired) {
              epilogue_dispatch<EV>(p, m, n0, z, r);
            } else {
              const Epilogue& e = p.epi;
              float v[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]) * e.scale;
              if (e.flags & EPI_BIAS) {
                const float4* b4 = reinterpret_cast<const float4*>(e.bias + n0);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const float4 b = __ldg(b4 + j);
                  v[4 * j] += b.x; v[4 * j + 1] += b.y; v[4 * j + 2] += b.z; v[4 * j + 3] += b.w;
                }
              }
              const int par = lane & 1;
              float* base = reinterpret_cast<float*>(e.out) + (size_t)(m - par) * e.ldo + n0 + 4 * par;
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                float snd[4], rcv[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  snd[k] = par ? v[8 * q + k] : v[8 * q + 4 + k];
                  rcv[k] = __shfl_xor_sync(0xffffffffu, snd[k], 1);
                }
                const float4 first = par ? make_float4(rcv[0], rcv[1], rcv[2], rcv[3])
                                         : make_float4(v[8 * q], v[8 * q + 1], v[8 * q + 2], v[8 * q + 3]);
                const float4 second = par ? make_float4(v[8 * q + 4], v[8 * q + 5], v[8 * q + 6], v[8 * q + 7])
                                          : make_float4(rcv[0], rcv[1], rcv[2], rcv[3]);
                *reinterpret_cast<float4*>(base + 8 * q) = first;             // row m - par
                *reinterpret_cast<float4*>(base + e.ldo + 8 * q) = second;    // row m - par + 1
              }
            }
          } else if constexpr (EV == EV_SPLIT) {
            // split-K fp32 partials: the same sector-aligned lane-pair stores
            const int n0 = tn * BN + c;
            const bool paired = __all_sync(0xffffffffu, m < p.M) && n0 + 16 <= p.N &&
                                (p.N & 7) == 0;
            if (!paired) {
              epilogue_dispatch<EV>(p, m, n0, z, r);
            } else {
              const int par = lane & 1;
              float* base = p.partial + ((size_t)z * p.M + (m - par)) * p.N + n0 + 4 * par;
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                uint32_t rcv[4];
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  rcv[k] = __shfl_xor_sync(0xffffffffu, par ? r[8 * q + k] : r[8 * q + 4 + k], 1);
                const uint4 first = par ? make_uint4(rcv[0], rcv[1], rcv[2], rcv[3])
                                        : make_uint4(r[8 * q], r[8 * q + 1], r[8 * q + 2], r[8 * q + 3]);
                const uint4 second = par ? make_uint4(r[8 * q + 4], r[8 * q + 5], r[8 * q + 6], r[8 * q + 7])
                                         : make_uint4(rcv[0], rcv[1], rcv[2], rcv[3]);
                *reinterpret_cast<uint4*>(base + 8 * q) = first;
                *reinterpret_cast<uint4*>(base + p.N + 8 * q) = second;
              }
            }
          } else {
            epilogue_dispatch<EV>(p, m, tn * BN + c, z, r);
          }
        }
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&acc_empty[acc]);
      if (warp == 2 && lane == 0) GEMM_PROF(6);
      if (++acc == C::NACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if constexpr (EV == EV_DELU_BSUM) {  // last CTA converts the bias-gradient sums
      const Epilogue& e = p.epi;
      __threadfence();
      asm volatile("bar.sync 2, %0;" ::"n"(32 * EPIW) : "memory");  // epilogue warps only
      __shared__ unsigned last_cta_b;
      if (warp == 2 && lane == 0) last_cta_b = atomicAdd(e.bsum_cnt, 1u) == gridDim.x - 1;
      asm volatile("bar.sync 2, %0;" ::"n"(32 * EPIW) : "memory");
      if (last_cta_b) {
        __threadfence();
        const int et = threadIdx.x - 64;
        for (int n = et; n < e.bsum_mod; n += 32 * EPIW) {
          unsigned long long v = 0;
          for (int k = 0; k < 16; ++k) v += atomicExch(e.bsum_acc + (size_t)k * e.bsum_mod + n, 0ull);
          e.bsum_out[n] = (float)((double)(long long)v * (1.0 / 4294967296.0));
        }
        if (et == 0) *e.bsum_cnt = 0;
      }
    }
    if constexpr (EV == EV_DGRAD) {
      // bias gradient: rows -> warp sums -> 2^-32 fixed-point atomics (order
      // independent), last CTA converts and re-zeroes (model_kernels.cu scheme)
      const DgradP& g = p.dg;
      if (lane < 16) {
#pragma unroll
        for (int ch = 0; ch < NCHB; ++ch)
          atomicAdd(g.bacc + (size_t)(blockIdx.x % 16) * CI + (half * HALF + ch * 16 + lane) % CI,
                    (unsigned long long)llrint((double)bsum[ch] * 4294967296.0));
      }
      __threadfence();
      asm volatile("bar.sync 2, %0;" ::"n"(32 * EPIW) : "memory");  // epilogue warps only
      __shared__ unsigned last_cta;
      if (warp == 2 && lane == 0) last_cta = atomicAdd(g.bcnt, 1u) == gridDim.x - 1;
      asm volatile("bar.sync 2, %0;" ::"n"(32 * EPIW) : "memory");
      if (last_cta) {
        __threadfence();
        const int et = threadIdx.x - 64;
        for (int n = et; n < CI; n += 32 * EPIW) {
          unsigned long long v = 0;
          for (int k = 0; k < 16; ++k) v += atomicExch(g.bacc + (size_t)k * CI + n, 0ull);
          g.bout[n] = (float)((double)(long long)v * (1.0 / 4294967296.0));
        }
        if (et == 0) *g.bcnt = 0;
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// Split-K reduction + epilogue (fp32 outputs only).  Block = 32 consecutive
// outputs x G split groups (G = 8 or 32 warps): group g sums splits z = g,
// g+G, ... in order, then the G group sums are added in order --
// deterministic, and enough loads in flight for the partial stream even when
// M*N is small and splits is large (G = 32 when the grid fits one wave: the
// conv1 weight gradient's 6,144 outputs x 148 splits take 2 load rounds per
// warp instead of 5).
template <int G>
__global__ void __launch_bounds__(G * 32)
    splitk_reduce_kernel(int M, int N, int splits, const float* __restrict__ partial, Epilogue e) {
  APPO_PDL_ENTRY();
  const int64_t total = (int64_t)M * N;
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t i = ((int64_t)blockIdx.x * 32 + lane) * 4;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (i < total) {
    const float4* p = reinterpret_cast<const float4*>(partial + (size_t)g * total + i);
    const size_t step = (size_t)G * total / 4;  // G splits, in float4 units
    int z = g;
    for (; z + 3 * G < splits; z += 4 * G, p += 4 * step) {
      const float4 a0 = __ldg(p), a1 = __ldg(p + step), a2 = __ldg(p + 2 * step),
                   a3 = __ldg(p + 3 * step);
      s.x += a0.x; s.y += a0.y; s.z += a0.z; s.w += a0.w;
      s.x += a1.x; s.y += a1.y; s.z += a1.z; s.w += a1.w;
      s.x += a2.x; s.y += a2.y; s.z += a2.z; s.w += a2.w;
      s.x += a3.x; s.y += a3.y; s.z += a3.z; s.w += a3.w;
    }
    for (; z < splits; z += G, p += step) {
      const float4 a0 = __ldg(p);
      s.x += a0.x; s.y += a0.y; s.z += a0.z; s.w += a0.w;
    }
  }
  __shared__ float4 sh[G][32];
  sh[g][lane] = s;
  __syncthreads();
  if (g != 0 || i >= total) return;
  float4 t = sh[0][lane];
#pragma unroll 8
  for (int k = 1; k < G; ++k) {
    const float4 u = sh[k][lane];
    t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
  }
  const float tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int m = (int)((i + q) / N), n = (int)((i + q) % N);
    float x = tv[q] * e.scale;
    if (e.flags & EPI_BIAS) x += e.bias[n];
    const size_t o = (e.flags & EPI_TRANS) ? (size_t)n * e.ldo + m : (size_t)m * e.ldo + n;
    float* dst = reinterpret_cast<float*>(e.out) + o;
    *dst = (e.flags & EPI_ACCUM) ? *dst + x : x;
  }
}

// Few splits, many outputs (GRU / FC weight gradients): one thread per 4
// consecutive outputs, splits summed in order (deterministic).
__global__ void __launch_bounds__(256)
    splitk_reduce4_kernel(int M, int N, int splits, const float* __restrict__ partial, Epilogue e) {
  APPO_PDL_ENTRY();
  const int64_t total = (int64_t)M * N;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i >= total) return;
  float4 s = __ldg(reinterpret_cast<const float4*>(partial + i));
  for (int z = 1; z < splits; ++z) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(partial + (size_t)z * total + i));
    s.x += v.x;
    s.y += v.y;
    s.z += v.z;
    s.w += v.w;
  }
  const float t[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int m = (int)((i + k) / N), n = (int)((i + k) % N);
    float x = t[k] * e.scale;
    if (e.flags & EPI_BIAS) x += e.bias[n];
    const size_t o = (e.flags & EPI_TRANS) ? (size_t)n * e.ldo + m : (size_t)m * e.ldo + n;
    float* dst = reinterpret_cast<float*>(e.out) + o;
    *dst = (e.flags & EPI_ACCUM) ? *dst + x : x;
  }
}

// Any shape (M*N not a multiple of 4): one thread per output, splits in order.
__global__ void __launch_bounds__(256)
    splitk_reduce1_kernel(int M, int N, int splits, const float* __restrict__ partial, Epilogue e) {
  APPO_PDL_ENTRY();
  const int64_t total = (int64_t)M * N;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  float t = 0.0f;
  for (int z = 0; z < splits; ++z) t += __ldg(partial + (size_t)z * total + i);
  const int m = (int)(i / N), n = (int)(i % N);
  float x = t * e.scale;
  if (e.flags & EPI_BIAS) x += e.bias[n];
  const size_t o = (e.flags & EPI_TRANS) ? (size_t)n * e.ldo + m : (size_t)m * e.ldo + n;
  float* dst = reinterpret_cast<float*>(e.out) + o;
  *dst = (e.flags & EPI_ACCUM) ? *dst + x : x;
}

int launch_splitk_reduce(Ctx* c, int M, int N, int splits, const float* partial,
                         const Epilogue& epi) {
  const int64_t total = (int64_t)M * N;
  c->next_bytes = (double)splits * total * 4 + (double)total * 4;
  if (total % 4 != 0) {
    APPO_LAUNCH(c, splitk_reduce1_kernel, (int)((total + 255) / 256), 256, 0, M, N, splits,
                partial, epi);
  } else if (splits <= 16) {
    APPO_LAUNCH(c, splitk_reduce4_kernel, (int)((total / 4 + 255) / 256), 256, 0, M, N, splits,
                partial, epi);
  } else {
    const int grid = (int)((total / 4 + 31) / 32);
    if ((int64_t)grid * 1024 <= (int64_t)c->num_sms * 2048)
      APPO_LAUNCH(c, splitk_reduce_kernel<32>, grid, 1024, 0, M, N, splits, partial, epi);
    else
      APPO_LAUNCH(c, splitk_reduce_kernel<8>, grid, 256, 0, M, N, splits, partial, epi);
  }
  return APPO_OK;
}

// ---- host side: tensor maps ----------------------------------------------------

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2D bf16 map over a row-major [outer][inner] region with leading dim ld
// (elements), box {64, box_outer}, 128B swizzle, zero OOB fill.
int make_map(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t ld,
             int box_outer) {
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return APPO_ERR_RESOURCE;
  }
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || ((ld * 2) & 15)) {
    set_error("gemm operand must be 16-byte aligned with a leading dim multiple of 8");
    return APPO_ERR_CONTRACT;
  }
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64u, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return APPO_ERR_CONTRACT;
  }
  return APPO_OK;
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Pick the compile-time epilogue for this call (generic when nothing fits).
int choose_ev(const KParams& p) {
  const Epilogue& e = p.epi;
  if (p.splits > 1) return (p.N % 4 == 0) ? EV_SPLIT : EV_GENERIC;
  const int f = e.flags;
  if (f & (EPI_TRANS | EPI_ACCUM)) return EV_GENERIC;
  if (f & EPI_BF16) {
    if ((e.ldo & 7) || !al16(e.out)) return EV_GENERIC;
    const int g = f & ~EPI_BF16;
    if (g == (EPI_BIAS | EPI_ELU) || g == EPI_ELU)
      return (!(f & EPI_BIAS) || al16(e.bias)) ? EV_ELU_BF16 : EV_GENERIC;
    if (g == EPI_DELU) {
      if ((e.ld_aux & 7) || !al16(e.aux)) return EV_GENERIC;
      return e.bsum_out ? EV_DELU_BSUM : EV_DELU_BF16;
    }
    if (g == 0) return EV_BF16;
    return EV_GENERIC;
  }
  if ((f & ~EPI_BIAS) == 0 && !(e.ldo & 3) && al16(e.out) && (!(f & EPI_BIAS) || al16(e.bias)))
    return EV_F32;
  return EV_GENERIC;
}

template <int BN, bool A_MN, bool B_MN, int EV, int AG = AG_NONE>
int launch_gemm(Ctx* c, const CUtensorMap& ma, const CUtensorMap& mb, const KParams& p) {
  using C = Cfg<BN>;
  auto kern = gemm_bf16_kernel<BN, A_MN, B_MN, EV, AG>;
  // conv1: input staging ring after the barriers (+16 B overread slack)
  const int smem_bytes =
      AG == AG_TAPS
          ? taps_stages(BN) * A_TILE_BYTES + p.nkb * BN * 128 + 1024 + BAR_BYTES
          : C::SMEM_BYTES +
                ((AG == AG_U8 || AG == AG_U8W) ? U8_NSTG * u8_stage_bytes(p.g.Cin) + 64 : 0);
  constexpr int kThreads = kernel_threads<EV, AG>();
  static int attr_bytes[64] = {};
  int dev = c->device & 63;
  if (attr_bytes[dev] < smem_bytes) {
    APPO_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem_bytes));
    attr_bytes[dev] = smem_bytes;
  }
  const int units = p.tiles_m * p.tiles_n * p.splits;
  int per_sm = (227 * 1024) / smem_bytes;
  const int tmem_per_sm = 512 / C::TMEM_COLS;
  per_sm = per_sm < tmem_per_sm ? per_sm : tmem_per_sm;
  if (per_sm < 1) per_sm = 1;
  int grid = c->num_sms * per_sm;
  if (grid > units) grid = units;
  c->next_name = "gemm_bf16_tcgen05";
  if (c->timing && c->timing_filter == "gemm_shapes") {
    // per-shape tag for the profiling scripts (names must outlive the report)
    static std::set<std::string> names;
    char buf[96];
    snprintf(buf, sizeof(buf), "gemm %dx%dx%d bn%d s%d %s%s%s", p.M, p.N, p.K, BN, p.splits,
             A_MN ? "M" : "K", B_MN ? "M" : "K",
             AG == AG_U8 ? " conv1-u8" : AG == AG_U8W ? " conv1-wgrad" : AG == AG_DGRAD ? " dgrad"
             : AG == AG_TAPS ? " conv-taps" : AG == AG_TAPSW ? " taps-wgrad"
             : AG ? " conv-nhwc" : "");
    c->next_name = names.insert(buf).first->c_str();
  }
  c->next_flops = 2.0 * p.M * p.N * p.K;
  c->next_bytes = 2.0 * ((double)p.M * p.K + (double)p.N * p.K) +
                  (double)p.M * p.N * ((p.epi.flags & EPI_BF16) ? 2 : 4) * (p.splits > 1 ? p.splits : 1);
  if (AG == AG_U8) {  // implicit conv1: the A operand is the u8 images, read once
    const double imgs = (double)p.M / p.g.P;
    c->next_bytes = imgs * p.g.Cin * p.g.Hi * p.g.Wi + 2.0 * p.N * p.K + 2.0 * p.M * p.N;
  } else if (AG == AG_NHWC) {
    const double imgs = (double)p.M / p.g.P;
    c->next_bytes = 2.0 * imgs * p.g.Hi * p.g.Wi * p.g.Cin + 2.0 * p.N * p.K + 2.0 * p.M * p.N;
  }
  if (AG == AG_DGRAD) {  // useful MACs only (taps inside the kernel), HBM bytes
    const DgradP& g = p.dg;
    c->next_flops = 2.0 * g.n_img * p.g.Hi * p.g.Wi * (double)p.g.Cin * g.Ci;
    c->next_bytes = 2.0 * g.n_img * ((double)p.g.Hi * p.g.Wi * p.g.Cin + 3.0 * g.Hi * g.Wi * g.Ci);
  }
  if (AG && !(c->timing && c->timing_filter == "gemm_shapes"))
    c->next_name = AG == AG_DGRAD  ? "gemm_dgrad_implicit_tcgen05"
                   : AG == AG_U8   ? "gemm_conv1_u8_implicit_tcgen05"
                   : AG == AG_U8W  ? "gemm_conv1_wgrad_implicit_tcgen05"
                   : AG == AG_TAPS ? "gemm_conv_taps_implicit_tcgen05"
                   : AG == AG_TAPSW ? "gemm_conv_taps_wgrad_tcgen05"
                                   : "gemm_conv_nhwc_gather_tcgen05";
  // phase timeline of CTA 0 (diagnostics): APPO_GEMM_PROF=<AG mode number>
  static long long* prof = nullptr;
  const char* pe = getenv("APPO_GEMM_PROF");
  if (pe && atoi(pe) == AG) {
    if (!prof) cudaMalloc(&prof, sizeof(long long) * 256);
    cudaMemsetAsync(prof, 0, sizeof(long long) * 256, c->stream);
    KParams q = p;
    q.prof = prof;
    APPO_LAUNCH(c, kern, grid, kThreads, smem_bytes, ma, mb, q);
    long long h[256];
    cudaStreamSynchronize(c->stream);
    cudaMemcpy(h, prof, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[gemm prof] AG=%d M=%d N=%d K=%d units of CTA0 (cycles): g0 g1 g2 | mma_accfree mma_commit | epi_start epi_done | g7 g8 g9 g10\n", AG, p.M, p.N, p.K);
    for (int i = 0; i < 16; ++i) {
      fprintf(stderr, "  u%-2d", i);
      for (int k = 0; k < 11; ++k) fprintf(stderr, " %7lld", h[i * 16 + k] ? h[i * 16 + k] - h[0] : -1);
      fprintf(stderr, "\n");
    }
    return APPO_OK;
  }
  APPO_LAUNCH(c, kern, grid, kThreads, smem_bytes, ma, mb, p);
  return APPO_OK;
}

template <int BN, int AG>
int launch_conv(Ctx* c, const CUtensorMap& ma, const CUtensorMap& mb, const KParams& p) {
  return choose_ev(p) == EV_ELU_BF16 ? launch_gemm<BN, false, false, EV_ELU_BF16, AG>(c, ma, mb, p)
                                     : launch_gemm<BN, false, false, EV_GENERIC, AG>(c, ma, mb, p);
}

// u8 tensor map (no swizzle) over images; dims innermost first, byte strides of dims 1..
int make_tmap_u8(CUtensorMap* map, const void* ptr, int rank, const uint64_t* dims,
                 const uint64_t* strides, const uint32_t* box) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return APPO_ERR_RESOURCE;
  if (reinterpret_cast<uintptr_t>(ptr) & 15) return APPO_ERR_CONTRACT;
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
    if (i + 1 < rank) {
      st[i] = strides[i];
      if (st[i] % 16) return APPO_ERR_CONTRACT;
    }
  }
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, rank, const_cast<void*>(ptr), d, st, b, e,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? APPO_OK : APPO_ERR_CONTRACT;
}

template <int BN, bool A_MN, bool B_MN>
int dispatch_ev(Ctx* c, const CUtensorMap& ma, const CUtensorMap& mb, const KParams& p) {
  switch (choose_ev(p)) {
    case EV_SPLIT: return launch_gemm<BN, A_MN, B_MN, EV_SPLIT>(c, ma, mb, p);
    case EV_F32: return launch_gemm<BN, A_MN, B_MN, EV_F32>(c, ma, mb, p);
    case EV_ELU_BF16: return launch_gemm<BN, A_MN, B_MN, EV_ELU_BF16>(c, ma, mb, p);
    case EV_DELU_BF16: return launch_gemm<BN, A_MN, B_MN, EV_DELU_BF16>(c, ma, mb, p);
    case EV_DELU_BSUM: return launch_gemm<BN, A_MN, B_MN, EV_DELU_BSUM>(c, ma, mb, p);
    case EV_BF16: return launch_gemm<BN, A_MN, B_MN, EV_BF16>(c, ma, mb, p);
    default: return launch_gemm<BN, A_MN, B_MN, EV_GENERIC>(c, ma, mb, p);
  }
}

template <int BN>
int dispatch_major(Ctx* c, bool amn, bool bmn, const CUtensorMap& ma, const CUtensorMap& mb,
                   const KParams& p) {
  if (!amn && !bmn) return dispatch_ev<BN, false, false>(c, ma, mb, p);
  if (!amn && bmn) return dispatch_ev<BN, false, true>(c, ma, mb, p);
  if (amn && !bmn) return dispatch_ev<BN, true, false>(c, ma, mb, p);
  return dispatch_ev<BN, true, true>(c, ma, mb, p);
}

}  // namespace

// module anchor for preload_library_kernels (slotq.cu)
const void* kanchor_gemm() { return reinterpret_cast<const void*>(&splitk_reduce_kernel<8>); }

int gemm_workspace(Ctx* c, size_t bytes, float** out) {
  if (bytes > c->ws_bytes) {
    if (c->d_ws) {
      cudaStreamSynchronize(c->stream);
      cudaFree(c->d_ws);
      c->d_ws = nullptr;
      c->ws_bytes = 0;
    }
    APPO_CUDA_TRY(cudaMalloc(&c->d_ws, bytes));
    c->ws_bytes = bytes;
  }
  *out = c->d_ws;
  return APPO_OK;
}

int gemm_bf16(Ctx* c, int M, int N, int K, const Operand& A, const Operand& B,
              const Epilogue& epi, int bn, int splits) {
  if (M <= 0 || N <= 0 || K <= 0) return APPO_OK;
  APPO_REQUIRE(bn == 32 || bn == 64 || bn == 128 || bn == 192 || bn == 256, APPO_ERR_CONTRACT,
               "gemm: unsupported BN");
  APPO_REQUIRE(!B.mn_major || bn % 64 == 0, APPO_ERR_CONTRACT, "gemm: MN-major B needs BN%64==0");
  CUtensorMap ma, mb;
  int st;
  // A: rows = M.  K-major: inner = K, outer = M.  MN-major: inner = M, outer = K.
  st = A.mn_major ? make_map(&ma, A.ptr, M, K, A.ld, BK) : make_map(&ma, A.ptr, K, M, A.ld, BM);
  if (st) return st;
  st = B.mn_major ? make_map(&mb, B.ptr, N, K, B.ld, BK) : make_map(&mb, B.ptr, K, N, B.ld, bn);
  if (st) return st;

  KParams p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.tiles_m = (M + BM - 1) / BM;
  p.tiles_n = (N + bn - 1) / bn;
  p.nkb = (K + BK - 1) / BK;
  if (splits < 1) splits = 1;
  if (splits > p.nkb) splits = p.nkb;
  p.kb_per_split = (p.nkb + splits - 1) / splits;
  p.splits = (p.nkb + p.kb_per_split - 1) / p.kb_per_split;
  p.epi = epi;
  p.partial = nullptr;
  APPO_REQUIRE(!epi.bsum_out || (p.splits == 1 && choose_ev(p) == EV_DELU_BSUM && epi.bsum_acc &&
                                 epi.bsum_cnt && epi.bsum_mod > 0 && N % 16 == 0),
               APPO_ERR_CONTRACT, "gemm: fused bias sums need an aligned bf16 DELU epilogue");
  if (p.splits > 1) {
    APPO_REQUIRE(!(epi.flags & (EPI_BF16 | EPI_ELU | EPI_DELU)), APPO_ERR_CONTRACT,
                 "gemm: split-K supports fp32 (+bias/accum/trans) epilogues only");
    st = gemm_workspace(c, (size_t)p.splits * M * N * sizeof(float), &p.partial);
    if (st) return st;
  }
  switch (bn) {
    case 32: st = dispatch_major<32>(c, A.mn_major, B.mn_major, ma, mb, p); break;
    case 64: st = dispatch_major<64>(c, A.mn_major, B.mn_major, ma, mb, p); break;
    case 128: st = dispatch_major<128>(c, A.mn_major, B.mn_major, ma, mb, p); break;
    case 192: st = dispatch_major<192>(c, A.mn_major, B.mn_major, ma, mb, p); break;
    default: st = dispatch_major<256>(c, A.mn_major, B.mn_major, ma, mb, p); break;
  }
  if (st) return st;
  if (p.splits > 1) {
    return launch_splitk_reduce(c, M, N, p.splits, p.partial, epi);
  }
  return APPO_OK;
}

// Image staging maps (p.map2 observations, p.map3 bootstrap observations) with
// boxes of box_rows input rows x all channels; false if the images are not
// 16-byte aligned (then the bulk-copy path is used).
bool make_image_maps(KParams& p, const ConvIn& in, int box_rows) {
  const uint64_t W = in.Wi, H = in.Hi, C = in.Cin, plane = W * H, od = plane * C;
  const uint32_t box[5] = {(uint32_t)W, (uint32_t)box_rows, (uint32_t)C, 1, 1};
  if (!in.slot_ids) {
    const uint64_t dims[4] = {W, H, C, (uint64_t)in.n_img};
    const uint64_t str[3] = {W, plane, (uint64_t)in.img_stride};
    return make_tmap_u8(&p.map2, in.src, 4, dims, str, box) == APPO_OK;
  }
  if (in.n_slots <= 0) return false;
  const uint64_t dims[5] = {W, H, C, (uint64_t)in.T, (uint64_t)in.n_slots};
  const uint64_t str[4] = {W, plane, od, in.slot_bytes};
  const uint64_t bdims[4] = {W, H, C, (uint64_t)in.n_slots};
  const uint64_t bstr[3] = {W, plane, in.slot_bytes};
  return make_tmap_u8(&p.map2, in.src + in.obs_off, 5, dims, str, box) == APPO_OK &&
         make_tmap_u8(&p.map3, in.src + in.boot_off, 4, bdims, bstr, box) == APPO_OK;
}

EncodeTiledFnPublic tensor_map_encoder() { return get_encode(); }

int splitk_reduce(Ctx* c, int M, int N, int splits, const float* partial, const Epilogue& epi) {
  return launch_splitk_reduce(c, M, N, splits, partial, epi);
}

bool make_u8_image_maps(CUtensorMap* obs, CUtensorMap* boot, const ConvIn& in, int box_rows) {
  KParams p{};
  if (!make_image_maps(p, in, box_rows)) return false;
  *obs = p.map2;
  *boot = p.map3;
  return true;
}

int conv_implicit_bf16(Ctx* c, const ConvIn& in, int N, const Operand& W, const Epilogue& epi,
                       int bn) {
  const int K = in.u8 ? in.Cin * 64 : in.ksz * in.ksz * in.Cin;
  const int M = in.n_img * in.Ho * in.Wo;
  if (M <= 0) return APPO_OK;
  APPO_REQUIRE(!W.mn_major && K % 64 == 0 && (in.u8 || in.Cin % 8 == 0), APPO_ERR_CONTRACT,
               "conv_implicit: K-major weights, K % 64 == 0 and Cin % 8 == 0 required");
  // staging copies whole 8-row blocks from 16-byte aligned addresses at or below
  // them (images need 8-byte alignment; blocks hold at most 8*128 + 16 bytes)
  APPO_REQUIRE(!in.u8 || (in.ksz == 8 && in.s == 4 && in.Wi % 16 == 0 && in.Wi <= 128 &&
                          in.Wo <= 32 && (reinterpret_cast<uintptr_t>(in.src) & 7) == 0 &&
                          in.img_stride % 8 == 0 && in.slot_bytes % 8 == 0 &&
                          in.obs_off % 8 == 0 && in.boot_off % 8 == 0 && in.Cin <= 4),
               APPO_ERR_CONTRACT,
               "conv_implicit u8: k8 s4, W % 16 == 0, W <= 128, C <= 4, 8-byte aligned images");
  CUtensorMap mb;
  int st = make_map(&mb, W.ptr, K, N, W.ld, bn);
  if (st) return st;
  KParams p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.tiles_m = (M + BM - 1) / BM;
  p.tiles_n = (N + bn - 1) / bn;
  p.nkb = K / BK;
  p.splits = 1;
  p.kb_per_split = p.nkb;
  p.epi = epi;
  p.partial = nullptr;
  p.g = GatherP{in.src, in.img_stride, in.Ho * in.Wo, in.Wo, in.Hi, in.Wi, in.Cin, in.ksz, in.s,
                in.slot_ids, in.slot_bytes, in.obs_off, in.boot_off, in.T, in.n_traj,
                in.n_img * in.Ho};
  if (in.u8) {
    // tiles of U8_ROWS output rows x 32 columns (see u8_stage_tma)
    p.tiles_m = (p.g.nq + U8_ROWS - 1) / U8_ROWS;
    // staging by tensor-map boxes when the images are 16-byte aligned, else bulk copies
    p.g.tma = make_image_maps(p, in, U8_BOX_ROWS) ? 1 : 0;


    switch (bn) {
      case 32: return launch_conv<32, AG_U8>(c, mb, mb, p);
      default: return APPO_ERR_CONTRACT;
    }
  }
  // whole images per M tile with per-tap strided TMA boxes (no gather warps)
  if ((in.Cin == 64 || (in.Cin == 32 && in.s == 2 && in.ksz % 2 == 0)) && in.Ho * in.Wo <= BM &&
      in.s <= 8 && bn <= 128 &&
      (int64_t)K * bn * 2 + taps_stages(bn) * A_TILE_BYTES + 1024 + BAR_BYTES <= 227 * 1024 &&
      (reinterpret_cast<uintptr_t>(in.src) & 15) == 0) {
    const int per = BM / (in.Ho * in.Wo);
    CUtensorMap ma, mw;
    EncodeTiledFn enc = get_encode();
    APPO_REQUIRE(enc != nullptr, APPO_ERR_RESOURCE, "cuTensorMapEncodeTiled unavailable");
    const CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B;
    // Cin 64: pixels; Cin 32 (stride 2, even kernel): pairs of adjacent pixels
    // (128-byte rows) whose traversal stride along W is 1 pair
    const bool pairs = in.Cin == 32;
    const int wdim = pairs ? in.Wi / 2 : in.Wi;
    const int wstr = pairs ? in.s / 2 : in.s;
    cuuint64_t dims[4] = {64, (cuuint64_t)wdim, (cuuint64_t)in.Hi, (cuuint64_t)in.n_img};
    cuuint64_t str[3] = {128, (cuuint64_t)in.Wi * in.Cin * 2, (cuuint64_t)in.Hi * in.Wi * in.Cin * 2};
    cuuint32_t box[4] = {64u, (cuuint32_t)(in.Wo * wstr), (cuuint32_t)(in.Ho * in.s), (cuuint32_t)per};
    cuuint32_t es[4] = {1u, (cuuint32_t)wstr, (cuuint32_t)in.s, 1u};
    CUresult r = enc(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint8_t*>(in.src), dims,
                     str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t wd[2] = {(cuuint64_t)K, (cuuint64_t)N};
    cuuint64_t ws[1] = {(cuuint64_t)W.ld * 2};
    cuuint32_t wb[2] = {64u, (cuuint32_t)bn};
    cuuint32_t we[2] = {1u, 1u};
    CUresult r2 = enc(&mw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(W.ptr), wd, ws,
                      wb, we, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS && r2 == CUDA_SUCCESS) {
      p.g.nq = per;
      p.tiles_m = (in.n_img + per - 1) / per;
      p.nkb = K / 64;  // one tap (Cin 64) or tap pair (Cin 32) per K block
      p.kb_per_split = p.nkb;
      switch (bn) {
        case 64: return launch_conv<64, AG_TAPS>(c, ma, mw, p);
        case 128: return launch_conv<128, AG_TAPS>(c, ma, mw, p);
        default: break;
      }
    }
  }
  switch (bn) {
    case 64: return launch_conv<64, AG_NHWC>(c, mb, mb, p);
    case 128: return launch_conv<128, AG_NHWC>(c, mb, mb, p);
    default: set_error("conv_implicit: unsupported BN"); return APPO_ERR_CONTRACT;
  }
}

// 4-D bf16 map over NHWC [n][h][w][c], box {64, bw, bh, bn}, 128B swizzle,
// zero OOB fill (negative / past-the-end coordinates read as zero).
int make_map_nhwc(CUtensorMap* map, const void* ptr, int n, int h, int w, int c, int bw, int bh,
                  int bn) {
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return APPO_ERR_RESOURCE;
  }
  cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  cuuint64_t strides[3] = {(cuuint64_t)c * 2, (cuuint64_t)w * c * 2, (cuuint64_t)h * w * c * 2};
  cuuint32_t box[4] = {64u, (cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bn};
  cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (nhwc) failed: " + std::to_string((int)r));
    return APPO_ERR_CONTRACT;
  }
  return APPO_OK;
}

// conv1 weight gradient without col1: dW[co][(c,kh,kw)] = scale * sum over
// pixels of dz1[pixel][co] * obs window[pixel][(c,kh,kw)], K split across the
// CTAs, deterministic split reduce.  Returns APPO_ERR_CONTRACT when the images
// cannot be staged by TMA (caller falls back to im2col + GEMM).
int conv1_wgrad_implicit(Ctx* c, const ConvIn& in, const uint16_t* dz1, float* dw, float scale) {
  const int Ho = in.Ho, Wo = in.Wo, Cout = 32;
  APPO_REQUIRE(in.u8 && in.ksz == 8 && in.s == 4 && in.Wo <= 32 && in.Cin <= 3 && in.Wi <= 128,
               APPO_ERR_CONTRACT, "conv1_wgrad: unsupported geometry");
  KParams p{};
  p.g = GatherP{in.src, in.img_stride, Ho * Wo, Wo, in.Hi, in.Wi, in.Cin, in.ksz, in.s,
                in.slot_ids, in.slot_bytes, in.obs_off, in.boot_off, in.T, in.n_traj,
                in.n_img * Ho};
  if (!make_image_maps(p, in, U8W_BOX_ROWS)) return APPO_ERR_CONTRACT;
  p.g.tma = 1;
  // A = dz1^T: 4-D map over dz1 [img][Ho][Wo][32] bf16, box {64 ch (32 real), 32 x, 2 rows, 1}
  CUtensorMap ma, mb;
  {
    EncodeTiledFn enc = get_encode();
    APPO_REQUIRE(enc != nullptr, APPO_ERR_RESOURCE, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[4] = {(cuuint64_t)Cout, (cuuint64_t)Wo, (cuuint64_t)Ho, (cuuint64_t)in.n_img};
    cuuint64_t str[3] = {(cuuint64_t)Cout * 2, (cuuint64_t)Wo * Cout * 2,
                         (cuuint64_t)Ho * Wo * Cout * 2};
    cuuint32_t box[4] = {64u, 32u, (cuuint32_t)U8W_ROWS, 1u};
    cuuint32_t es[4] = {1u, 1u, 1u, 1u};
    CUresult r = enc(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(dz1), dims, str,
                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    APPO_REQUIRE(r == CUDA_SUCCESS, APPO_ERR_CONTRACT, "conv1_wgrad: dz1 tensor map");
    mb = ma;  // unused (B is gathered)
  }
  const int N = in.Cin * 64;
  const int kpi = (Ho + U8W_ROWS - 1) / U8W_ROWS;
  p.M = Cout;
  p.N = N;
  p.K = in.n_img * kpi * 64;
  p.tiles_m = 1;
  p.tiles_n = 1;
  p.nkb = in.n_img * kpi;
  int splits = c->num_sms;
  if (splits > p.nkb) splits = p.nkb;
  p.kb_per_split = (p.nkb + splits - 1) / splits;
  p.splits = (p.nkb + p.kb_per_split - 1) / p.kb_per_split;
  APPO_REQUIRE(N == 192, APPO_ERR_CONTRACT, "conv1_wgrad: 3 input channels expected");
  int st = gemm_workspace(c, (size_t)p.splits * Cout * N * sizeof(float), &p.partial);
  if (st) return st;
  p.epi.flags = 0;
  st = launch_gemm<192, true, true, EV_SPLIT, AG_U8W>(c, ma, mb, p);
  if (st) return st;
  Epilogue e;
  e.scale = scale;
  e.out = dw;
  e.ldo = N;
  return launch_splitk_reduce(c, Cout, N, p.splits, p.partial, e);
}

// Weight gradient of conv2-like layers (NHWC bf16 input with 32 channels,
// stride 2, even kernel, output <= 8 x 16): dw[co][(kh, kw, ci)] = sum over
// output pixels of dz[pixel][co] * x[2oy+kh][2ox+kw][ci], both operands by TMA
// (no im2col): K blocks of 4 x 16 zero-padded output pixels, B = tap-pair
// windows of the pixel-pair view.  Split-K over the CTAs + deterministic reduce.
int conv_taps_wgrad(Ctx* c, const uint16_t* x, int n_img, int Hi, int Wi, int Cin,
                    const uint16_t* dz, int Ho, int Wo, int Cout, int k, float* dw) {
  // K block = 64 zero-padded output pixels: Wb columns x Hb rows x ipk images
  const bool pairs = Cin == 32;
  const int Wb = Wo <= 8 ? 8 : 16;
  const int Hb = Wb == 16 ? 4 : (Ho <= 4 ? 4 : 8);
  const int ipk = 64 / (Wb * Hb);          // images per K block (1 when row blocks)
  const int kpi = ipk == 1 ? (Ho + Hb - 1) / Hb : 1;  // K blocks per image
  APPO_REQUIRE((Cout == 64 || Cout == 128) && (Cin == 64 || (pairs && k % 2 == 0)) && Wo <= 16 &&
                   ipk >= 1 && Wb * Hb * ipk == 64,
               APPO_ERR_CONTRACT, "conv_taps_wgrad: unsupported geometry");
  const int N = k * k * Cin;
  const int bn = N % 256 == 0 ? 256 : 192;
  APPO_REQUIRE(N % bn == 0, APPO_ERR_CONTRACT, "conv_taps_wgrad: N must be a multiple of 192/256");
  EncodeTiledFn enc = get_encode();
  APPO_REQUIRE(enc != nullptr, APPO_ERR_RESOURCE, "cuTensorMapEncodeTiled unavailable");
  KParams p{};
  CUtensorMap ma;
  {  // A = dz^T: [img][Ho][Wo][Cout] bf16, box {64, Wb, Hb, ipk} (outside Ho x Wo -> 0)
    cuuint64_t dims[4] = {(cuuint64_t)Cout, (cuuint64_t)Wo, (cuuint64_t)Ho, (cuuint64_t)n_img};
    cuuint64_t str[3] = {(cuuint64_t)Cout * 2, (cuuint64_t)Wo * Cout * 2,
                         (cuuint64_t)Ho * Wo * Cout * 2};
    cuuint32_t box[4] = {64u, (cuuint32_t)Wb, (cuuint32_t)Hb, (cuuint32_t)ipk};
    cuuint32_t es[4] = {1u, 1u, 1u, 1u};
    CUresult r = enc(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(dz), dims, str,
                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    APPO_REQUIRE(r == CUDA_SUCCESS, APPO_ERR_CONTRACT, "conv_taps_wgrad: dz map");
  }
  {  // B = input windows (pixel-pair view for 32 channels), stride-2 traversal
    const int wdim = pairs ? Wi / 2 : Wi;
    const int ws = pairs ? 1 : 2;
    cuuint64_t dims[4] = {64, (cuuint64_t)wdim, (cuuint64_t)Hi, (cuuint64_t)n_img};
    cuuint64_t str[3] = {128, (cuuint64_t)Wi * Cin * 2, (cuuint64_t)Hi * Wi * Cin * 2};
    cuuint32_t box[4] = {64u, (cuuint32_t)(Wb * ws), (cuuint32_t)(Hb * 2), (cuuint32_t)ipk};
    cuuint32_t es[4] = {1u, (cuuint32_t)ws, 2u, 1u};
    CUresult r = enc(&p.map2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(x), dims,
                     str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    APPO_REQUIRE(r == CUDA_SUCCESS, APPO_ERR_CONTRACT, "conv_taps_wgrad: input map");
  }
  p.g.ksz = k;
  p.g.Cin = Cin;
  p.g.P = Hb;    // output rows per K block
  p.g.nq = ipk;  // images per K block
  p.g.T = kpi;   // K blocks per image
  p.M = Cout;
  p.N = N;
  p.nkb = ipk == 1 ? n_img * kpi : (n_img + ipk - 1) / ipk;
  p.K = p.nkb * 64;
  p.tiles_m = 1;
  p.tiles_n = N / bn;
  int splits = (2 * c->num_sms) / p.tiles_n;
  if (splits > p.nkb) splits = p.nkb;
  if (splits < 1) splits = 1;
  p.kb_per_split = (p.nkb + splits - 1) / splits;
  p.splits = (p.nkb + p.kb_per_split - 1) / p.kb_per_split;
  int st = gemm_workspace(c, (size_t)p.splits * Cout * N * sizeof(float), &p.partial);
  if (st) return st;
  st = bn == 256 ? launch_gemm<256, true, true, EV_SPLIT, AG_TAPSW>(c, ma, ma, p)
                 : launch_gemm<192, true, true, EV_SPLIT, AG_TAPSW>(c, ma, ma, p);
  if (st) return st;
  Epilogue e;
  e.out = dw;
  e.ldo = N;
  return launch_splitk_reduce(c, Cout, N, p.splits, p.partial, e);
}

int make_tmap_bf16_3d(CUtensorMap* map, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2,
                      uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0, uint32_t b1,
                      uint32_t b2, int swizzle_bytes) {
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return APPO_ERR_RESOURCE;
  }
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (3d) failed: " + std::to_string((int)r));
    return APPO_ERR_CONTRACT;
  }
  return APPO_OK;
}

int make_tmap_bf16_4d(CUtensorMap* map, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2,
                      uint64_t d3, uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3,
                      int swizzle_bytes) {
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return APPO_ERR_RESOURCE;
  }
  cuuint64_t dims[4] = {d0, d1, d2, d3};
  cuuint64_t strides[3] = {d0 * 2, d0 * d1 * 2, d0 * d1 * d2 * 2};
  cuuint32_t box[4] = {b0, b1, b2, b3};
  cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (4d) failed: " + std::to_string((int)r));
    return APPO_ERR_CONTRACT;
  }
  return APPO_OK;
}

int conv_dgrad_s2_bf16(Ctx* c, const DgradIn& in) {
  APPO_REQUIRE(in.N == 32 || in.N == 64, APPO_ERR_CONTRACT, "conv_dgrad: N must be 32 or 64");
  APPO_REQUIRE(in.Co % 64 == 0 && (in.k == 3 || in.k == 4), APPO_ERR_CONTRACT,
               "conv_dgrad: Co % 64 == 0 and k in {3, 4}");
  APPO_REQUIRE(in.bias.out && in.bias.acc && in.bias.counter, APPO_ERR_CONTRACT,
               "conv_dgrad: bias outputs required");
  APPO_REQUIRE((reinterpret_cast<uintptr_t>(in.dz_next) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(in.dz) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(in.aprev) & 15) == 0,
               APPO_ERR_CONTRACT, "conv_dgrad: 16-byte aligned tensors required");
  DgradP g{};
  g.Hi = in.Hi;
  g.Wi = in.Wi;
  g.Ci = in.N;
  g.n_img = in.n_img;
  g.apt = in.Co / 64;
  g.Hcc = (in.Hi + 1) / 2;
  g.Wcc = (in.Wi + 1) / 2;
  // live coarse region: rows with at least one tap inside dz_next
  const int hl = in.Ho + 1 < g.Hcc ? in.Ho + 1 : g.Hcc;
  const int wl = in.Wo + 1 < g.Wcc ? in.Wo + 1 : g.Wcc;
  int wb = 1;
  while (wb < g.Wcc) wb *= 2;  // box covers every coarse column (dead ones write zeros)
  int hb = 1;
  while (hb < hl) hb *= 2;
  APPO_REQUIRE(wb * hb <= 128 && wl <= wb, APPO_ERR_CONTRACT, "conv_dgrad: image too large");
  g.Wb = wb;
  g.Hb = hb;
  g.Ib = 128 / (wb * hb);
  g.bacc = in.bias.acc;
  g.bcnt = in.bias.counter;
  g.bout = in.bias.out;
  // coarse rows beyond the box (y >= Hb) have no taps: their outputs are zero
  for (int yy = hb; yy < g.Hcc; ++yy)
    for (int py = 0; py < 2; ++py) {
      const int yi = 2 * yy + py;
      if (yi >= in.Hi) continue;
      APPO_CUDA_TRY(cudaMemset2DAsync(in.dz + (size_t)yi * in.Wi * in.N,
                                      (size_t)in.Hi * in.Wi * in.N * 2, 0,
                                      (size_t)in.Wi * in.N * 2, in.n_img, c->stream));
    }
  CUtensorMap ma, mb;
  int st = make_map_nhwc(&ma, in.dz_next, in.n_img, in.Ho, in.Wo, in.Co, g.Wb, g.Hb, g.Ib);
  if (st) return st;
  const int kdim = 4 * in.Co, ndim = 4 * in.N;
  st = make_map(&mb, in.wt, kdim, ndim, kdim, ndim);
  if (st) return st;
  KParams p{};
  p.N = ndim;
  p.K = kdim;
  p.tiles_m = (in.n_img + g.Ib - 1) / g.Ib;
  p.M = p.tiles_m * BM;
  p.tiles_n = 1;
  p.splits = 1;
  p.nkb = kdim / BK;
  p.kb_per_split = p.nkb;
  p.epi.aux = in.aprev;
  p.epi.out = in.dz;
  p.g.Hi = in.Ho;  // for the byte / flop accounting
  p.g.Wi = in.Wo;
  p.g.Cin = in.Co * in.k * in.k;
  p.dg = g;
  if (in.N == 32) return launch_gemm<128, false, false, EV_DGRAD, AG_DGRAD>(c, ma, mb, p);
  return launch_gemm<256, false, false, EV_DGRAD, AG_DGRAD>(c, ma, mb, p);
}

}  // namespace appo_b200

// ---- test hook (include/appo_internal.h) ------------------------------------------
#include "../../include/appo_internal.h"
extern "C" int appo_dbg_gemm(appo_ctx* ctx, int M, int N, int K, const void* a, int64_t lda,
                             int a_mn, const void* b, int64_t ldb, int b_mn, void* out,
                             int64_t ldo, int flags, float scale, const float* bias,
                             const void* aux, int64_t ld_aux, int bn, int splits) {
  using namespace appo_b200;
  APPO_REQUIRE(ctx != nullptr, APPO_ERR_CONTRACT, "null ctx");
  APPO_CUDA_TRY(cudaSetDevice(ctx->device));
  Epilogue e;
  e.flags = flags;
  e.scale = scale;
  e.bias = bias;
  e.aux = static_cast<const uint16_t*>(aux);
  e.ld_aux = ld_aux;
  e.out = out;
  e.ldo = ldo;
  return gemm_bf16(ctx, M, N, K, Operand{a, lda, a_mn != 0}, Operand{b, ldb, b_mn != 0}, e, bn,
                   splits);
}
