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
constexpr int STAGES = 4;
constexpr int THREADS = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue
constexpr int A_TILE_BYTES = BM * BK * 2;  // 16 KB

struct KParams {
  int M, N, K;
  int tiles_m, tiles_n, splits, kb_per_split, nkb;
  Epilogue epi;
  float* partial;  // split-K workspace [splits][M][N]
};

template <int BN>
struct Cfg {
  static constexpr int B_TILE_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_TILE_BYTES + B_TILE_BYTES;
  static constexpr int TMEM_COLS = (2 * BN <= 32)    ? 32
                                   : (2 * BN <= 64)  ? 64
                                   : (2 * BN <= 128) ? 128
                                   : (2 * BN <= 256) ? 256
                                                     : 512;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

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
    if (e.flags & EPI_ELU) x = x > 0.0f ? x : expm1f(x);
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
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int EV>
__device__ __forceinline__ void epilogue_dispatch(const KParams& p, int m, int n0, int z,
                                                  const uint32_t (&r)[16]) {
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
      for (int j = 0; j < 16; ++j) v[j] = v[j] > 0.0f ? v[j] : expm1f(v[j]);
    }
    if constexpr (EV == EV_DELU_BF16) {
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
      dst[0] = make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                          pack_bf16(v[6], v[7]));
      dst[1] = make_uint4(pack_bf16(v[8], v[9]), pack_bf16(v[10], v[11]),
                          pack_bf16(v[12], v[13]), pack_bf16(v[14], v[15]));
    }
  }
}

template <int BN, bool A_MN, bool B_MN, int EV>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapB, const KParams p) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&mapA);
    sm100::tma_prefetch(&mapB);
    for (int s = 0; s < STAGES; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&acc_full[s], 1);
      sm100::mbar_init(&acc_empty[s], 8);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) {
    sm100::tmem_alloc(tmem_slot, C::TMEM_COLS);
    sm100::tmem_relinquish();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int units = p.tiles_m * p.tiles_n * p.splits;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int tm = u % p.tiles_m;
        const int tn = (u / p.tiles_m) % p.tiles_n;
        const int z = u / (p.tiles_m * p.tiles_n);
        const int kb0 = z * p.kb_per_split;
        const int kb1 = min(kb0 + p.kb_per_split, p.nkb);
        const int m0 = tm * BM, n0 = tn * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = smem + stage * C::STAGE_BYTES;
          uint8_t* sB = sA + A_TILE_BYTES;
          sm100::mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          if (!A_MN) {
            sm100::tma_load_2d(sA, &mapA, &full[stage], kb * BK, m0);
          } else {
            sm100::tma_load_2d(sA, &mapA, &full[stage], m0, kb * BK);
            sm100::tma_load_2d(sA + 8192, &mapA, &full[stage], m0 + 64, kb * BK);
          }
          if (!B_MN) {
            sm100::tma_load_2d(sB, &mapB, &full[stage], kb * BK, n0);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              sm100::tma_load_2d(sB + j * 8192, &mapB, &full[stage], n0 + 64 * j, kb * BK);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = sm100::make_idesc_bf16(BM, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int z = u / (p.tiles_m * p.tiles_n);
        const int kb0 = z * p.kb_per_split;
        const int kb1 = min(kb0 + p.kb_per_split, p.nkb);
        sm100::mbar_wait(&acc_empty[acc], acc_phase ^ 1);
        sm100::tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(&full[stage], phase);
          sm100::tc_fence_after();
          const uint32_t a0 = sm100::smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t b0 = a0 + A_TILE_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? sm100::make_sdesc(a0 + k * 2048, 8192, 1024)
                                     : sm100::make_sdesc(a0 + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? sm100::make_sdesc(b0 + k * 2048, 8192, 1024)
                                     : sm100::make_sdesc(b0 + k * 32, 16, 1024);
            sm100::umma_f16(tmem_d, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          sm100::umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        sm100::umma_commit(&acc_full[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // epilogue warps 2..9: TMEM lane quarter (warp % 4), column half (warp - 2) / 4
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    constexpr int HALF = BN / 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int tm = u % p.tiles_m;
      const int tn = (u / p.tiles_m) % p.tiles_n;
      const int z = u / (p.tiles_m * p.tiles_n);
      sm100::mbar_wait(&acc_full[acc], acc_phase);
      sm100::tc_fence_after();
      const int m = tm * BM + q * 32 + lane;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = half * HALF; c < (half + 1) * HALF; c += 16) {
        if (tn * BN + c >= p.N) break;  // warp-uniform
        uint32_t r[16];
        sm100::tmem_ld16(tbase + c, r);
        sm100::tmem_ld_wait();
        epilogue_dispatch<EV>(p, m, tn * BN + c, z, r);
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&acc_empty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
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

// Split-K reduction + epilogue (fp32 outputs only).
__global__ void splitk_reduce_kernel(int M, int N, int splits, const float* __restrict__ partial,
                                     Epilogue e) {
  const int64_t total = (int64_t)M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.0f;
    for (int z = 0; z < splits; ++z) s += partial[(size_t)z * total + i];
    const int m = (int)(i / N), n = (int)(i % N);
    float x = s * e.scale;
    if (e.flags & EPI_BIAS) x += e.bias[n];
    const size_t o = (e.flags & EPI_TRANS) ? (size_t)n * e.ldo + m : (size_t)m * e.ldo + n;
    float* dst = reinterpret_cast<float*>(e.out) + o;
    *dst = (e.flags & EPI_ACCUM) ? *dst + x : x;
  }
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
    if (g == EPI_DELU) return ((e.ld_aux & 7) || !al16(e.aux)) ? EV_GENERIC : EV_DELU_BF16;
    if (g == 0) return EV_BF16;
    return EV_GENERIC;
  }
  if ((f & ~EPI_BIAS) == 0 && !(e.ldo & 3) && al16(e.out) && (!(f & EPI_BIAS) || al16(e.bias)))
    return EV_F32;
  return EV_GENERIC;
}

template <int BN, bool A_MN, bool B_MN, int EV>
int launch_gemm(Ctx* c, const CUtensorMap& ma, const CUtensorMap& mb, const KParams& p) {
  using C = Cfg<BN>;
  auto kern = gemm_bf16_kernel<BN, A_MN, B_MN, EV>;
  static bool attr_set[64] = {};
  int dev = c->device & 63;
  if (!attr_set[dev]) {
    APPO_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       C::SMEM_BYTES));
    attr_set[dev] = true;
  }
  const int units = p.tiles_m * p.tiles_n * p.splits;
  int per_sm = (227 * 1024) / C::SMEM_BYTES;
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
    snprintf(buf, sizeof(buf), "gemm %dx%dx%d bn%d s%d %s%s", p.M, p.N, p.K, BN, p.splits,
             A_MN ? "M" : "K", B_MN ? "M" : "K");
    c->next_name = names.insert(buf).first->c_str();
  }
  c->next_flops = 2.0 * p.M * p.N * p.K;
  c->next_bytes = 2.0 * ((double)p.M * p.K + (double)p.N * p.K) +
                  (double)p.M * p.N * ((p.epi.flags & EPI_BF16) ? 2 : 4) * (p.splits > 1 ? p.splits : 1);
  APPO_LAUNCH(c, kern, grid, THREADS, C::SMEM_BYTES, ma, mb, p);
  return APPO_OK;
}

template <int BN, bool A_MN, bool B_MN>
int dispatch_ev(Ctx* c, const CUtensorMap& ma, const CUtensorMap& mb, const KParams& p) {
  switch (choose_ev(p)) {
    case EV_SPLIT: return launch_gemm<BN, A_MN, B_MN, EV_SPLIT>(c, ma, mb, p);
    case EV_F32: return launch_gemm<BN, A_MN, B_MN, EV_F32>(c, ma, mb, p);
    case EV_ELU_BF16: return launch_gemm<BN, A_MN, B_MN, EV_ELU_BF16>(c, ma, mb, p);
    case EV_DELU_BF16: return launch_gemm<BN, A_MN, B_MN, EV_DELU_BF16>(c, ma, mb, p);
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

  KParams p;
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
    const int64_t total = (int64_t)M * N;
    int grid = (int)((total + 255) / 256);
    if (grid > c->num_sms * 8) grid = c->num_sms * 8;
    APPO_LAUNCH(c, splitk_reduce_kernel, grid, 256, 0, M, N, p.splits, p.partial, epi);
  }
  return APPO_OK;
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
