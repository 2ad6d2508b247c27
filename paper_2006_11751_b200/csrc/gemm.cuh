// Host interface of the tcgen05 GEMM engine (gemm.cu).
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "appo_common.cuh"

namespace appo_b200 {

enum EpiFlags : int {
  EPI_BIAS = 1,    // + bias[n]
  EPI_ELU = 2,     // ELU(x) after scale/bias
  EPI_DELU = 4,    // x * ELU'(aux[m][n]) where aux is the post-ELU activation (bf16)
  EPI_BF16 = 8,    // store bf16 (else fp32)
  EPI_TRANS = 16,  // store D[m][n] at out[n*ldo + m]
  EPI_ACCUM = 32,  // out += result (fp32 only)
};

struct Epilogue {
  int flags = 0;
  float scale = 1.0f;
  const float* bias = nullptr;
  const uint16_t* aux = nullptr;  // bf16 bits
  int64_t ld_aux = 0;
  void* out = nullptr;
  int64_t ldo = 0;
  // optional fused bias gradient of a DELU/bf16 epilogue: column sums of the
  // stored values folded modulo bsum_mod (NHWC channel), 2^-32 fixed-point
  // accumulators [16][bsum_mod] + CTA counter, last CTA writes bsum_out
  unsigned long long* bsum_acc = nullptr;
  unsigned* bsum_cnt = nullptr;
  float* bsum_out = nullptr;
  int bsum_mod = 0;
};

// One GEMM operand in global memory (bf16).
//   K-major : element (row r, k) at ptr[r*ld + k]   (rows = M for A, N for B)
//   MN-major: element (row r, k) at ptr[k*ld + r]
struct Operand {
  const void* ptr = nullptr;
  int64_t ld = 0;
  bool mn_major = false;
};

// D[M,N] = sum_k A[m,k] B[n,k] with epilogue.  bn in {32,64,128,192,256}
// (MN-major B needs bn % 64 == 0).  splits > 1 splits K; partial sums go to
// the ctx's workspace and a reduce kernel applies the epilogue (fp32 only).
int gemm_bf16(Ctx* c, int M, int N, int K, const Operand& A, const Operand& B,
              const Epilogue& epi, int bn, int splits = 1);

// Implicit-GEMM convolution forward: out[img, y, x][n] = epi(sum_k A[...] W[n][k])
// with the A tile gathered on the fly (no im2col in HBM).
//   u8   : CHW u8 images (conv1; K = Cin*64 in (c, kh, kw) order, k8 s4)
//   NHWC : bf16 activations [img][Hi][Wi][Cin] (K = ksz*ksz*Cin in (kh, kw, c) order)
struct ConvIn {
  const uint8_t* src = nullptr;  // first image (u8) / activation base (NHWC bf16 bytes)
  int64_t img_stride = 0;        // u8: bytes between images
  int n_img = 0, Hi = 0, Wi = 0, Cin = 0, ksz = 0, s = 0, Ho = 0, Wo = 0;
  bool u8 = false;
  // u8 images in trajectory slots: src = slot region, image r < n_traj*T is
  // step r % T of slot slot_ids[r / T], later ones the bootstrap observations
  const int32_t* slot_ids = nullptr;
  uint64_t slot_bytes = 0, obs_off = 0, boot_off = 0;
  int T = 0, n_traj = 0;
  int n_slots = 0;  // slots in the region (max slot id + 1): bounds of the tensor maps
};
int conv_implicit_bf16(Ctx* c, const ConvIn& in, int N, const Operand& W, const Epilogue& epi,
                       int bn);

// u8 image staging tensor maps (observations; bootstrap observations in slot
// mode) with boxes {W, box_rows, C}; false when the images are not 16-byte aligned.
bool make_u8_image_maps(CUtensorMap* obs, CUtensorMap* boot, const ConvIn& in, int box_rows);

// conv1 forward as a space-to-depth taps GEMM (conv1.cu): out = ELU(scale *
// (1024 + obs) . W1h^T + bias') as bf16 NHWC rows; w1h = fp16 [32][C*64].
// conv1_s2d_supported tells whether the shape / epilogue fits the kernel.
bool conv1_s2d_supported(const ConvIn& in, int N, const Epilogue& e);
int conv1_s2d_forward(Ctx* c, const ConvIn& in, const uint16_t* w1h, const Epilogue& e);
// conv1 weight gradient in the same space-to-depth form (conv1.cu):
// dw[co][(c,kh,kw)] = scale * sum_pixels dz1[pixel][co] * obs window, per-CTA
// partial sums + deterministic split-K reduce.  APPO_ERR_CONTRACT when the
// shape or the image alignment is outside the kernel's envelope.
int conv1_s2d_wgrad(Ctx* c, const ConvIn& in, const uint16_t* dz1, float* dw, float scale);

// Bias-gradient output of a fused column sum: deterministic int64 fixed-point
// accumulation (acc[16][N], zero between calls) + last-block conversion to out[N].
struct BiasOut {
  float* out = nullptr;
  unsigned long long* acc = nullptr;
  unsigned* counter = nullptr;
  int N = 0;
};

// Input gradient of a stride-2 convolution (no padding) fused with ELU' of the
// layer below and its bias gradient, as ONE implicit GEMM over the four
// sub-pixel parity classes (no dcol matrix, no col2im):
//   dz[r][y][x][n] = ELU'(aprev[r][y][x][n]) * sum_{kh,kw,co} dz_next[r][(y-kh)/2][(x-kw)/2][co] W[co][kh][kw][n]
// wt = rearranged weights [4 classes][N][4 taps][Co] (k_publish_derived); k <= 4.
struct DgradIn {
  const uint16_t* dz_next = nullptr;  // bf16 NHWC [n_img][Ho][Wo][Co]
  const uint16_t* wt = nullptr;
  const uint16_t* aprev = nullptr;    // bf16 NHWC [n_img][Hi][Wi][N] (post-ELU activation)
  uint16_t* dz = nullptr;             // bf16 NHWC [n_img][Hi][Wi][N]
  int n_img = 0, Ho = 0, Wo = 0, Co = 0, Hi = 0, Wi = 0, N = 0, k = 0;
  BiasOut bias;
};
int conv_dgrad_s2_bf16(Ctx* c, const DgradIn& in);
// conv2's input gradient (N 32, Co 64, k 4, 17x31 <- 7x14) with the shifted-view
// trick (conv2.cu); APPO_ERR_CONTRACT for any other geometry.
int conv2_dgrad(Ctx* c, const DgradIn& in);
// conv2's weight gradient dw[co][(kh, kw, ci)] from a1 / dz2 with the same planes
// (conv2.cu), per-CTA partials + deterministic reduce; APPO_ERR_CONTRACT outside.
int conv2_wgrad(Ctx* c, const uint16_t* a1, int n_img, int Hi, int Wi, const uint16_t* dz2, int Ho,
                int Wo, float* dw);

// 3-D bf16 tensor map (dims innermost first, byte strides of dims 1 and 2),
// 128B swizzle, zero OOB fill.
int make_tmap_bf16_3d(CUtensorMap* map, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2,
                      uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0, uint32_t b1,
                      uint32_t b2, int swizzle_bytes = 128);

// 4-D bf16 tensor map over a dense [d3][d2][d1][d0] array, 128B (or 64B) swizzle, zero OOB fill.
int make_tmap_bf16_4d(CUtensorMap* map, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2,
                      uint64_t d3, uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3,
                      int swizzle_bytes = 128);

// conv1 weight gradient straight from the u8 images (no im2col):
// dw[co][(c,kh,kw)] = scale * sum_pixels dz1[pixel][co] * obs window; in
// describes the images exactly as for the forward.  APPO_ERR_CONTRACT when the
// images are not TMA-stageable (16-byte alignment).
int conv1_wgrad_implicit(Ctx* c, const ConvIn& in, const uint16_t* dz1, float* dw, float scale);

// Weight gradient of a stride-2 convolution over NHWC bf16 input with 32
// (even kernel) or 64 channels (conv2, conv3), both operands by TMA (no
// im2col): dw[co][(kh,kw,ci)], Cout 64 or 128.
int conv_taps_wgrad(Ctx* c, const uint16_t* x, int n_img, int Hi, int Wi, int Cin,
                    const uint16_t* dz, int Ho, int Wo, int Cout, int k, float* dw);

// Workspace management for split-K partials (grown on demand).
int gemm_workspace(Ctx* c, size_t bytes, float** out);
// cuTensorMapEncodeTiled from the driver (nullptr if unavailable)
typedef CUresult (*EncodeTiledFnPublic)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                        const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                        const cuuint32_t*, CUtensorMapInterleave,
                                        CUtensorMapSwizzle, CUtensorMapL2promotion,
                                        CUtensorMapFloatOOBfill);
EncodeTiledFnPublic tensor_map_encoder();
// conv2 forward (k4 s2, 32 -> 64, bf16 NHWC, bias + ELU) as a space-to-depth
// taps GEMM (conv2.cu); APPO_ERR_CONTRACT outside its envelope.
int conv2_s2d_forward(Ctx* c, const uint16_t* a1, int n_img, int Hi, int Wi, int Ho, int Wo,
                      const uint16_t* w2, const Epilogue& e);
// Inference GRU step fused into its gate GEMMs + heads + sampling (gru_infer.cu):
// x, hbf bf16 [B][512]; partials scratch >= 16*B*8 floats; A <= 7.
bool gru_infer_fused_supported(int B, int A);
int gru_infer_fused(Ctx* c, int B, int A, const uint16_t* x, const uint16_t* hbf,
                    const uint16_t* w_ih, const uint16_t* w_hh, const float* b_ih,
                    const float* b_hh, const float* h_in, const float* wpi, const float* bpi,
                    const float* wv, const float* bv, uint64_t key, uint64_t counter0,
                    float* part, float* h_out, int32_t* actions, float* logp, float* values,
                    float* logits);
// Deterministic split-K reduction: out = epi(sum over `splits` fp32 partials [splits][M][N]).
int splitk_reduce(Ctx* c, int M, int N, int splits, const float* partial, const Epilogue& epi);

}  // namespace appo_b200
