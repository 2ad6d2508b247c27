/*
 * appo_internal.h -- engine-level hooks of libappo_b200.so used by the parity
 * tests and the profiler scripts (not part of the reference-facing surface in
 * appo_capi.h).
 */
#ifndef APPO_INTERNAL_H
#define APPO_INTERNAL_H

#include "appo_capi.h"

#ifdef __cplusplus
extern "C" {
#endif

/* One call of the tcgen05 GEMM engine: D[M,N] = sum_k A[m,k] B[n,k] (bf16
 * operands, fp32 accumulate) with the fused epilogue (flags: 1 bias, 2 ELU,
 * 4 ELU' by aux, 8 bf16 out, 16 transposed store, 32 accumulate).
 * a_mn / b_mn select MN-major operands (element (r,k) at ptr[k*ld + r]). */
APPO_API int appo_dbg_gemm(appo_ctx* ctx, int M, int N, int K, const void* d_a, int64_t lda,
                           int a_mn, const void* d_b, int64_t ldb, int b_mn, void* d_out,
                           int64_t ldo, int flags, float scale, const float* d_bias,
                           const void* d_aux, int64_t ld_aux, int bn, int splits);

/* Device pointers of the model's fp32 master parameters / last gradient /
 * published bf16 copy (for tests that compare against the oracle). */
APPO_API int appo_dbg_model_ptrs(appo_ctx* ctx, float** theta, float** grad, void** pub_bf16);

/* The learner's fused PPO loss kernel on injected logits [B][A] / values [B]:
 * d_dlog [B][A+1] receives dL/dlogits and dL/dV per sample (batch-mean loss);
 * h_stats8 = {policy, value, entropy, total, mean_ratio, -, lag mean, lag max}. */
APPO_API int appo_dbg_ppo_loss(appo_ctx* ctx, int B, int A, const float* d_logits,
                               const float* d_values, const int32_t* d_actions,
                               const float* d_blogp, const float* d_adv, const float* d_vt,
                               float clip_low, float clip_high, float value_coef,
                               float entropy_coef, float* d_dlog, double* h_stats8);

/* Synchronous device->host copy on the ctx stream (test plumbing). */
APPO_API int appo_dbg_copy_d2h(appo_ctx* ctx, void* h_dst, const void* d_src, uint64_t bytes);

#ifdef __cplusplus
}
#endif
#endif
