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

/* The learner's fused per-trajectory loss block (traj_loss_kernel) on injected
 * core rows d_core [B + n_traj][512] (steps s = i*T + t, then the bootstrap
 * rows) and head weights: logits [B + n_traj][A], values [B + n_traj], V-trace
 * targets / pg advantages [B], GAE advantages [B] (adv_source 1, 2), dcore
 * [B][512], head gradients d_ghead = {W_pi [A][512], b_pi [A], w_v [512],
 * b_v} (the parameter layout), h_stats8 as appo_dbg_ppo_loss; versions 0,
 * current version 0.  T <= 32, A <= 7, n_traj <= 320. */
APPO_API int appo_dbg_traj_loss(appo_ctx* ctx, int n_traj, int T, int A, const float* d_core,
                                const float* d_wpi, const float* d_bpi, const float* d_wv,
                                const float* d_bv, const int32_t* d_actions,
                                const float* d_rewards, const float* d_blogp,
                                const uint8_t* d_dones, float gamma, float rho_bar,
                                float c_bar, int adv_source, float gae_lambda, float clip_low,
                                float clip_high, float value_coef, float entropy_coef,
                                float* d_logits, float* d_values, float* d_vt, float* d_pg,
                                float* d_adv, float* d_dcore, float* d_ghead, double* h_stats8);

/* Synchronous device->host copy on the ctx stream (test plumbing). */
APPO_API int appo_dbg_copy_d2h(appo_ctx* ctx, void* h_dst, const void* d_src, uint64_t bytes);

#ifdef __cplusplus
}
#endif
#endif
