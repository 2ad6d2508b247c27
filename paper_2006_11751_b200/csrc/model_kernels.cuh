// Launchers for the model's SIMT kernels (model_kernels.cu).
#pragma once
#include <stdint.h>

#include "gemm.cuh"
#include "model.cuh"

namespace appo_b200 {

constexpr int kMaxActions = 16;

// Where encoder images come from: contiguous [R][obs_dim] (slot_ids == null)
// or trajectory slots (layout v2): rows 0..n_traj*T-1 are steps s = i*T + t,
// rows n_traj*T + i are the bootstrap observations.
struct ObsSrc {
  const uint8_t* base = nullptr;
  int64_t img_stride = 0;
  const int32_t* slot_ids = nullptr;
  uint64_t slot_bytes = 0, obs_off = 0, boot_off = 0;
  int T = 0, n_traj = 0;
  int64_t obs_dim = 0;
  int n_slots = 0;  // slots in the region (max slot id + 1), 0 = unknown
};

struct SlotOffsets {
  uint64_t obs, hidden, actions, rewards, logp, dones, versions, boot_obs, boot_hidden, total;
};

struct LossHP {
  float clip_low, clip_high, value_coef, entropy_coef;
};

int k_im2col_u8(Ctx* c, const ObsSrc& src, int64_t R, const Dims& d, uint16_t* col);
int k_im2col_nhwc(Ctx* c, const uint16_t* act, int64_t R, int Hi, int Wi, int Cin, int k, int s,
                  int Ho, int Wo, uint16_t* col);
// All operands derived from a published copy, one launch: conv1 fp16 weights +
// offset-corrected bias (gemm.cu u8 path) and the sub-pixel dgrad operands
// wt[class (py,px)][ci][(2a + b)*Co + co] = W[co][py+2a][px+2b][ci] (0 outside
// the kernel) of conv2 / conv3
int k_publish_derived(Ctx* c, const uint16_t* wb, const float* pf, const Dims& d, uint16_t* c1h,
                      float* c1b, uint16_t* wt2, uint16_t* wt3);
int k_f32_to_bf16(Ctx* c, int64_t rows, const float* src, int64_t src_ld, uint16_t* dst,
                  int64_t dst_ld, int cols);
int k_gru_infer(Ctx* c, int B, int A, const float* gi, const float* gh, const float* h_in,
                const float* wpi, const float* bpi, const float* wv, const float* bv,
                uint64_t key, uint64_t counter0, float* h_out, int32_t* actions, float* logp,
                float* values, float* logits);
int k_stage_h(Ctx* c, int n_traj, int T, int t, const float* hcur, float* hin, uint16_t* hbf);
int k_gru_train(Ctx* c, int n_traj, int T, int t, const float* gi, const float* gh,
                const uint8_t* done, float* hcur, float* core, uint16_t* core_bf, float* gates);
// act != null: rows < B also get tlogp / ent of the stored action (fused log_prob_and_entropy)
int k_heads_fwd(Ctx* c, int64_t R, int A, const float* core, const float* wpi, const float* bpi,
                const float* wv, const float* bv, float* logits, float* values, int64_t B = 0,
                const int32_t* act = nullptr, float* tlogp = nullptr, float* ent = nullptr);
int k_gather_slots(Ctx* c, int n_traj, int T, const uint8_t* region, uint64_t slot_bytes,
                   const int32_t* slot_ids, const SlotOffsets& off, int32_t* act, float* rew,
                   float* blogp, uint8_t* done, int64_t* ver, float* h0);
int k_normalize(Ctx* c, int n, float* adv);
int k_ppo_loss(Ctx* c, int B, int A, const float* logits, const float* values,
               const int32_t* act, const float* blogp, const float* adv, const float* vt,
               const LossHP& hp, float* dlog, uint16_t* dhead, double* stats, const int64_t* ver,
               int64_t cur);
// dcore + head weight / bias gradients (fp32, deterministic) in one launch;
// part: >= 148 * (A+1) * 513 floats of workspace
int k_heads_bwd_fused(Ctx* c, int B, int A, const float* dlog, const float* core,
                      const float* wpi, const float* wv, float* dcore, float* part, float* gwpi,
                      float* gbpi, float* gwv, float* gbv);
// sums nb per-block head-gradient partials (layout of k_heads_bwd_fused) in block order
int k_heads_grad_reduce(Ctx* c, int A, int nb, const float* part, float* gwpi, float* gbpi,
                        float* gwv, float* gbv);
// The loss block fused per trajectory (traj_loss.cu): heads, target logp,
// V-trace (+ GAE when gae), PPO loss gradient, dcore and the head gradients
// (+ heads_grad_reduce); stats as k_ppo_loss.  part: n_traj * (A+1) * 513 floats.
bool traj_loss_supported(int n_traj, int T, int A, bool normalize_adv);
int k_traj_loss(Ctx* c, int n_traj, int T, int A, const float* core, const float* wpi,
                const float* bpi, const float* wv, const float* bv, const int32_t* act,
                const float* rew, const float* blogp, const uint8_t* done, const int64_t* ver,
                int64_t cur_version, float gamma, float rho_bar, float c_bar, bool gae,
                float lambda, const LossHP& hp, float* logits, float* values, float* vt, float* pg,
                float* adv, float* dcore, float* part, double* stats, float* gwpi, float* gbpi,
                float* gwv, float* gbv, bool reduce_heads = true);
int k_gru_bwd(Ctx* c, int n_traj, int T, int t, const float* dcore, const uint8_t* done,
              const float* gates, const float* hin, float* dnext, uint16_t* dgi, uint16_t* dgh);
int k_colsum(Ctx* c, int64_t M, int N, const void* src, int64_t ld, bool bf16, float* part,
             float* out, bool accumulate);

// persistent GRU recurrence (gru_seq.cu)
int gru_seq_supported(int n_traj);
int k_gru_seq_fwd(Ctx* c, int n_traj, int T, const float* gi, const uint16_t* whh,
                  const float* bhh, const uint8_t* done, float* hbuf, uint16_t* hbuf_bf,
                  float* core, uint16_t* core_bf, float* gates, float* hin, uint16_t* hbf);
// also writes the bias gradients gb_ih / gb_hh (sums of the gate gradients)
int k_gru_seq_bwd(Ctx* c, int n_traj, int T, const float* dcore, const uint8_t* done,
                  const float* gates, const float* hin, const uint16_t* whh, uint16_t* dghx,
                  uint16_t* dgi, uint16_t* dgh, float* gbih, float* gbhh);

}  // namespace appo_b200
