/*
 * appo_capi.h -- C ABI of the B200-native APPO hot path (libappo_b200.so).
 *
 * The reference (/root/reference/proj, header-only C++20) has no FFI: its hot
 * path is a set of inline free functions called by PolicyWorkerUnit::run_once
 * (orchestrator.hpp:602-673) and LearnerUnit::step (orchestrator.hpp:760-901).
 * Each entry point below names the reference function(s) it replaces.  A host
 * that used the reference calls these instead (see INTEGRATION.md for the C++
 * shim that restores the reference's exception types and std::span signatures).
 *
 * Conventions
 *   - Every call returns appo_status.  0 ok; 1 ContractError (shape / range /
 *     order, common.hpp:23-26); 2 ConfigError (invalid rho_bar/c_bar/gamma/clip,
 *     common.hpp:30-33); 3 NumericError (non-finite input / gradient / loss,
 *     common.hpp:37-40); 4 resource (CUDA / allocation failure).
 *     appo_last_error() returns the thread's last message.
 *   - Pointers named d_* are caller-owned DEVICE memory; h_* are caller-owned
 *     HOST memory (pinned for the *_host variants' best throughput).  The
 *     library owns only ctx-internal parameters, optimizer state and scratch.
 *   - Work is enqueued on the ctx stream (appo_ctx_set_stream) and is
 *     asynchronous unless stated.  Kernels that find non-finite inputs raise a
 *     sticky device flag; appo_ctx_sync() waits for the stream and returns 3 if
 *     the flag was raised (then clears it), mirroring the reference throwing
 *     NumericError from the same call.
 *   - Layout of per-step arrays is [n_traj x T] row-major, i.e. the learner's
 *     gather order s = i*T + t (orchestrator.hpp:781-795).
 */
#ifndef APPO_CAPI_H
#define APPO_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define APPO_CAPI_VERSION 1

#if defined(__GNUC__)
#define APPO_API __attribute__((visibility("default")))
#else
#define APPO_API
#endif

typedef enum {
  APPO_OK = 0,
  APPO_ERR_CONTRACT = 1,
  APPO_ERR_CONFIG = 2,
  APPO_ERR_NUMERIC = 3,
  APPO_ERR_RESOURCE = 4
} appo_status;

typedef struct appo_ctx appo_ctx;

/* Model contract: convnet_simple over u8 obs [C][H][W] -> GRU(512)
 * -> categorical head (n_actions) + value.  Replaces ModelShape
 * (policy.hpp:39-59), whose MLP trunk the reference uses as a stand-in. */
typedef struct {
  int32_t obs_c, obs_h, obs_w; /* 3, 72, 128 at the Doom shape */
  int32_t n_actions;           /* 6 (ActionHeadsSpec{6}, policy.hpp:25-35) */
  int32_t T;                   /* rollout / recurrence length, 32 */
  int32_t reserved[3];
} appo_model_desc;

/* Learner hyper-parameters: AdamConfig (policy.hpp:88-94), LossConfig
 * (offpolicy.hpp:130-134), VTraceConfig (offpolicy.hpp:18-28), advantage
 * source / normalisation (orchestrator.hpp:47,838-845). */
typedef struct {
  float lr, beta1, beta2, eps, grad_clip;
  float entropy_coef, value_coef, clip_low, clip_high;
  float rho_bar, c_bar, gamma, gae_lambda;
  int32_t adv_source; /* 0 = V-trace pg_adv, 1 = n-step - V, 2 = GAE(lambda) */
  int32_t normalize_adv;
  int32_t reserved;
} appo_hparams;

/* LearnerStepRow (orchestrator.hpp:700-711) loss fields + extras. */
typedef struct {
  double policy_loss, value_loss, entropy, total_loss; /* LossComponents */
  double mean_ratio;                                   /* GradientResult::mean_ratio */
  double grad_norm;                                    /* pre-clip global norm */
  double lag_mean, lag_max;                            /* orchestrator.hpp:862-863 */
  int64_t version;                                     /* version after the step */
} appo_step_out;

APPO_API const char* appo_last_error(void);
APPO_API int appo_capi_version(void);

/* ---- context ----------------------------------------------------------- */
/* desc may be NULL for a context that only runs the stateless kernels. */
APPO_API int appo_ctx_create(const appo_model_desc* desc, int device, uint64_t seed, appo_ctx** out);
APPO_API int appo_ctx_destroy(appo_ctx* ctx);
/* A second context on the same device sharing base's model (parameters,
 * published copies, Adam state) with its own stream and scratch flags: run
 * the sampler / policy inference on it concurrently with the learner on base
 * (the policy-worker / learner split of orchestrator.hpp:938-946).  Inference
 * takes the newest COMPLETED publish (cross-stream events, triple-buffered),
 * so it never reads a half-written version.  base must outlive it. */
APPO_API int appo_ctx_create_shared(appo_ctx* base, appo_ctx** out);
APPO_API int appo_ctx_set_stream(appo_ctx* ctx, void* cuda_stream);
/* Size persistent / grid-stride grids of this context for n_sms SMs (default:
 * all), leaving the rest to a concurrently running context (e.g. the learner). */
APPO_API int appo_ctx_set_sm_budget(appo_ctx* ctx, int n_sms);
/* Programmatic dependent launch for this context's kernels: the next
 * kernel's launch and prologue overlap the current kernel's tail.  Default:
 * on for contexts that own a model (learners), off for shared contexts
 * (samplers running next to a learner); env APPO_PDL=0/1/B/S overrides
 * (none / all / owners only / shared only). */
APPO_API int appo_ctx_set_pdl(appo_ctx* ctx, int enable);
/* Learner backward on two streams: the weight-gradient kernels run on a side
 * stream beside the input-gradient chain (bit-identical results, joined
 * before the optimizer).  Default on; env APPO_LEARNER_FORK=0 turns the
 * default off. */
APPO_API int appo_ctx_set_learner_fork(appo_ctx* ctx, int enable);
APPO_API int appo_ctx_sync(appo_ctx* ctx);
/* Number of launches of this library's kernels enqueued on ctx so far. */
APPO_API int64_t appo_ctx_launch_count(appo_ctx* ctx);
/* Per-launch CUDA-event timing of this library's kernels on the ctx stream
 * (name_filter: only kernels of that name, or of any of several names
 * separated by '|'; NULL = all; a prefix "@N:" brackets only every N-th
 * matching launch, since the events end the programmatic-dependent-launch
 * overlap of the launches they separate).  The report is JSON
 * lines {"name", "launches", "ms", "flops", "bytes"} (algorithmic work per
 * launch as recorded by the launcher); it synchronizes and resets. */
APPO_API int appo_ctx_set_timing(appo_ctx* ctx, int enable, const char* name_filter);
APPO_API int appo_ctx_timing_report(appo_ctx* ctx, char* buf, int buflen);

/* ---- off-policy returns (offpolicy.hpp) --------------------------------- */
/* Replaces vtrace (offpolicy.hpp:61-100) for n_traj trajectories at once.
 * d_rho_out / d_c_out may be NULL.  Validation as VTraceConfig::validate. */
APPO_API int appo_vtrace(appo_ctx* ctx, int n_traj, int T, const float* d_rewards, const float* d_values,
                const float* d_bootstrap, const float* d_target_logp,
                const float* d_behavior_logp, const uint8_t* d_dones, float gamma, float rho_bar,
                float c_bar, float* d_v_out, float* d_pg_adv_out, float* d_rho_out,
                float* d_c_out);
/* Replaces nstep_returns (offpolicy.hpp:104-114). */
APPO_API int appo_nstep_returns(appo_ctx* ctx, int n_traj, int T, const float* d_rewards,
                       const float* d_bootstrap, const uint8_t* d_dones, float gamma,
                       float* d_ret_out);
/* GAE(lambda) (new; lambda = 1 equals nstep_returns - V).  d_ret_out may be NULL. */
APPO_API int appo_gae(appo_ctx* ctx, int n_traj, int T, const float* d_rewards, const float* d_values,
             const float* d_bootstrap, const uint8_t* d_dones, float gamma, float lambda,
             float* d_adv_out, float* d_ret_out);
/* Replaces total_loss (offpolicy.hpp:146-168); h_out4 = {policy, value, entropy,
 * total} in fp64, written after an internal sync (this call is synchronous). */
APPO_API int appo_total_loss(appo_ctx* ctx, int n, const float* d_ratios, const float* d_adv,
                    const float* d_values, const float* d_v_targets, const float* d_entropies,
                    float clip_low, float clip_high, float value_coef, float entropy_coef,
                    double* h_out4);

/* ---- heads (policy.hpp:214-281) ----------------------------------------- */
/* Target log-prob of the stored action and entropy per sample (single head of
 * n_actions), replaces log_prob_and_entropy.  Out-of-range actions are a
 * contract error (device flag, reported by appo_ctx_sync as 1). */
APPO_API int appo_logp_entropy(appo_ctx* ctx, int B, int n_actions, const float* d_logits,
                      const int32_t* d_actions, float* d_logp_out, float* d_entropy_out);
/* sample_action (policy.hpp:232-258) with a counter-based uniform per row:
 * u_b = U(key, counter0 + b).  Writes action and joint log-prob. */
APPO_API int appo_sample_actions(appo_ctx* ctx, int B, int n_actions, const float* d_logits, uint64_t key,
                        uint64_t counter0, int32_t* d_actions, float* d_logp);
/* Factored action spaces (ActionHeadsSpec{sizes}, policy.hpp:25-35): n_heads
 * (1..8) independent categorical heads of h_sizes[j] (1..64) actions; a
 * logits row is the heads concatenated (logits_dim = sum of sizes), actions
 * are [B][n_heads].  log_prob_and_entropy (policy.hpp:262-281): joint logp =
 * sum over heads, entropy = sum of per-head entropies.  sample_action
 * (policy.hpp:232-258): one uniform per (row b, head j), U(key, counter0 +
 * b*n_heads + j), so n_heads = 1 equals the single-head calls above. */
APPO_API int appo_logp_entropy_heads(appo_ctx* ctx, int B, int n_heads, const int32_t* h_sizes,
                                     const float* d_logits, const int32_t* d_actions,
                                     float* d_logp_out, float* d_entropy_out);
APPO_API int appo_sample_actions_heads(appo_ctx* ctx, int B, int n_heads, const int32_t* h_sizes,
                                       const float* d_logits, uint64_t key, uint64_t counter0,
                                       int32_t* d_actions, float* d_logp);

/* ---- optimizer (policy.hpp:431-455) -------------------------------------- */
/* Global-norm clip + Adam over flat fp32 vectors, step t (1-based, after the
 * increment).  Non-finite gradient -> params untouched, status 3 at sync.
 * h_grad_norm (optional) receives the pre-clip norm after an internal sync. */
APPO_API int appo_adam_step(appo_ctx* ctx, int64_t n, float* d_theta, float* d_m, float* d_v,
                   const float* d_grad, int64_t t, float lr, float beta1, float beta2, float eps,
                   float grad_clip, double* h_grad_norm);

/* ---- model-level calls (need a ctx created with a model desc) ------------ */
APPO_API int64_t appo_param_count(const appo_model_desc* desc);
/* Trajectory slot layout v2 (trajstore.hpp:62-87 with u8 obs and f32
 * hidden/reward/logp): 10 offsets {obs, hidden, actions, rewards, logp, dones,
 * versions, boot_obs, boot_hidden, total}. */
APPO_API int appo_slot_layout(const appo_model_desc* desc, uint64_t* out10);

/* ParamStore::fetch/publish (policy.hpp:487-509): copies the learner's fp32
 * parameters (flat contract order) to h_dst / from h_src.  Setting
 * parameters resets Adam moments to zero and bumps the version. */
APPO_API int appo_params_get(appo_ctx* ctx, float* h_dst, int64_t* version_out);
APPO_API int appo_params_set(appo_ctx* ctx, const float* h_src, int64_t version);
APPO_API int appo_adam_get(appo_ctx* ctx, float* h_m, float* h_v, int64_t* t_out);
APPO_API int appo_adam_set(appo_ctx* ctx, const float* h_m, const float* h_v, int64_t t);
APPO_API int64_t appo_params_version(appo_ctx* ctx);

/* Checkpoint / resume in the reference's APPOCKP1 format: replaces
 * save_checkpoint / load_checkpoint (policy.hpp:545-605; byte layout
 * docs/shared_memory_layout.md:95-107).  load: ConfigError on a spec-hash or
 * parameter-count mismatch, resource error on I/O / checksum failures; the
 * published copy, Adam moments, step counter and version are all restored. */
APPO_API int appo_checkpoint_save(appo_ctx* ctx, const char* path);
APPO_API int appo_checkpoint_load(appo_ctx* ctx, const char* path);
/* Any APPOCKP1 file (also the reference's own): header, and theta|m|v as f64
 * when tmv != NULL (*n_inout = capacity in, n out); magic + checksum checked. */
APPO_API int appo_checkpoint_read_raw(const char* path, uint64_t* spec_hash, int64_t* version,
                                      int64_t* adam_t, uint64_t* n_inout, double* tmv);
/* ModelShape::spec_hash analogue (policy.hpp:54-58) of this model contract. */
APPO_API uint64_t appo_model_spec_hash(const appo_model_desc* desc);
/* fnv1a64 (common.hpp:66-74). */
APPO_API uint64_t appo_fnv1a64(const void* data, uint64_t n);

/* Batched policy inference: replaces forward_batch + sample_action + the row
 * writes of PolicyWorkerUnit::run_once (orchestrator.hpp:643-656).
 * d_obs u8 [B][C*H*W], d_h_in f32 [B][512] -> d_actions i32 [B], d_logp f32 [B],
 * d_h_out f32 [B][512], d_values f32 [B], d_logits (optional) f32 [B][A].
 * Sampling uses u = U(ctx key, rng_counter0 + b).  *h_version_out (optional)
 * receives the parameter version used (ExchangeLayout version field). */
APPO_API int appo_policy_forward(appo_ctx* ctx, int B, const uint8_t* d_obs, const float* d_h_in,
                        uint64_t rng_counter0, int32_t* d_actions, float* d_logp,
                        float* d_h_out, float* d_values, float* d_logits,
                        int64_t* h_version_out);

/* Learner step over n_traj trajectory slots of layout v2 living in one device
 * slot region: replaces assemble_minibatch's gather + LearnerUnit::step
 * (orchestrator.hpp:770-868): forward (encoder + GRU unrolled from the stored
 * h0 with resets after done) + bootstrap forward, target logp/entropy, V-trace
 * (or n-step / GAE), advantage normalisation, PPO + value + entropy loss,
 * BPTT, encoder backward, global-norm clip + Adam, version += 1, publish of the
 * bf16 inference copy.  h_slot_ids are in FIFO arrival order (index i of the
 * minibatch = trajectory i).  Synchronous: fills *out. */
APPO_API int appo_learner_step(appo_ctx* ctx, const void* d_slot_region, uint64_t slot_bytes,
                      const int32_t* h_slot_ids, int n_traj, const appo_hparams* hp,
                      appo_step_out* out);

/* Asynchronous form of appo_learner_step: _submit validates the arguments and
 * enqueues the whole step (including Adam and the publish of the inference
 * copy) on the ctx stream without waiting; _collect waits for everything
 * submitted, returns the statistics of the last submitted step and the first
 * device-detected error (a rejected step leaves the parameters untouched and
 * does not advance the version, as when optimizer_step throws). */
APPO_API int appo_learner_submit(appo_ctx* ctx, const void* d_slot_region, uint64_t slot_bytes,
                                 const int32_t* h_slot_ids, int n_traj, const appo_hparams* hp);
APPO_API int appo_learner_collect(appo_ctx* ctx, appo_step_out* out);

/* ---- data-parallel learner (NCCL over NVLink) ----------------------------- */
/* One policy on nranks GPUs: rank 0 creates the id, the host broadcasts it
 * (e.g. torch.distributed), every rank calls appo_dp_init on its ctx.  From
 * then on appo_learner_step averages the flat gradient with ncclAllReduce
 * before the global-norm clip and Adam (no reference counterpart: the
 * reference runs one learner thread per policy, orchestrator.hpp:938-946):
 * three buckets in reverse layer order on a side stream, each launched as
 * soon as the backward pass finished it (overlapping the rest of the
 * backward), the last one grouped with a max-reduction of the ranks' step
 * rejection flags so a step any rank rejects is rejected on every rank.
 * nranks = 1 is allowed (the same path over a one-rank communicator). */
APPO_API int appo_dp_unique_id(char* out128);
APPO_API int appo_dp_init(appo_ctx* ctx, int nranks, int rank, const char* id128);
/* The gradient buckets in reduction order as (offset, count) pairs over the
 * flat parameter vector (host-only; *n_out = 3). */
APPO_API int appo_dp_bucket_plan(const appo_model_desc* desc, int64_t* out_pairs, int cap,
                                 int* n_out);

/* ---- device sampler: synthetic envs + rollout-side writer ---------------- */
/* Restates SyntheticLatencyEnv (envs.hpp:103-158) on the device with u8 pixels
 * and RolloutWorker::step_group/submit_group (orchestrator.hpp:435-552): every
 * appo_sampler_step advances all n_envs envs by one step, writing step t of
 * env e's rollout into slot slot_base + e of a layout-v2 slot region
 * (obs, input hidden, action, behaviour logp, version, reward, done; at
 * t == T-1 also the bootstrap obs/hidden and the in-slot header), running the
 * batched policy on the obs in place.  h_obs != NULL: observations come from
 * (pinned) host memory [n_envs][obs_dim] instead of the device generator (CPU
 * actors); h_actions != NULL: sampled actions are copied back (exchange-row
 * reply, orchestrator.hpp:652).  Asynchronous on the ctx stream. */
typedef struct appo_sampler appo_sampler;
APPO_API int appo_sampler_create(appo_ctx* ctx, int n_envs, int episode_len, uint64_t env_seed,
                                 appo_sampler** out);
APPO_API int appo_sampler_destroy(appo_sampler* s);
APPO_API int appo_sampler_step(appo_sampler* s, void* d_region, uint64_t slot_bytes,
                               int32_t slot_base, int t, const uint8_t* h_obs,
                               int32_t* h_actions);

/* CPU actors (the paper's setting): RolloutWorker::submit_group + step_group
 * (orchestrator.hpp:435-552) in two calls per env step t of the rollout into
 * slots [slot_base, slot_base + n_envs), strictly in the order act(0),
 * feedback(0), act(1), ... feedback(T-1) (write_step's ordering contract,
 * trajstore.hpp:172-174: anything else is a contract error).
 *   act: h_obs [n_envs][obs_dim] (pinned host memory for an asynchronous
 *     copy; it must stay unchanged until appo_rollout_wait returns) becomes
 *     slot row t's obs; batched inference on it with the sampler's per-env
 *     hidden state writes row t's input hidden, action, behaviour logp and
 *     policy version (the exchange-row reply, :512-521); the actions are
 *     copied to h_actions (optional), valid once appo_rollout_wait returns.
 *   feedback: the env transition's h_rewards f32 [n_envs] and h_dones u8
 *     [n_envs] (copied before the call returns) become row t's reward / done;
 *     hidden <- h' (zero after done, reset_env :402); at t == T-1 h_next_obs
 *     [n_envs][obs_dim] is REQUIRED -- the bootstrap obs (set_bootstrap,
 *     :529-534; valid until the next appo_rollout_wait) with bootstrap hidden
 *     h', the header is sealed and the slots go to the ready queue (if set).
 * Asynchronous on the ctx stream. */
APPO_API int appo_rollout_act(appo_sampler* s, void* d_region, uint64_t slot_bytes,
                              int32_t slot_base, int t, const uint8_t* h_obs, int32_t* h_actions);
APPO_API int appo_rollout_wait(appo_sampler* s);
APPO_API int appo_rollout_feedback(appo_sampler* s, void* d_region, uint64_t slot_bytes,
                                   int32_t slot_base, int t, const float* h_rewards,
                                   const uint8_t* h_dones, const uint8_t* h_next_obs);

/* ---- device slot queues: ready queue + free list ------------------------- */
/* Replaces the host BoundedFifo ready_q drained by assemble_minibatch
 * (trajstore.hpp:293-331; fed by RolloutWorker::submit_group,
 * orchestrator.hpp:535-552) and the slot release after the learner step
 * (orchestrator.hpp:870) with device-resident FIFOs of slot ids in
 * [0, n_slots).  Pushes (any stream, any number of producers) keep the ids of
 * one push contiguous and in order; pops (one consumer per queue) wait on the
 * device until the whole request is published, up to timeout_s, and on timeout
 * consume nothing and raise APPO_ERR_RESOURCE at the next sync/collect.
 * capacity is rounded up to a power of two >= n_slots; at most capacity ids
 * may be queued at once (each slot in at most one queue never overflows it).
 * Kernels a consumer waits for must already be loaded (CUDA lazy loading):
 * appo_slotq_create loads every kernel of this library. */
typedef struct appo_slotq appo_slotq;
APPO_API int appo_slotq_create(int device, int32_t n_slots, int32_t capacity, double timeout_s,
                               appo_slotq** out);
APPO_API int appo_slotq_destroy(appo_slotq* q);
/* enqueue n device-resident ids / the range [first_id, first_id + n) on ctx's stream */
APPO_API int appo_slotq_push(appo_ctx* ctx, appo_slotq* q, const int32_t* d_ids, int n);
APPO_API int appo_slotq_push_range(appo_ctx* ctx, appo_slotq* q, int32_t first_id, int n);
/* dequeue n ids (FIFO) into device memory d_out on ctx's stream */
APPO_API int appo_slotq_pop(appo_ctx* ctx, appo_slotq* q, int32_t* d_out, int n);
/* counters (synchronous read; call after syncing the streams that use q) */
APPO_API int appo_slotq_stats(appo_slotq* q, int64_t* pushed, int64_t* popped, int64_t* timeouts);

/* appo_learner_submit whose minibatch is the next n_traj slots of ready_q
 * (assemble_minibatch: strict FIFO, lag statistics from the slots' versions);
 * after the step the slots are pushed to free_q (may be NULL).  The host never
 * sees the slot ids. */
APPO_API int appo_learner_submit_queued(appo_ctx* ctx, const void* d_slot_region,
                                        uint64_t slot_bytes, appo_slotq* ready_q,
                                        appo_slotq* free_q, int n_traj, const appo_hparams* hp);

/* The sampler pushes slots [slot_base, slot_base + n_envs) to q after writing
 * step T-1 of a rollout (submit_group).  q = NULL detaches. */
APPO_API int appo_sampler_set_ready_queue(appo_sampler* s, appo_slotq* q);

/* ---- population-based training over per-GPU learners --------------------- */
/* pbt_step (population.hpp:131-186) and PbtController (runner.hpp:169-252):
 * per-policy score windows (ScoreWindow, population.hpp:72-98), PBT steps on
 * pbt_period frame boundaries, mutation of the bottom cohort, weight +
 * hyper-parameter exchange into the worst cohort through copy_weights.  The
 * decision stream is the reference's std::mt19937_64 stream: seeded alike, it
 * reproduces the reference's decision log byte for byte. */
#define APPO_PBT_MAX_REWARD_WEIGHTS 8
typedef struct {
  int64_t pbt_period;           /* frames between PBT steps (<= 0: never)    */
  double mutate_fraction;       /* 0.70 */
  double mutation_rate;         /* 0.15, per hyper-parameter                 */
  double mutation_factor;       /* 1.2 */
  double replace_fraction;      /* 0.30 */
  double exchange_threshold;    /* win-rate gap gate (0.35 in duel mode)     */
  int32_t has_exchange_threshold;
  int32_t window;               /* ScoreWindow capacity, 100                 */
} appo_pbt_config;
typedef struct {                /* AgentMeta (population.hpp:41-58) */
  uint32_t policy_id;
  int32_t n_reward_weights;
  double learning_rate, entropy_coef, adam_beta1;
  double reward_weights[APPO_PBT_MAX_REWARD_WEIGHTS];
} appo_agent_meta;
typedef struct {                /* PbtEvent (population.hpp:100-107) */
  int64_t frame;
  uint32_t agent;
  int32_t event;                /* 0 mutate, 1 exchange, 2 skip-threshold    */
  char field[32];
  double old_value, new_value;
} appo_pbt_event;
/* copy_weights(dst, src): dst learner takes src's theta + Adam state */
typedef int (*appo_pbt_copy_fn)(void* user, uint32_t dst, uint32_t src);
typedef struct appo_pbt appo_pbt;

/* init may be NULL (lr 1e-4, entropy 0.003, beta1 0.9, no reward weights);
 * policy ids are 0..P-1.  rng_seed seeds the decision stream directly; the
 * reference controller uses appo_pbt_controller_seed(pipeline seed). */
APPO_API int appo_pbt_create(const appo_pbt_config* cfg, int P, uint64_t rng_seed,
                             const appo_agent_meta* init, appo_pbt** out);
APPO_API int appo_pbt_destroy(appo_pbt* pbt);
APPO_API uint64_t appo_pbt_controller_seed(uint64_t pipeline_seed);
/* an episode result of policy: return, or 1/0 for win/(tie, loss) */
APPO_API int appo_pbt_record(appo_pbt* pbt, uint32_t policy, double value);
APPO_API int appo_pbt_score(appo_pbt* pbt, uint32_t policy, double* score, int* has_score);
/* one PBT step on explicit scores (has_score[i] == 0: exempt) */
APPO_API int appo_pbt_step(appo_pbt* pbt, const double* scores, const uint8_t* has_score,
                           int64_t frame, appo_pbt_copy_fn copy_weights, void* user,
                           appo_pbt_event* events, int max_events, int* n_events);
/* PbtController::tick: a step on the window scores once frames reach the next
 * period boundary (*fired = 1), else nothing */
APPO_API int appo_pbt_tick(appo_pbt* pbt, int64_t frames, appo_pbt_copy_fn copy_weights,
                           void* user, appo_pbt_event* events, int max_events, int* n_events,
                           int* fired);
APPO_API int appo_pbt_get_agent(appo_pbt* pbt, int i, appo_agent_meta* out);
APPO_API int appo_pbt_max_events(appo_pbt* pbt);
/* CSV text of append_pbt_events_csv (population.hpp:110-118) */
APPO_API int appo_pbt_format_events(const appo_pbt_event* events, int n, int header, char* buf,
                                    uint64_t cap, uint64_t* len);
/* dst takes src's parameters and Adam state (device to device, peer copy
 * across GPUs) and publishes them as its next version (PbtController's
 * copy_weights, runner.hpp:211-219); dst must have no uncollected steps */
APPO_API int appo_params_copy(appo_ctx* dst, appo_ctx* src);
/* copy_weights over user = appo_ctx*[P] (learner of policy i at index i);
 * dst == src is a no-op (the reference's self-copy) */
APPO_API int appo_pbt_copy_contexts(void* user, uint32_t dst, uint32_t src);

/* copy_weights between PROCESSES (one learner per process / GPU, configs[4]):
 * the source exports its state -- CUDA IPC handles of theta, m, v plus Adam t
 * and version, APPO_STATE_HANDLE_BYTES of plain bytes the host ships to the
 * destination (e.g. torch.distributed) -- and the destination imports it:
 * a device-to-device copy (NVLink peer copy across GPUs, the copy engines of
 * one GPU otherwise) published as its next version, as appo_params_copy.
 * Export waits for the source's queued work; the source must not run another
 * learner step until the import returned (runner.hpp:217-218 holds both
 * learners' pbt_lock for the copy).  Import from this same process is a
 * contract error (use appo_params_copy). */
#define APPO_STATE_HANDLE_BYTES 512
APPO_API int appo_params_export(appo_ctx* ctx, void* handle_out);
APPO_API int appo_params_import(appo_ctx* dst, const void* handle);

#ifdef __cplusplus
}
#endif
#endif /* APPO_CAPI_H */
