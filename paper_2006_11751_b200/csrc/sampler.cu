// Device-resident sampler: n_envs synthetic environments + the rollout-side
// writer, one call per environment step for all envs.
//
//   * synthetic env: restates SyntheticLatencyEnv (envs.hpp:103-158) for u8
//     pixels -- obs bytes from the keyed hash of make_obs (envs.hpp:143-151),
//     one splitmix64 per 8 pixels; reward schedule envs.hpp:127; done at
//     episode_len (envs.hpp:128); env seed derive_seed(seed, (env<<24)^episode)
//     as RolloutWorker::reset_env (orchestrator.hpp:403-404).
//   * rollout writer: RolloutWorker::step_group / submit_group
//     (orchestrator.hpp:435-552): the obs is written straight into the env's
//     trajectory slot (layout v2) and the policy reads it there; the step
//     record stores the INPUT hidden (orchestrator.hpp:518), behaviour logp and
//     policy version (ExchangeLayout fields, :652-656); hidden <- h' and reset
//     to zero after done (:402,528,545-547); at t == T-1 the bootstrap obs /
//     hidden and the in-slot header are written (set_bootstrap + seal,
//     trajstore.hpp:208-215,265-280).
// Host-staged variant: obs arrive from pinned host memory (CPU actors) and the
// sampled actions are copied back, i.e. the exchange-row round trip.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>

#include "gemm.cuh"
#include "model.cuh"
#include "model_kernels.cuh"
#include "slotq.cuh"

namespace appo_b200 {
int sampler_infer(Ctx* c, const uint8_t* obs_base, int64_t obs_stride, int B, const float* h_in,
                  uint64_t counter0, int32_t* actions, float* logp, float* h_out, float* values,
                  float* logits, int64_t* version_out);
}

using namespace appo_b200;

struct appo_sampler {
  appo_ctx* ctx = nullptr;
  int n_envs = 0;
  int episode_len = 0;
  uint64_t seed = 0;
  uint32_t* step = nullptr;     // [n_envs] step within episode
  uint32_t* episode = nullptr;  // [n_envs]
  float* hidden = nullptr;      // [n_envs][512]
  float* h_out = nullptr;
  int32_t* actions = nullptr;
  float* logp = nullptr;
  float* values = nullptr;
  uint64_t steps_done = 0;
  appo_slotq* ready_q = nullptr;  // sealed slots are pushed here at t == T-1
  // host observations (CPU actors): contiguous pinned -> device copies on the
  // context's copy stream into two staging buffers, so step t+1's transfer
  // overlaps step t's inference; a scatter kernel on the ctx stream moves them
  // into the slots (region writes stay ordered on the ctx stream)
  uint8_t* staging[2] = {nullptr, nullptr};
  cudaEvent_t copied[2] = {nullptr, nullptr};
  cudaEvent_t consumed[2] = {nullptr, nullptr};
  int stage_next = 0;
  // CPU-actor rollout (appo_rollout_act / _feedback): per-step rewards and
  // dones staged through a pinned double buffer (the caller's arrays are free
  // to reuse when the call returns), the next expected (t, phase) as
  // write_step's ordering contract, and the event the host waits on for the
  // actions / the end of the caller-buffer reads
  uint8_t* fb_host = nullptr;     // pinned [2][n_envs * 5]
  uint8_t* fb_dev = nullptr;      // [2][n_envs * 5]: rewards f32 then dones u8
  cudaEvent_t fb_ev[2] = {nullptr, nullptr};
  int fb_next = 0;
  cudaEvent_t host_ev = nullptr;  // after the last D2H of actions / read of caller obs
  int next_t = 0;
  bool acted = false;             // act(t) done, feedback(t) pending
};

namespace {

__device__ __forceinline__ uint64_t dev_derive_seed(uint64_t seed, uint64_t stream) {
  return splitmix64(seed ^ splitmix64(stream + 1));
}

constexpr int kObsWordsPerThread = 8;

// obs for env e at its current (episode, step): 8 pixels per hash.
// grid (ceil(words / 256), n_envs): env from blockIdx.y, no 64-bit division
__global__ void gen_obs_kernel(int n_envs, int64_t obs_dim, uint64_t seed,
                               const uint32_t* __restrict__ step,
                               const uint32_t* __restrict__ episode, uint8_t* region,
                               uint64_t slot_bytes, int64_t slot_base, uint64_t off) {
  APPO_PDL_ENTRY();
  const int words = (int)(obs_dim >> 3);
  const int e = blockIdx.y;
  const int w0 = blockIdx.x * (kObsWordsPerThread * 256) + threadIdx.x;
  if (w0 >= words) return;
  // the env's episode seed once per thread, then kObsWordsPerThread hashes
  // (coalesced: word w0 + 256 k)
  const uint64_t es = dev_derive_seed(seed, ((uint64_t)e << 24) ^ episode[e]);
  const uint64_t key = es ^ ((uint64_t)step[e] << 20);
  uint64_t* dst = reinterpret_cast<uint64_t*>(region + (uint64_t)(slot_base + e) * slot_bytes + off);
#pragma unroll
  for (int k = 0; k < kObsWordsPerThread; ++k) {
    const int w = w0 + 256 * k;
    if (w < words) dst[w] = splitmix64(key ^ (uint64_t)w);
  }
}

// Staged host observations [n_envs][obs_dim] -> slot rows (16-byte vectors).
__global__ void scatter_obs_kernel(int n_envs, int64_t obs_dim, const uint4* __restrict__ src,
                                   uint8_t* region, uint64_t slot_bytes, int64_t slot_base,
                                   uint64_t off) {
  APPO_PDL_ENTRY();
  const int64_t v = obs_dim >> 4;
  const int e = blockIdx.y;
  uint4* dst = reinterpret_cast<uint4*>(region + (uint64_t)(slot_base + e) * slot_bytes + off);
  const uint4* srow = src + (int64_t)e * v;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < v;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __ldg(srow + i);
}

// Step record + env transition; one block (128 threads) per env.
__global__ void record_kernel(int n_envs, int T, int t, int episode_len, uint32_t obs_dim,
                              uint64_t seed,
                              int64_t version, uint32_t* __restrict__ step,
                              uint32_t* __restrict__ episode, float* __restrict__ hidden,
                              const float* __restrict__ h_out, const int32_t* __restrict__ act,
                              const float* __restrict__ logp, uint8_t* region,
                              uint64_t slot_bytes, int64_t slot_base, SlotOffsets off) {
  APPO_PDL_ENTRY();
  const int e = blockIdx.x;
  if (e >= n_envs) return;
  uint8_t* slot = region + (uint64_t)(slot_base + e) * slot_bytes;
  const uint32_t st = step[e];
  const uint32_t ep = episode[e];
  const bool done = (st + 1) >= (uint32_t)episode_len;
  // slot arrays are only guaranteed 8-byte aligned (align8 layout): float2 stores
  float2* hs = reinterpret_cast<float2*>(hidden + (int64_t)e * kHidden);
  const float2* ho = reinterpret_cast<const float2*>(h_out + (int64_t)e * kHidden);
  float2* dst = reinterpret_cast<float2*>(slot + off.hidden + (uint64_t)t * kHidden * 4);
  float2* boot = reinterpret_cast<float2*>(slot + off.boot_hidden);
  for (int j = threadIdx.x; j < kHidden / 2; j += blockDim.x) {
    dst[j] = hs[j];  // stored hidden = the step's INPUT hidden
    const float2 n = ho[j];
    if (t == T - 1) boot[j] = n;  // bootstrap hidden = h' (before any reset)
    hs[j] = done ? make_float2(0.f, 0.f) : n;
  }
  if (threadIdx.x == 0) {
    const uint64_t es = dev_derive_seed(seed, ((uint64_t)e << 24) ^ ep);
    reinterpret_cast<int32_t*>(slot + off.actions)[t] = act[e];
    reinterpret_cast<float*>(slot + off.logp)[t] = logp[e];
    reinterpret_cast<float*>(slot + off.rewards)[t] =
        0.1f * (float)((st + 1 + es % 7) % 11) - 0.5f;
    slot[off.dones + t] = done ? 1 : 0;
    reinterpret_cast<int64_t*>(slot + off.versions)[t] = version;
    if (done) {
      step[e] = 0;
      episode[e] = ep + 1;
    } else {
      step[e] = st + 1;
    }
    if (t == T - 1 || t == 0) {
      uint32_t* h = reinterpret_cast<uint32_t*>(slot);
      h[0] = T;
      h[1] = obs_dim;
      h[2] = kHidden;
      h[3] = 1;
      h[4] = t + 1;
      h[5] = e;
      h[6] = 0;
      h[7] = 0;
      h[8] = 0;
      h[9] = (t == T - 1) ? 1u : 0u;  // bit0: bootstrap written
    }
  }
}

// CPU-actor step records (RolloutWorker::step_group, orchestrator.hpp:486-552);
// one block (128 threads) per env.
//   act phase (feedback == nullptr): the step's INPUT hidden, action, behaviour
//     logp and policy version into row t (StepRecord fields, :512-521);
//   feedback phase: the env transition's reward and done into row t, hidden <-
//     h' or 0 after done (:524, reset_env :402); at t == T-1 the bootstrap
//     hidden h' (set_bootstrap before the reset, :531-534); the in-slot header.
__global__ void host_record_kernel(int n_envs, int T, int t, uint32_t obs_dim, int64_t version,
                                   float* __restrict__ hidden, const float* __restrict__ h_out,
                                   const int32_t* __restrict__ act,
                                   const float* __restrict__ logp,
                                   const uint8_t* __restrict__ feedback, uint8_t* region,
                                   uint64_t slot_bytes, int64_t slot_base, SlotOffsets off) {
  APPO_PDL_ENTRY();
  const int e = blockIdx.x;
  if (e >= n_envs) return;
  uint8_t* slot = region + (uint64_t)(slot_base + e) * slot_bytes;
  float2* hs = reinterpret_cast<float2*>(hidden + (int64_t)e * kHidden);
  if (feedback == nullptr) {
    float2* dst = reinterpret_cast<float2*>(slot + off.hidden + (uint64_t)t * kHidden * 4);
    for (int j = threadIdx.x; j < kHidden / 2; j += blockDim.x) dst[j] = hs[j];
    if (threadIdx.x == 0) {
      reinterpret_cast<int32_t*>(slot + off.actions)[t] = act[e];
      reinterpret_cast<float*>(slot + off.logp)[t] = logp[e];
      reinterpret_cast<int64_t*>(slot + off.versions)[t] = version;
    }
    return;
  }
  const float reward = reinterpret_cast<const float*>(feedback)[e];
  const bool done = feedback[(size_t)n_envs * 4 + e] != 0;
  const float2* ho = reinterpret_cast<const float2*>(h_out + (int64_t)e * kHidden);
  float2* boot = reinterpret_cast<float2*>(slot + off.boot_hidden);
  for (int j = threadIdx.x; j < kHidden / 2; j += blockDim.x) {
    const float2 n = ho[j];
    if (t == T - 1) boot[j] = n;
    hs[j] = done ? make_float2(0.f, 0.f) : n;
  }
  if (threadIdx.x == 0) {
    reinterpret_cast<float*>(slot + off.rewards)[t] = reward;
    slot[off.dones + t] = done ? 1 : 0;
    if (t == T - 1 || t == 0) {
      uint32_t* h = reinterpret_cast<uint32_t*>(slot);
      h[0] = T;
      h[1] = obs_dim;
      h[2] = kHidden;
      h[3] = 1;
      h[4] = t + 1;
      h[5] = e;
      h[6] = 0;
      h[7] = 0;
      h[8] = 0;
      h[9] = (t == T - 1) ? 1u : 0u;  // bit0: bootstrap written
    }
  }
}

__global__ void init_env_kernel(int n_envs, int episode_len, uint32_t* step, uint32_t* episode) {
  APPO_PDL_ENTRY();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_envs) return;
  // desynchronise episodes so dones are spread over the batch
  step[e] = (uint32_t)(((uint64_t)e * 2654435761ull) % (uint64_t)episode_len);
  episode[e] = 0;
}

}  // namespace

// module anchor for preload_library_kernels (slotq.cu)
namespace appo_b200 {
const void* kanchor_sampler() { return reinterpret_cast<const void*>(&init_env_kernel); }
}  // namespace appo_b200

namespace {
// Host observations [n_envs][obs_dim] into field offset `off` of slots
// [slot_base, slot_base + n_envs): a contiguous pinned -> device copy on the
// sampler's copy stream into one of two staging buffers (so the next copy
// overlaps this step's inference), then a scatter kernel on the ctx stream;
// when the rows are not 16-byte aligned, one strided 2-D copy on the ctx
// stream instead.
int stage_host_obs(appo_sampler* s, const uint8_t* h_obs, uint8_t* region, uint64_t slot_bytes,
                   int32_t slot_base, uint64_t off) {
  appo_ctx* c = s->ctx;
  const Dims& d = c->model->d;
  const bool staged = d.obs_dim % 16 == 0 && slot_bytes % 16 == 0 &&
                      ((reinterpret_cast<uintptr_t>(region) + off) & 15) == 0;
  if (!staged) {
    APPO_CUDA_TRY(cudaMemcpy2DAsync(region + (uint64_t)slot_base * slot_bytes + off, slot_bytes,
                                    h_obs, d.obs_dim, d.obs_dim, s->n_envs,
                                    cudaMemcpyHostToDevice, c->stream));
    return APPO_OK;
  }
  const size_t bytes = (size_t)s->n_envs * d.obs_dim;
  if (!c->copy_stream)
    APPO_CUDA_TRY(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  if (!s->staging[0]) {
    for (int k = 0; k < 2; ++k) {
      APPO_CUDA_TRY(cudaMalloc(&s->staging[k], bytes));
      APPO_CUDA_TRY(cudaEventCreateWithFlags(&s->copied[k], cudaEventDisableTiming));
      APPO_CUDA_TRY(cudaEventCreateWithFlags(&s->consumed[k], cudaEventDisableTiming));
      APPO_CUDA_TRY(cudaEventRecord(s->consumed[k], c->stream));
    }
  }
  const int k = s->stage_next;
  s->stage_next ^= 1;
  // the buffer's previous contents were scattered (ctx stream) before it is refilled
  APPO_CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, s->consumed[k], 0));
  APPO_CUDA_TRY(cudaMemcpyAsync(s->staging[k], h_obs, bytes, cudaMemcpyHostToDevice,
                                c->copy_stream));
  APPO_CUDA_TRY(cudaEventRecord(s->copied[k], c->copy_stream));
  APPO_CUDA_TRY(cudaStreamWaitEvent(c->stream, s->copied[k], 0));
  const dim3 grid((unsigned)std::min<int64_t>(((d.obs_dim >> 4) + 255) / 256, 8),
                  (unsigned)s->n_envs);
  c->next_bytes = 2.0 * (double)bytes;
  APPO_LAUNCH(c, scatter_obs_kernel, grid, 256, 0, s->n_envs, d.obs_dim,
              reinterpret_cast<const uint4*>(s->staging[k]), region, slot_bytes,
              (int64_t)slot_base, off);
  APPO_CUDA_TRY(cudaEventRecord(s->consumed[k], c->stream));
  return APPO_OK;
}
}  // namespace

#define SMP_OR_RETURN(s)                                                            \
  do {                                                                              \
    APPO_REQUIRE((s) != nullptr && (s)->ctx != nullptr, APPO_ERR_CONTRACT,          \
                 "null sampler");                                                   \
    APPO_CUDA_TRY(cudaSetDevice((s)->ctx->device));                                 \
  } while (0)

extern "C" {

APPO_API int appo_sampler_create(appo_ctx* ctx, int n_envs, int episode_len, uint64_t env_seed,
                                 appo_sampler** out) {
  APPO_REQUIRE(ctx && ctx->model && out, APPO_ERR_CONTRACT,
               "sampler_create: needs a model context");
  APPO_REQUIRE(n_envs >= 1 && n_envs <= 65535 && episode_len >= 1, APPO_ERR_CONTRACT,
               "sampler_create: 1 <= n_envs <= 65535 and episode_len >= 1 required");
  APPO_REQUIRE(ctx->model->d.obs_dim % 8 == 0, APPO_ERR_CONTRACT, "obs_dim must be a multiple of 8");
  APPO_CUDA_TRY(cudaSetDevice(ctx->device));
  appo_sampler* s = new appo_sampler();
  s->ctx = ctx;
  s->n_envs = n_envs;
  s->episode_len = episode_len;
  s->seed = env_seed;
  const size_t H = (size_t)n_envs * kHidden * 4;
  if (cudaMalloc(&s->step, n_envs * 4) != cudaSuccess ||
      cudaMalloc(&s->episode, n_envs * 4) != cudaSuccess ||
      cudaMalloc(&s->hidden, H) != cudaSuccess || cudaMalloc(&s->h_out, H) != cudaSuccess ||
      cudaMalloc(&s->actions, n_envs * 4) != cudaSuccess ||
      cudaMalloc(&s->logp, n_envs * 4) != cudaSuccess ||
      cudaMalloc(&s->values, n_envs * 4) != cudaSuccess) {
    set_error("sampler_create: allocation failed");
    delete s;
    return APPO_ERR_RESOURCE;
  }
  cudaMemsetAsync(s->hidden, 0, H, ctx->stream);
  APPO_LAUNCH(ctx, init_env_kernel, (n_envs + 255) / 256, 256, 0, n_envs, episode_len, s->step,
              s->episode);
  *out = s;
  return APPO_OK;
}

APPO_API int appo_sampler_destroy(appo_sampler* s) {
  if (!s) return APPO_OK;
  cudaSetDevice(s->ctx->device);
  cudaStreamSynchronize(s->ctx->stream);
  cudaFree(s->step);
  cudaFree(s->episode);
  cudaFree(s->hidden);
  cudaFree(s->h_out);
  cudaFree(s->actions);
  cudaFree(s->logp);
  cudaFree(s->values);
  for (int k = 0; k < 2; ++k) {
    if (s->staging[k]) cudaFree(s->staging[k]);
    if (s->copied[k]) cudaEventDestroy(s->copied[k]);
    if (s->consumed[k]) cudaEventDestroy(s->consumed[k]);
  }
  if (s->ctx->copy_stream) cudaStreamSynchronize(s->ctx->copy_stream);
  if (s->fb_host) cudaFreeHost(s->fb_host);
  if (s->fb_dev) cudaFree(s->fb_dev);
  for (int k = 0; k < 2; ++k)
    if (s->fb_ev[k]) cudaEventDestroy(s->fb_ev[k]);
  if (s->host_ev) cudaEventDestroy(s->host_ev);
  delete s;
  return APPO_OK;
}

// One environment step for all envs into slots [slot_base, slot_base + n_envs),
// step index t of the rollout.  h_obs == NULL: on-GPU generator; otherwise obs
// [n_envs][obs_dim] are copied from (pinned) host memory.  h_actions (optional)
// receives the sampled actions (device -> host, the exchange-row reply).
APPO_API int appo_sampler_step(appo_sampler* s, void* d_region, uint64_t slot_bytes,
                               int32_t slot_base, int t, const uint8_t* h_obs,
                               int32_t* h_actions) {
  SMP_OR_RETURN(s);
  appo_ctx* c = s->ctx;
  Model* M = c->model;
  const Dims& d = M->d;
  APPO_REQUIRE(t >= 0 && t < d.T, APPO_ERR_CONTRACT, "sampler_step: t outside [0, T)");
  APPO_REQUIRE(slot_bytes >= d.slot[9] && d_region, APPO_ERR_CONTRACT,
               "sampler_step: bad slot region");
  uint8_t* region = static_cast<uint8_t*>(d_region);
  const uint64_t obs_off = d.slot[0] + (uint64_t)t * d.obs_dim;
  if (h_obs) {
    const int st = stage_host_obs(s, h_obs, region, slot_bytes, slot_base, obs_off);
    if (st) return st;
  } else {
    const dim3 grid((unsigned)(((d.obs_dim >> 3) + 256 * kObsWordsPerThread - 1) /
                             (256 * kObsWordsPerThread)),
                  (unsigned)s->n_envs);
    c->next_bytes = (double)s->n_envs * d.obs_dim;
    APPO_LAUNCH(c, gen_obs_kernel, grid, 256, 0, s->n_envs, d.obs_dim, s->seed, s->step,
                s->episode, region, slot_bytes, (int64_t)slot_base, obs_off);
  }
  int64_t version = 0;  // version of the parameters this inference used (ExchangeLayout field)
  int st = sampler_infer(c, region + (uint64_t)slot_base * slot_bytes + obs_off, slot_bytes,
                         s->n_envs, s->hidden, s->steps_done * (uint64_t)s->n_envs, s->actions,
                         s->logp, s->h_out, s->values, nullptr, &version);
  if (st) return st;
  SlotOffsets off;
  std::memcpy(&off, d.slot, sizeof(off));
  APPO_LAUNCH(c, record_kernel, s->n_envs, 128, 0, s->n_envs, d.T, t, s->episode_len,
              (uint32_t)d.obs_dim, s->seed,
              version, s->step, s->episode, s->hidden, s->h_out, s->actions, s->logp, region,
              slot_bytes, (int64_t)slot_base, off);
  if (t == d.T - 1) {
    // bootstrap obs = next observation of every env (post-transition state)
    const dim3 grid((unsigned)(((d.obs_dim >> 3) + 256 * kObsWordsPerThread - 1) /
                             (256 * kObsWordsPerThread)),
                  (unsigned)s->n_envs);
    APPO_LAUNCH(c, gen_obs_kernel, grid, 256, 0, s->n_envs, d.obs_dim, s->seed, s->step,
                s->episode, region, slot_bytes, (int64_t)slot_base, d.slot[7]);
  }
  if (t == d.T - 1 && s->ready_q) {
    // submit_group: the sealed trajectories enter the ready queue in env order
    APPO_REQUIRE((int64_t)slot_base + s->n_envs <= s->ready_q->n_slots, APPO_ERR_CONTRACT,
                 "sampler_step: slots outside the ready queue's range");
    const int pst = slotq_push_launch(c, s->ready_q, nullptr, slot_base, s->n_envs, nullptr);
    if (pst != APPO_OK) return pst;
  }
  if (h_actions)
    APPO_CUDA_TRY(cudaMemcpyAsync(h_actions, s->actions, sizeof(int32_t) * s->n_envs,
                                  cudaMemcpyDeviceToHost, c->stream));
  s->steps_done++;
  return APPO_OK;
}

APPO_API int appo_rollout_act(appo_sampler* s, void* d_region, uint64_t slot_bytes,
                              int32_t slot_base, int t, const uint8_t* h_obs,
                              int32_t* h_actions) {
  SMP_OR_RETURN(s);
  appo_ctx* c = s->ctx;
  const Dims& d = c->model->d;
  APPO_REQUIRE(h_obs && d_region && slot_bytes >= d.slot[9], APPO_ERR_CONTRACT,
               "rollout_act: bad arguments");
  APPO_REQUIRE(t >= 0 && t < d.T, APPO_ERR_CONTRACT, "write_step: index beyond rollout length");
  APPO_REQUIRE(!s->acted && t == s->next_t, APPO_ERR_CONTRACT,
               "write_step: out-of-order step write");
  if (!s->host_ev) APPO_CUDA_TRY(cudaEventCreateWithFlags(&s->host_ev, cudaEventDisableTiming));
  uint8_t* region = static_cast<uint8_t*>(d_region);
  const uint64_t obs_off = d.slot[0] + (uint64_t)t * d.obs_dim;
  int st = stage_host_obs(s, h_obs, region, slot_bytes, slot_base, obs_off);
  if (st) return st;
  int64_t version = 0;
  st = sampler_infer(c, region + (uint64_t)slot_base * slot_bytes + obs_off, slot_bytes,
                     s->n_envs, s->hidden, s->steps_done * (uint64_t)s->n_envs, s->actions,
                     s->logp, s->h_out, s->values, nullptr, &version);
  if (st) return st;
  SlotOffsets off;
  std::memcpy(&off, d.slot, sizeof(off));
  APPO_LAUNCH(c, host_record_kernel, s->n_envs, 128, 0, s->n_envs, d.T, t, (uint32_t)d.obs_dim,
              version, s->hidden, s->h_out, s->actions, s->logp,
              static_cast<const uint8_t*>(nullptr), region, slot_bytes, (int64_t)slot_base, off);
  if (h_actions)
    APPO_CUDA_TRY(cudaMemcpyAsync(h_actions, s->actions, sizeof(int32_t) * s->n_envs,
                                  cudaMemcpyDeviceToHost, c->stream));
  APPO_CUDA_TRY(cudaEventRecord(s->host_ev, c->stream));
  s->acted = true;
  s->steps_done++;
  return APPO_OK;
}

APPO_API int appo_rollout_wait(appo_sampler* s) {
  SMP_OR_RETURN(s);
  if (s->host_ev) APPO_CUDA_TRY(cudaEventSynchronize(s->host_ev));
  return APPO_OK;
}

APPO_API int appo_rollout_feedback(appo_sampler* s, void* d_region, uint64_t slot_bytes,
                                   int32_t slot_base, int t, const float* h_rewards,
                                   const uint8_t* h_dones, const uint8_t* h_next_obs) {
  SMP_OR_RETURN(s);
  appo_ctx* c = s->ctx;
  const Dims& d = c->model->d;
  APPO_REQUIRE(h_rewards && h_dones && d_region && slot_bytes >= d.slot[9], APPO_ERR_CONTRACT,
               "rollout_feedback: bad arguments");
  APPO_REQUIRE(s->acted && t == s->next_t, APPO_ERR_CONTRACT,
               "write_step: out-of-order step write");
  APPO_REQUIRE(t < d.T - 1 || h_next_obs, APPO_ERR_CONTRACT,
               "seal: trajectory incomplete (missing steps or bootstrap)");
  const size_t fb = (size_t)s->n_envs * 5;
  if (!s->fb_host) {
    APPO_CUDA_TRY(cudaMallocHost(&s->fb_host, 2 * fb));
    APPO_CUDA_TRY(cudaMalloc(&s->fb_dev, 2 * fb));
    for (int k = 0; k < 2; ++k)
      APPO_CUDA_TRY(cudaEventCreateWithFlags(&s->fb_ev[k], cudaEventDisableTiming));
  }
  const int k = s->fb_next;
  s->fb_next ^= 1;
  // the half's previous upload has left the host buffer before it is refilled
  APPO_CUDA_TRY(cudaEventSynchronize(s->fb_ev[k]));
  uint8_t* hb = s->fb_host + k * fb;
  std::memcpy(hb, h_rewards, sizeof(float) * s->n_envs);
  std::memcpy(hb + (size_t)s->n_envs * 4, h_dones, s->n_envs);
  uint8_t* db = s->fb_dev + k * fb;
  APPO_CUDA_TRY(cudaMemcpyAsync(db, hb, fb, cudaMemcpyHostToDevice, c->stream));
  APPO_CUDA_TRY(cudaEventRecord(s->fb_ev[k], c->stream));
  uint8_t* region = static_cast<uint8_t*>(d_region);
  SlotOffsets off;
  std::memcpy(&off, d.slot, sizeof(off));
  APPO_LAUNCH(c, host_record_kernel, s->n_envs, 128, 0, s->n_envs, d.T, t, (uint32_t)d.obs_dim,
              (int64_t)0, s->hidden, s->h_out, s->actions, s->logp,
              static_cast<const uint8_t*>(db), region, slot_bytes, (int64_t)slot_base, off);
  if (t == d.T - 1) {
    // set_bootstrap: the step's next observation (orchestrator.hpp:529-534)
    const int st = stage_host_obs(s, h_next_obs, region, slot_bytes, slot_base, d.slot[7]);
    if (st) return st;
    if (!s->host_ev) APPO_CUDA_TRY(cudaEventCreateWithFlags(&s->host_ev, cudaEventDisableTiming));
    APPO_CUDA_TRY(cudaEventRecord(s->host_ev, c->stream));
    if (s->ready_q) {
      APPO_REQUIRE((int64_t)slot_base + s->n_envs <= s->ready_q->n_slots, APPO_ERR_CONTRACT,
                   "rollout_feedback: slots outside the ready queue's range");
      const int pst = slotq_push_launch(c, s->ready_q, nullptr, slot_base, s->n_envs, nullptr);
      if (pst != APPO_OK) return pst;
    }
  }
  s->acted = false;
  s->next_t = (t + 1) % d.T;
  return APPO_OK;
}

int appo_sampler_set_ready_queue(appo_sampler* s, appo_slotq* q) {
  SMP_OR_RETURN(s);
  APPO_REQUIRE(!q || (uint32_t)s->n_envs <= q->capacity, APPO_ERR_CONTRACT,
               "sampler_set_ready_queue: queue smaller than one rollout group");
  s->ready_q = q;
  return APPO_OK;
}

}  // extern "C"
