// Shared plumbing for libappo_b200.so: error handling (status codes of
// include/appo_capi.h mirroring ContractError/ConfigError/NumericError,
// common.hpp:20-45), the context, and small device helpers.
#pragma once
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/appo_capi.h"

namespace appo_b200 {

void set_error(const std::string& msg);

struct Model;   // model.cu
struct Reader;  // model.cuh: per-context inference scratch + read events

// Optional per-launch CUDA-event timing (appo_ctx_set_timing): the bench uses
// it to measure the dominant kernel's average duration live, on the stream
// the kernel runs on.
struct TimedLaunch {
  const char* name;
  cudaEvent_t a, b;
  double flops, bytes;
};

// Device flag slots raised by kernels; read by appo_ctx_sync.
enum : int { kFlagNumeric = 0, kFlagContract = 1, kFlagQueue = 2, kNumFlags = 4 };

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t seed = 0;
  int* d_flags = nullptr;        // [kNumFlags] live + [kNumFlags] frozen by the global norm
  double* d_red = nullptr;       // reduction workspace (partials), kRedSlots doubles
  unsigned* d_counter = nullptr; // last-block counters
  double* h_pinned = nullptr;    // small pinned readback buffer
  int64_t launches = 0;
  float* d_ws = nullptr;         // split-K GEMM workspace
  size_t ws_bytes = 0;
  int num_sms = 148;
  bool pdl = true;  // launch with programmatic stream serialisation (APPO_PDL_ENTRY)
  // timing
  bool timing = false;
  std::string timing_filter;
  int timing_stride = 1;      // time every N-th matching launch ("@N:" filter prefix)
  uint64_t timing_seq = 0;
  std::vector<TimedLaunch> timed;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  const char* next_name = nullptr;  // overrides the kernel symbol name
  double next_flops = 0.0, next_bytes = 0.0;
  // data-parallel learner (dp.cu): communicator, side stream for the bucketed
  // gradient all-reduce, its events, and the rank-consensus rejection flags
  void* dp_comm = nullptr;
  int dp_size = 1, dp_rank = 0;
  cudaStream_t dp_stream = nullptr;
  static constexpr int kDpEvents = 8;
  cudaEvent_t dp_ev[kDpEvents] = {};
  unsigned dp_ev_next = 0;
  int* d_dp_flags = nullptr;
  bool has_model = false;
  bool owns_model = true;  // false for appo_ctx_create_shared contexts
  appo_model_desc desc{};
  Model* model = nullptr;
  Reader* reader = nullptr;  // inference state of this context (model.cu)
  // host -> device observation copies of every sampler on this context, in
  // issue order on one stream: groups' transfers queue back to back instead
  // of splitting the link (sampler.cu)
  cudaStream_t copy_stream = nullptr;
  // GRU recurrence kernels (gru_seq.cu): per-group step counters (fwd [0, 4),
  // bwd [4, 8)), bias-gradient combine counters [32, 64), per-group bias
  // partial sums [4][512][4]; allocated zeroed on first use
  unsigned* d_gru_sync = nullptr;
  // GRU step counters are never reset: each launch waits for base + epoch *
  // CTAs, with the base per counter tracked here (no memset node between the
  // kernels, so the GRU launches keep programmatic dependent launch)
  unsigned gru_epochs[8] = {};
  float* d_gru_part = nullptr;
  // learner side stream (model.cu): weight-gradient kernels of the backward
  // run here beside the input-gradient chain on `stream`, with their own
  // split-K workspace; fork/join by events
  bool fork = true;  // appo_ctx_set_learner_fork
  bool on_side = false;  // launches go to side_stream (timing class name gets "@side")
  cudaStream_t side_stream = nullptr;
  static constexpr int kSideEvents = 16;
  cudaEvent_t side_ev[kSideEvents] = {};
  unsigned side_ev_next = 0;
  float* side_ws = nullptr;
  size_t side_ws_bytes = 0;
  // the rest of a learner step's Adam (past the convolution parameters) runs
  // on the side stream beside the next step's convolutions; that step joins
  // adam_tail_ev before its FC forward
  cudaEvent_t adam_tail_ev = nullptr;
  bool adam_tail_pending = false;
};
constexpr int kRedSlots = 148 * 8 * 16;

}  // namespace appo_b200

struct appo_ctx : appo_b200::Ctx {};

#define APPO_CUDA_TRY(expr)                                                          \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      appo_b200::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));      \
      return APPO_ERR_RESOURCE;                                                      \
    }                                                                                \
  } while (0)

#define APPO_TRY(x)                       \
  do {                                    \
    int _st_ = (x);                       \
    if (_st_ != APPO_OK) return _st_;     \
  } while (0)

#define APPO_REQUIRE(cond, code, msg)  \
  do {                                 \
    if (!(cond)) {                     \
      appo_b200::set_error(msg);       \
      return (code);                   \
    }                                  \
  } while (0)

// Programmatic dependent launch: every kernel of the library starts with
// APPO_PDL_ENTRY() (wait for the previous kernel's completion + memory, then
// let the next kernel launch), so kernels are launched with
// programmatic stream serialisation and the next kernel's launch and
// prologue overlap the current one's tail.  APPO_PDL=0 disables it.
namespace appo_b200 {
// default for a new context: APPO_PDL unset/B = contexts that own a model
// (learners) only, 1 = all, 0 = none, S = shared contexts (samplers) only.
// Measured in bench.py: PDL on the learner +4%, on the concurrently running
// sampler -5% (its early-launched, waiting CTAs hold SMs the learner needs).
inline bool pdl_default(bool shared) {
  const char* e = getenv("APPO_PDL");
  if (!e || !e[0] || e[0] == 'B') return !shared;
  if (e[0] == '1') return true;
  if (e[0] == 'B') return !shared;
  if (e[0] == 'S') return shared;
  return false;
}
// learner backward on two streams (model.cu); APPO_LEARNER_FORK=0 turns the
// default off
inline bool learner_fork_default() {
  const char* v = getenv("APPO_LEARNER_FORK");
  return !(v && v[0] == '0');
}
}  // namespace appo_b200
#define APPO_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
#define APPO_PDL_TRIGGER() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")
#define APPO_PDL_ENTRY() \
  do {                   \
    APPO_PDL_WAIT();     \
    APPO_PDL_TRIGGER();  \
  } while (0)

// Launch-and-count: every kernel of the library goes through this so
// appo_ctx_launch_count reports how many of OUR kernels ran.
#define APPO_LAUNCH(ctx, kernel, grid, block, smem, ...)                        \
  do {                                                                         \
    const char* _nm = (ctx)->next_name ? (ctx)->next_name : #kernel;           \
    cudaEvent_t _ea = appo_b200::timing_begin((ctx), _nm);                     \
    cudaLaunchConfig_t _cfg = {};                                              \
    _cfg.gridDim = dim3(grid);                                                 \
    _cfg.blockDim = dim3(block);                                               \
    _cfg.dynamicSmemBytes = (smem);                                            \
    _cfg.stream = (ctx)->stream;                                               \
    cudaLaunchAttribute _at[1];                                                \
    _at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;            \
    _at[0].val.programmaticStreamSerializationAllowed = 1;                     \
    _cfg.attrs = _at;                                                          \
    _cfg.numAttrs = (ctx)->pdl ? 1 : 0;                                        \
    cudaError_t _le = cudaLaunchKernelEx(&_cfg, kernel, __VA_ARGS__);          \
    appo_b200::timing_end((ctx), _nm, _ea);                                    \
    (ctx)->launches++;                                                         \
    if (_le == cudaSuccess) _le = cudaGetLastError();                          \
    if (_le != cudaSuccess) {                                                  \
      appo_b200::set_error(std::string("launch " #kernel ": ") +               \
                           cudaGetErrorString(_le));                           \
      return APPO_ERR_RESOURCE;                                                \
    }                                                                          \
  } while (0)

namespace appo_b200 {

cudaEvent_t timing_event(Ctx* c);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize, bytes) for `kernel` on the
// current device, once per (kernel, device): the attribute is per device, so a
// process driving learners on several GPUs must set it on each.
int ensure_smem_attr(const void* kernel, int bytes, int device);
// interned "<name>@side": kernels on the learner side stream run beside the
// main chain, so their event-timed durations are a separate timing class
const char* side_class_name(const char* name);
// host-side wait for everything this context enqueued (main + side stream)
inline cudaError_t ctx_streams_sync(Ctx* c) {
  if (c->side_stream) {
    const cudaError_t e = cudaStreamSynchronize(c->side_stream);
    if (e != cudaSuccess) return e;
  }
  return cudaStreamSynchronize(c->stream);
}
inline cudaEvent_t timing_begin(Ctx* c, const char* name) {
  if (!c->timing) return nullptr;
  if (c->on_side) name = side_class_name(name);
  // filter: one kernel class name, or several separated by '|'
  if (!c->timing_filter.empty() && c->timing_filter != "gemm_shapes" &&
      ("|" + c->timing_filter + "|").find("|" + std::string(name) + "|") == std::string::npos)
    return nullptr;
  // sampling: only every timing_stride-th matching launch is bracketed (an
  // event between two kernels ends their programmatic-dependent-launch overlap)
  if (c->timing_stride > 1 && (c->timing_seq++ % (uint64_t)c->timing_stride) != 0) return nullptr;
  cudaEvent_t e = timing_event(c);
  cudaEventRecord(e, c->stream);
  return e;
}
inline void timing_end(Ctx* c, const char* name, cudaEvent_t a) {
  if (a) {
    if (c->on_side) name = side_class_name(name);
    cudaEvent_t b = timing_event(c);
    cudaEventRecord(b, c->stream);
    c->timed.push_back(TimedLaunch{name, a, b, c->next_flops, c->next_bytes});
  }
  c->next_name = nullptr;
  c->next_flops = 0.0;
  c->next_bytes = 0.0;
}

__device__ __forceinline__ bool finitef(float x) { return isfinite(x); }

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// Counter-based uniform in [0,1) (oracle: orc_uniform).
__device__ __forceinline__ double uniform01(uint64_t key, uint64_t counter) {
  uint64_t h = splitmix64(key ^ splitmix64(counter));
  return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

inline uint64_t host_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
inline uint64_t host_derive_seed(uint64_t seed, uint64_t stream) {
  return host_splitmix64(seed ^ host_splitmix64(stream + 1));
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Kernel-side launchers implemented in the .cu files (return appo_status).
int launch_vtrace(Ctx* c, int n_traj, int T, const float* r, const float* v, const float* boot,
                  const float* tl, const float* bl, const uint8_t* d, float gamma, float rho_bar,
                  float c_bar, float* v_out, float* pg_out, float* rho_out, float* c_out);
int launch_nstep(Ctx* c, int n_traj, int T, const float* r, const float* boot, const uint8_t* d,
                 float gamma, float* ret);
int launch_gae(Ctx* c, int n_traj, int T, const float* r, const float* v, const float* boot,
               const uint8_t* d, float gamma, float lambda, float* adv, float* ret);
int launch_total_loss(Ctx* c, int n, const float* ratios, const float* adv, const float* values,
                      const float* vt, const float* ent, float lo, float hi, float vc, float ec,
                      double* d_out4);
// Factored action heads (ActionHeadsSpec, policy.hpp:25-35): head j's logits
// are columns [off[j], off[j+1]) of a row; off[n] = logits_dim.
constexpr int kMaxHeads = 8;
struct HeadsSpec {
  int n;
  int off[kMaxHeads + 1];
};
int launch_logp_entropy(Ctx* c, int B, const HeadsSpec& hs, const float* logits,
                        const int32_t* actions, float* logp, float* ent);
int launch_sample(Ctx* c, int B, const HeadsSpec& hs, const float* logits, uint64_t key,
                  uint64_t counter0, int32_t* actions, float* logp);
// peer_flags (data-parallel): the ranks' max-reduced rejection flags, folded
// into c's flags before the update so every rank accepts or rejects together
int launch_adam(Ctx* c, int64_t n, float* theta, float* m, float* v, const float* g, int64_t t,
                float lr, float b1, float b2, float eps, float clip, double* d_norm_out,
                uint16_t* bf16_copy, float* f32_copy, unsigned* applied,
                const int* peer_flags = nullptr, int64_t n_head = -1);
// n_head >= 0 above: Adam ran over [0, n_head) only; this runs it over
// [lo, n) with the same norm and frozen accept/reject decision
int launch_adam_rest(Ctx* c, int64_t n, int64_t lo, float* theta, float* m, float* v,
                     const float* g, int64_t t, float lr, float b1, float b2, float eps,
                     double* d_norm_out, uint16_t* bf16_copy, float* f32_copy);

}  // namespace appo_b200
