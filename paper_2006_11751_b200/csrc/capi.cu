// C ABI entry points (include/appo_capi.h): context management and the
// stateless hot-path kernels.  Model-level entry points live in model.cu.
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "appo_common.cuh"

namespace appo_b200 {
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

cudaEvent_t timing_event(Ctx* c) {
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[c->ev_used++];
}
int ensure_smem_attr(const void* kernel, int bytes, int device) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> set;
  std::lock_guard<std::mutex> lk(mu);
  int& have = set[{kernel, device}];
  if (have >= bytes) return APPO_OK;
  APPO_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  have = bytes;
  return APPO_OK;
}
}  // namespace appo_b200

using namespace appo_b200;

namespace {
int check_ctx(appo_ctx* ctx) {
  if (!ctx) {
    set_error("null appo_ctx");
    return APPO_ERR_CONTRACT;
  }
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) {
    set_error(std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    return APPO_ERR_RESOURCE;
  }
  return APPO_OK;
}
// VTraceConfig::validate (offpolicy.hpp:23-27)
int validate_vtrace(float gamma, float rho_bar, float c_bar) {
  if (!(rho_bar >= c_bar && c_bar > 0.0f)) {
    set_error("vtrace requires rho_bar >= c_bar > 0");
    return APPO_ERR_CONFIG;
  }
  if (!(gamma > 0.0f && gamma <= 1.0f)) {
    set_error("discount must be in (0,1]");
    return APPO_ERR_CONFIG;
  }
  return APPO_OK;
}
}  // namespace

#define CTX_OR_RETURN(ctx)             \
  do {                                 \
    int _s = check_ctx(ctx);           \
    if (_s != APPO_OK) return _s;      \
  } while (0)

namespace appo_b200 {
void dp_destroy(Ctx* c);      // dp.cu
void reader_release(Ctx* c);  // model.cu
}
int model_create(appo_b200::Ctx* c);   // model.cu
void model_destroy(appo_b200::Ctx* c); // model.cu

extern "C" {

const char* appo_last_error(void) { return g_last_error.c_str(); }
int appo_capi_version(void) { return APPO_CAPI_VERSION; }

int appo_ctx_create(const appo_model_desc* desc, int device, uint64_t seed, appo_ctx** out) {
  APPO_REQUIRE(out != nullptr, APPO_ERR_CONTRACT, "appo_ctx_create: null out");
  int n = 0;
  APPO_CUDA_TRY(cudaGetDeviceCount(&n));
  APPO_REQUIRE(device >= 0 && device < n, APPO_ERR_CONTRACT, "appo_ctx_create: bad device");
  APPO_CUDA_TRY(cudaSetDevice(device));
  appo_ctx* c = new appo_ctx();
  c->device = device;
  c->seed = seed;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (c->num_sms <= 0) c->num_sms = 148;
  c->pdl = pdl_default(false);
  c->fork = learner_fork_default();
  if (cudaMalloc(&c->d_flags, sizeof(int) * 2 * kNumFlags) != cudaSuccess ||
      cudaMalloc(&c->d_red, sizeof(double) * kRedSlots) != cudaSuccess ||
      cudaMalloc(&c->d_counter, sizeof(unsigned) * 16) != cudaSuccess ||
      cudaMallocHost(&c->h_pinned, sizeof(double) * 64) != cudaSuccess) {
    set_error("appo_ctx_create: allocation failed");
    delete c;
    return APPO_ERR_RESOURCE;
  }
  cudaMemset(c->d_flags, 0, sizeof(int) * 2 * kNumFlags);
  cudaMemset(c->d_counter, 0, sizeof(unsigned) * 16);
  cudaDeviceSynchronize();
  if (desc) {
    c->has_model = true;
    c->desc = *desc;
    int st = model_create(c);
    if (st != APPO_OK) {
      appo_ctx_destroy(c);
      return st;
    }
  }
  *out = c;
  return APPO_OK;
}

int appo_ctx_set_learner_fork(appo_ctx* ctx, int enable) {
  CTX_OR_RETURN(ctx);
  ctx->fork = enable != 0;
  return APPO_OK;
}

int appo_ctx_set_pdl(appo_ctx* ctx, int enable) {
  CTX_OR_RETURN(ctx);
  ctx->pdl = enable != 0;
  return APPO_OK;
}

int appo_ctx_create_shared(appo_ctx* base, appo_ctx** out) {
  APPO_REQUIRE(base && base->model && out, APPO_ERR_CONTRACT,
               "appo_ctx_create_shared: base context with a model required");
  appo_ctx* c = nullptr;
  int st = appo_ctx_create(nullptr, base->device, base->seed, &c);
  if (st) return st;
  c->has_model = true;
  c->desc = base->desc;
  c->model = base->model;
  c->owns_model = false;
  c->pdl = pdl_default(true);
  *out = c;
  return APPO_OK;
}

int appo_ctx_destroy(appo_ctx* ctx) {
  if (!ctx) return APPO_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  cudaDeviceSynchronize();
  if (ctx->model) appo_b200::reader_release(ctx);
  if (ctx->model && ctx->owns_model) model_destroy(ctx);
  appo_b200::dp_destroy(ctx);
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
  }
  if (ctx->side_stream) {
    cudaStreamSynchronize(ctx->side_stream);
    cudaStreamDestroy(ctx->side_stream);
  }
  if (ctx->adam_tail_ev) cudaEventDestroy(ctx->adam_tail_ev);
  for (auto e : ctx->side_ev)
    if (e) cudaEventDestroy(e);
  cudaFree(ctx->side_ws);
  cudaFree(ctx->d_gru_sync);
  cudaFree(ctx->d_gru_part);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  cudaFree(ctx->d_flags);
  cudaFree(ctx->d_red);
  cudaFree(ctx->d_counter);
  cudaFreeHost(ctx->h_pinned);
  delete ctx;
  return APPO_OK;
}

int appo_ctx_set_sm_budget(appo_ctx* ctx, int n_sms) {
  CTX_OR_RETURN(ctx);
  int dev_sms = 0;
  APPO_CUDA_TRY(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, ctx->device));
  APPO_REQUIRE(n_sms >= 1, APPO_ERR_CONTRACT, "sm budget must be >= 1");
  ctx->num_sms = n_sms < dev_sms ? n_sms : dev_sms;
  return APPO_OK;
}

int appo_ctx_set_stream(appo_ctx* ctx, void* stream) {
  CTX_OR_RETURN(ctx);
  ctx->stream = static_cast<cudaStream_t>(stream);
  return APPO_OK;
}

int appo_ctx_sync(appo_ctx* ctx) {
  CTX_OR_RETURN(ctx);
  int flags[kNumFlags];
  APPO_CUDA_TRY(cudaMemcpyAsync(flags, ctx->d_flags, sizeof(flags), cudaMemcpyDeviceToHost,
                                ctx->stream));
  APPO_CUDA_TRY(ctx_streams_sync(ctx));
  if (flags[kFlagNumeric] || flags[kFlagContract] || flags[kFlagQueue]) {
    APPO_CUDA_TRY(cudaMemsetAsync(ctx->d_flags, 0, sizeof(flags), ctx->stream));
    APPO_CUDA_TRY(ctx_streams_sync(ctx));
    if (flags[kFlagQueue]) {
      set_error("slot queue: timed out waiting on the device for published slot ids");
      return APPO_ERR_RESOURCE;
    }
    if (flags[kFlagContract]) {
      set_error("contract violation detected on device (action index out of range?)");
      return APPO_ERR_CONTRACT;
    }
    set_error("non-finite value detected on device (NumericError)");
    return APPO_ERR_NUMERIC;
  }
  return APPO_OK;
}

int64_t appo_ctx_launch_count(appo_ctx* ctx) { return ctx ? ctx->launches : -1; }

int appo_ctx_set_timing(appo_ctx* ctx, int enable, const char* name_filter) {
  CTX_OR_RETURN(ctx);
  APPO_CUDA_TRY(ctx_streams_sync(ctx));
  ctx->timing = enable != 0;
  std::string f = name_filter ? name_filter : "";
  ctx->timing_stride = 1;
  ctx->timing_seq = 0;
  if (f.size() > 1 && f[0] == '@') {  // "@N:names": sample every N-th matching launch
    const size_t colon = f.find(':');
    ctx->timing_stride = atoi(f.substr(1, colon == std::string::npos ? std::string::npos : colon - 1).c_str());
    if (ctx->timing_stride < 1) ctx->timing_stride = 1;
    f = colon == std::string::npos ? std::string() : f.substr(colon + 1);
  }
  ctx->timing_filter = f;
  ctx->timed.clear();
  ctx->ev_used = 0;
  return APPO_OK;
}

// Aggregated per-kernel timing since appo_ctx_set_timing, as JSON lines
// {"name":..,"launches":..,"ms":..,"flops":..,"bytes":..}.  Synchronizes.
int appo_ctx_timing_report(appo_ctx* ctx, char* buf, int buflen) {
  CTX_OR_RETURN(ctx);
  APPO_CUDA_TRY(ctx_streams_sync(ctx));
  struct Agg {
    std::string name;
    long n = 0;
    double ms = 0, flops = 0, bytes = 0;
  };
  std::vector<Agg> agg;
  for (const auto& t : ctx->timed) {
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, t.a, t.b);
    Agg* a = nullptr;
    for (auto& x : agg)
      if (x.name == t.name) a = &x;
    if (!a) {
      agg.push_back(Agg{t.name});
      a = &agg.back();
    }
    a->n++;
    a->ms += ms;
    a->flops += t.flops;
    a->bytes += t.bytes;
  }
  std::string out;
  for (const auto& a : agg) {
    char line[512];
    snprintf(line, sizeof(line),
             "{\"name\": \"%s\", \"launches\": %ld, \"ms\": %.6f, \"flops\": %.6e, "
             "\"bytes\": %.6e}\n",
             a.name.c_str(), a.n, a.ms, a.flops, a.bytes);
    out += line;
  }
  APPO_REQUIRE((int)out.size() < buflen, APPO_ERR_CONTRACT, "timing report buffer too small");
  std::memcpy(buf, out.c_str(), out.size() + 1);
  ctx->timed.clear();
  ctx->ev_used = 0;
  return APPO_OK;
}

int appo_vtrace(appo_ctx* ctx, int n_traj, int T, const float* r, const float* v,
                const float* boot, const float* tl, const float* bl, const uint8_t* d,
                float gamma, float rho_bar, float c_bar, float* v_out, float* pg_out,
                float* rho_out, float* c_out) {
  CTX_OR_RETURN(ctx);
  int st = validate_vtrace(gamma, rho_bar, c_bar);
  if (st) return st;
  APPO_REQUIRE(n_traj >= 0 && T >= 0, APPO_ERR_CONTRACT, "vtrace: negative shape");
  APPO_REQUIRE(n_traj == 0 || T == 0 || (r && v && boot && tl && bl && d && v_out && pg_out),
               APPO_ERR_CONTRACT, "vtrace: null buffer");
  return launch_vtrace(ctx, n_traj, T, r, v, boot, tl, bl, d, gamma, rho_bar, c_bar, v_out,
                       pg_out, rho_out, c_out);
}

int appo_nstep_returns(appo_ctx* ctx, int n_traj, int T, const float* r, const float* boot,
                       const uint8_t* d, float gamma, float* ret) {
  CTX_OR_RETURN(ctx);
  APPO_REQUIRE(n_traj >= 0 && T >= 0, APPO_ERR_CONTRACT, "nstep: negative shape");
  return launch_nstep(ctx, n_traj, T, r, boot, d, gamma, ret);
}

int appo_gae(appo_ctx* ctx, int n_traj, int T, const float* r, const float* v, const float* boot,
             const uint8_t* d, float gamma, float lambda, float* adv, float* ret) {
  CTX_OR_RETURN(ctx);
  APPO_REQUIRE(n_traj >= 0 && T >= 0, APPO_ERR_CONTRACT, "gae: negative shape");
  APPO_REQUIRE(gamma > 0.0f && gamma <= 1.0f, APPO_ERR_CONFIG, "discount must be in (0,1]");
  APPO_REQUIRE(lambda >= 0.0f && lambda <= 1.0f, APPO_ERR_CONFIG, "gae lambda must be in [0,1]");
  return launch_gae(ctx, n_traj, T, r, v, boot, d, gamma, lambda, adv, ret);
}

int appo_total_loss(appo_ctx* ctx, int n, const float* ratios, const float* adv,
                    const float* values, const float* vt, const float* ent, float lo, float hi,
                    float vc, float ec, double* h_out4) {
  CTX_OR_RETURN(ctx);
  APPO_REQUIRE(0.0f < lo && lo < 1.0f && 1.0f < hi, APPO_ERR_CONFIG,
               "ppo clip requires 0 < low < 1 < high");
  APPO_REQUIRE(n >= 0 && h_out4, APPO_ERR_CONTRACT, "total_loss: bad arguments");
  double* d_out = ctx->d_red + kRedSlots - 8;
  int st = launch_total_loss(ctx, n, ratios, adv, values, vt, ent, lo, hi, vc, ec, d_out);
  if (st) return st;
  APPO_CUDA_TRY(cudaMemcpyAsync(ctx->h_pinned, d_out, sizeof(double) * 4, cudaMemcpyDeviceToHost,
                                ctx->stream));
  st = appo_ctx_sync(ctx);
  std::memcpy(h_out4, ctx->h_pinned, sizeof(double) * 4);
  return st;
}

namespace {
// ActionHeadsSpec validation: 1..kMaxHeads heads of 1..64 actions each
int make_heads(int n_heads, const int32_t* sizes, HeadsSpec* hs) {
  APPO_REQUIRE(n_heads >= 1 && n_heads <= kMaxHeads && sizes != nullptr, APPO_ERR_CONTRACT,
               "action heads: need 1..8 heads");
  hs->n = n_heads;
  hs->off[0] = 0;
  for (int j = 0; j < n_heads; ++j) {
    APPO_REQUIRE(sizes[j] >= 1 && sizes[j] <= 64, APPO_ERR_CONTRACT,
                 "action heads: head size must be in [1, 64]");
    hs->off[j + 1] = hs->off[j] + sizes[j];
  }
  return APPO_OK;
}
}  // namespace

int appo_logp_entropy(appo_ctx* ctx, int B, int A, const float* logits, const int32_t* actions,
                      float* logp, float* ent) {
  return appo_logp_entropy_heads(ctx, B, 1, &A, logits, actions, logp, ent);
}

int appo_sample_actions(appo_ctx* ctx, int B, int A, const float* logits, uint64_t key,
                        uint64_t counter0, int32_t* actions, float* logp) {
  return appo_sample_actions_heads(ctx, B, 1, &A, logits, key, counter0, actions, logp);
}

int appo_logp_entropy_heads(appo_ctx* ctx, int B, int n_heads, const int32_t* h_sizes,
                            const float* logits, const int32_t* actions, float* logp,
                            float* ent) {
  CTX_OR_RETURN(ctx);
  APPO_REQUIRE(B >= 0, APPO_ERR_CONTRACT, "logp_entropy: bad shape");
  HeadsSpec hs;
  if (int st = make_heads(n_heads, h_sizes, &hs)) return st;
  return launch_logp_entropy(ctx, B, hs, logits, actions, logp, ent);
}

int appo_sample_actions_heads(appo_ctx* ctx, int B, int n_heads, const int32_t* h_sizes,
                              const float* logits, uint64_t key, uint64_t counter0,
                              int32_t* actions, float* logp) {
  CTX_OR_RETURN(ctx);
  APPO_REQUIRE(B >= 0, APPO_ERR_CONTRACT, "sample: bad shape");
  HeadsSpec hs;
  if (int st = make_heads(n_heads, h_sizes, &hs)) return st;
  return launch_sample(ctx, B, hs, logits, key, counter0, actions, logp);
}

int appo_adam_step(appo_ctx* ctx, int64_t n, float* theta, float* m, float* v, const float* g,
                   int64_t t, float lr, float b1, float b2, float eps, float clip,
                   double* h_grad_norm) {
  CTX_OR_RETURN(ctx);
  APPO_REQUIRE(n >= 0 && t >= 1, APPO_ERR_CONTRACT, "adam: n >= 0 and t >= 1 required");
  double* d_norm = ctx->d_red + kRedSlots - 16;
  int st = launch_adam(ctx, n, theta, m, v, g, t, lr, b1, b2, eps, clip, d_norm, nullptr, nullptr,
                       nullptr);
  if (st) return st;
  if (h_grad_norm) {
    APPO_CUDA_TRY(cudaMemcpyAsync(ctx->h_pinned, d_norm, sizeof(double), cudaMemcpyDeviceToHost,
                                  ctx->stream));
    st = appo_ctx_sync(ctx);
    *h_grad_norm = ctx->h_pinned[0];
    return st;
  }
  return APPO_OK;
}

}  // extern "C"
