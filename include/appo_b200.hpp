// appo_b200.hpp -- header-only C++ host mirror of the reference's hot-path API
// over the C ABI (appo_capi.h).  A host that used
//   appo::vtrace / appo::nstep_returns / appo::total_loss          (offpolicy.hpp)
//   appo::sample_action / appo::log_prob_and_entropy /
//   appo::optimizer_step                                           (policy.hpp)
//   PolicyWorkerUnit::run_once / LearnerUnit::step                 (orchestrator.hpp)
// switches to the same names in namespace appo_b200, with the same std::span
// arguments and output structs, and the same exceptions: when the reference's
// <appo/common.hpp> is on the include path (the drop-in case) the mirror
// throws ::appo::ContractError / ConfigError / NumericError themselves
// (common.hpp:20-40), so the reference's own catch sites -- e.g. the CLI's
// exit-code mapping, tools/appo_cli.cpp:151-163 -- keep working unchanged;
// otherwise it defines look-alike types (define APPO_B200_OWN_ERRORS to force
// them).  Host-span overloads stage through device memory (the
// reference-facing e2e path); device-pointer overloads are the zero-copy path.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "appo_capi.h"

#if !defined(APPO_B200_OWN_ERRORS) && __has_include(<appo/common.hpp>)
#include <appo/common.hpp>
#define APPO_B200_REFERENCE_ERRORS 1
namespace appo_b200 {
using ContractError = ::appo::ContractError;  // common.hpp:23-26
using ConfigError = ::appo::ConfigError;      // common.hpp:30-33
using NumericError = ::appo::NumericError;    // common.hpp:37-40
}  // namespace appo_b200
#else
#define APPO_B200_REFERENCE_ERRORS 0
namespace appo_b200 {
class ContractError : public std::logic_error {
 public:
  explicit ContractError(const std::string& w) : std::logic_error(w) {}
};
class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};
class NumericError : public std::runtime_error {
 public:
  explicit NumericError(const std::string& w) : std::runtime_error(w) {}
};
}  // namespace appo_b200
#endif

namespace appo_b200 {

// CUDA / allocation failures.  The reference has no type of its own for these
// (std::bad_alloc / std::runtime_error); the CLI's catch-all maps them to
// kExitResource (appo_cli.cpp:157-163, runner.hpp:28-33).
class ResourceError : public std::runtime_error {
 public:
  explicit ResourceError(const std::string& w) : std::runtime_error(w) {}
};

inline void check(int st) {
  if (st == APPO_OK) return;
  const std::string m = appo_last_error();
  switch (st) {
    case APPO_ERR_CONTRACT: throw ContractError(m);
    case APPO_ERR_CONFIG: throw ConfigError(m);
    case APPO_ERR_NUMERIC: throw NumericError(m);
    default: throw ResourceError(m);
  }
}

// ActionHeadsSpec / FactoredAction (policy.hpp:25-37)
struct ActionHeadsSpec {
  std::vector<int> sizes;
  int n_heads() const { return static_cast<int>(sizes.size()); }
  int logits_dim() const {
    int d = 0;
    for (int s : sizes) d += s;
    return d;
  }
};
using FactoredAction = std::vector<std::int32_t>;

// AdamConfig / AdamState / PolicyParams' optimizer fields (policy.hpp:88-105)
struct AdamConfig {
  double lr = 1e-4;
  double beta1 = 0.9;
  double beta2 = 0.999;
  double eps = 1e-6;
  double grad_clip = 4.0;  // global-norm threshold, 0 disables
};
struct AdamState {
  std::vector<double> m, v;
  std::int64_t t = 0;
};
struct PolicyParams {
  std::vector<double> theta;  // flat parameter vector
  std::int64_t version = 0;   // SGD-step counter
  AdamState adam;
};

// offpolicy.hpp:18-45 defaults
struct VTraceConfig {
  double rho_bar = 1.0;
  double c_bar = 1.0;
  double gamma = 0.99;
};
struct VTraceOutput {  // offpolicy.hpp:30-35
  std::vector<double> v, pg_adv, rho, c;
};
struct LossComponents {  // offpolicy.hpp:136-141
  double policy = 0, value = 0, entropy = 0, total = 0;
};

// RAII device buffer (plumbing only).
template <class T>
class DeviceBuffer {
 public:
  explicit DeviceBuffer(size_t n) : n_(n) {
    if (n && cudaMalloc(&p_, n * sizeof(T)) != cudaSuccess) throw ResourceError("cudaMalloc");
  }
  ~DeviceBuffer() { cudaFree(p_); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  T* get() const { return p_; }
  size_t size() const { return n_; }
  void upload(const T* h) { cudaMemcpy(p_, h, n_ * sizeof(T), cudaMemcpyHostToDevice); }
  void download(T* h) const { cudaMemcpy(h, p_, n_ * sizeof(T), cudaMemcpyDeviceToHost); }

 private:
  T* p_ = nullptr;
  size_t n_;
};

// One device context (appo_ctx): stream, optional model (parameters + Adam).
class Context {
 public:
  explicit Context(int device = 0, uint64_t seed = 1, const appo_model_desc* model = nullptr) {
    if (model) desc_ = *model;
    check(appo_ctx_create(model, device, seed, &h_));
  }
  ~Context() { appo_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  appo_ctx* get() const { return h_; }
  void sync() const { check(appo_ctx_sync(h_)); }

  // vtrace (offpolicy.hpp:61): one trajectory, host spans, fp64 in/out like
  // the reference (computed in fp32 on the device; |err| <= 1e-5 max(|ref|,1)).
  VTraceOutput vtrace(std::span<const double> rewards, std::span<const double> values,
                      double bootstrap_value, std::span<const double> target_logp,
                      std::span<const double> behavior_logp, std::span<const uint8_t> dones,
                      const VTraceConfig& cfg) const {
    const size_t T = rewards.size();
    if (values.size() != T || target_logp.size() != T || behavior_logp.size() != T ||
        dones.size() != T)
      throw ContractError("vtrace inputs must share length T");
    auto f = [](std::span<const double> s) { return std::vector<float>(s.begin(), s.end()); };
    const std::vector<float> r = f(rewards), v = f(values), tl = f(target_logp),
                             bl = f(behavior_logp);
    const float boot = static_cast<float>(bootstrap_value);
    DeviceBuffer<float> dr(T), dv(T), dtl(T), dbl(T), dboot(1), o0(T), o1(T), o2(T), o3(T);
    DeviceBuffer<uint8_t> dd(T);
    dr.upload(r.data()); dv.upload(v.data()); dtl.upload(tl.data()); dbl.upload(bl.data());
    dboot.upload(&boot); dd.upload(dones.data());
    check(appo_vtrace(h_, 1, static_cast<int>(T), dr.get(), dv.get(), dboot.get(), dtl.get(),
                      dbl.get(), dd.get(), static_cast<float>(cfg.gamma),
                      static_cast<float>(cfg.rho_bar), static_cast<float>(cfg.c_bar), o0.get(),
                      o1.get(), o2.get(), o3.get()));
    sync();
    std::vector<float> a(T), b(T), c(T), d(T);
    o0.download(a.data()); o1.download(b.data()); o2.download(c.data()); o3.download(d.data());
    VTraceOutput out;
    out.v.assign(a.begin(), a.end());
    out.pg_adv.assign(b.begin(), b.end());
    out.rho.assign(c.begin(), c.end());
    out.c.assign(d.begin(), d.end());
    return out;
  }

  // nstep_returns (offpolicy.hpp:104-114): one trajectory, host spans.
  std::vector<double> nstep_returns(std::span<const double> rewards, double bootstrap_value,
                                    std::span<const uint8_t> dones, double gamma) const {
    const size_t T = rewards.size();
    if (dones.size() != T) throw ContractError("nstep_returns inputs must share length T");
    const std::vector<float> r(rewards.begin(), rewards.end());
    const float boot = static_cast<float>(bootstrap_value);
    DeviceBuffer<float> dr(T), dboot(1), dret(T);
    DeviceBuffer<uint8_t> dd(T);
    dr.upload(r.data()); dboot.upload(&boot); dd.upload(dones.data());
    check(appo_nstep_returns(h_, 1, static_cast<int>(T), dr.get(), dboot.get(), dd.get(),
                             static_cast<float>(gamma), dret.get()));
    sync();
    std::vector<float> o(T);
    dret.download(o.data());
    return std::vector<double>(o.begin(), o.end());
  }

  // sample_action (policy.hpp:232-258): one row of concatenated head logits.
  // The device draws counter-based uniforms; one draw of the caller's
  // mt19937_64 keys them, so a seeded rng gives a reproducible stream
  // (test_policy.cpp:226-239) with the reference's distribution, though not
  // the reference's individual draws.
  std::pair<FactoredAction, double> sample_action(const ActionHeadsSpec& heads,
                                                  std::span<const double> logits,
                                                  std::mt19937_64& rng) const {
    if (static_cast<int>(logits.size()) != heads.logits_dim())
      throw ContractError("sample_action: logits size != heads.logits_dim()");
    const std::vector<float> lg(logits.begin(), logits.end());
    DeviceBuffer<float> dl(lg.size()), dlp(1);
    DeviceBuffer<int32_t> da(heads.sizes.size());
    dl.upload(lg.data());
    sample_actions(heads, 1, dl.get(), rng(), 0, da.get(), dlp.get());
    sync();
    FactoredAction a(heads.sizes.size());
    float lp = 0;
    da.download(a.data());
    dlp.download(&lp);
    return {std::move(a), static_cast<double>(lp)};
  }
  // Batched device form: B rows, actions [B][n_heads], u = U(key, counter0 + b*n_heads + j).
  void sample_actions(const ActionHeadsSpec& heads, int B, const float* d_logits, uint64_t key,
                      uint64_t counter0, int32_t* d_actions, float* d_logp) const {
    check(appo_sample_actions_heads(h_, B, heads.n_heads(), heads.sizes.data(), d_logits, key,
                                    counter0, d_actions, d_logp));
  }

  // log_prob_and_entropy (policy.hpp:262-281): joint logp of `action`, summed
  // per-head entropy; out-of-range actions throw ContractError.
  std::pair<double, double> log_prob_and_entropy(const ActionHeadsSpec& heads,
                                                 std::span<const double> logits,
                                                 const FactoredAction& action) const {
    if (static_cast<int>(action.size()) != heads.n_heads())
      throw ContractError("action arity mismatch");
    if (static_cast<int>(logits.size()) != heads.logits_dim())
      throw ContractError("log_prob_and_entropy: logits size != heads.logits_dim()");
    const std::vector<float> lg(logits.begin(), logits.end());
    DeviceBuffer<float> dl(lg.size()), dlp(1), den(1);
    DeviceBuffer<int32_t> da(action.size());
    dl.upload(lg.data());
    da.upload(action.data());
    check(appo_logp_entropy_heads(h_, 1, heads.n_heads(), heads.sizes.data(), dl.get(), da.get(),
                                  dlp.get(), den.get()));
    sync();
    float lp = 0, en = 0;
    dlp.download(&lp);
    den.download(&en);
    return {static_cast<double>(lp), static_cast<double>(en)};
  }

  // optimizer_step (policy.hpp:431-455): global-norm clip + Adam on p (fp32 on
  // the device), t += 1, version += 1.  A non-finite gradient throws
  // NumericError and leaves p untouched, as the reference does.
  void optimizer_step(PolicyParams& p, std::span<const double> grads,
                      const AdamConfig& cfg) const {
    const size_t n = p.theta.size();
    if (grads.size() != n) throw ContractError("gradient size mismatch");
    if (p.adam.m.size() != n) p.adam.m.assign(n, 0.0);
    if (p.adam.v.size() != n) p.adam.v.assign(n, 0.0);
    auto f = [](const std::vector<double>& x) { return std::vector<float>(x.begin(), x.end()); };
    std::vector<float> th = f(p.theta), m = f(p.adam.m), v = f(p.adam.v);
    const std::vector<float> g(grads.begin(), grads.end());
    DeviceBuffer<float> dth(n), dm(n), dv(n), dg(n);
    dth.upload(th.data()); dm.upload(m.data()); dv.upload(v.data()); dg.upload(g.data());
    double norm = 0;
    check(appo_adam_step(h_, static_cast<int64_t>(n), dth.get(), dm.get(), dv.get(), dg.get(),
                         p.adam.t + 1, static_cast<float>(cfg.lr), static_cast<float>(cfg.beta1),
                         static_cast<float>(cfg.beta2), static_cast<float>(cfg.eps),
                         static_cast<float>(cfg.grad_clip), &norm));
    dth.download(th.data()); dm.download(m.data()); dv.download(v.data());
    p.theta.assign(th.begin(), th.end());
    p.adam.m.assign(m.begin(), m.end());
    p.adam.v.assign(v.begin(), v.end());
    p.adam.t += 1;
    p.version += 1;
  }

  // Batched device form: [n_traj x T] row-major, the learner gather order.
  void vtrace(int n_traj, int T, const float* d_rewards, const float* d_values,
              const float* d_boot, const float* d_tlogp, const float* d_blogp,
              const uint8_t* d_dones, const VTraceConfig& cfg, float* d_v, float* d_pg) const {
    check(appo_vtrace(h_, n_traj, T, d_rewards, d_values, d_boot, d_tlogp, d_blogp, d_dones,
                      static_cast<float>(cfg.gamma), static_cast<float>(cfg.rho_bar),
                      static_cast<float>(cfg.c_bar), d_v, d_pg, nullptr, nullptr));
  }

  // total_loss (offpolicy.hpp:146), device arrays of length n
  LossComponents total_loss(int n, const float* d_ratios, const float* d_adv,
                            const float* d_values, const float* d_vt, const float* d_ent,
                            double clip_low = 1.0 / 1.1, double clip_high = 1.1,
                            double value_coef = 0.5, double entropy_coef = 0.003) const {
    double o[4];
    check(appo_total_loss(h_, n, d_ratios, d_adv, d_values, d_vt, d_ent,
                          static_cast<float>(clip_low), static_cast<float>(clip_high),
                          static_cast<float>(value_coef), static_cast<float>(entropy_coef), o));
    return LossComponents{o[0], o[1], o[2], o[3]};
  }

  // Policy-worker batch inference (orchestrator.hpp:643-656).
  int64_t policy_forward(int B, const uint8_t* d_obs, const float* d_h_in, uint64_t counter,
                         int32_t* d_actions, float* d_logp, float* d_h_out, float* d_values,
                         float* d_logits = nullptr) const {
    int64_t version = -1;
    check(appo_policy_forward(h_, B, d_obs, d_h_in, counter, d_actions, d_logp, d_h_out,
                              d_values, d_logits, &version));
    return version;
  }

  // LearnerUnit::step (orchestrator.hpp:760-868) over layout-v2 slots.
  appo_step_out learner_step(const void* d_region, uint64_t slot_bytes,
                             std::span<const int32_t> slot_ids, const appo_hparams& hp) const {
    appo_step_out out{};
    check(appo_learner_step(h_, d_region, slot_bytes, slot_ids.data(),
                            static_cast<int>(slot_ids.size()), &hp, &out));
    return out;
  }

  // ParamStore::fetch (policy.hpp:498): newest parameters + version
  int64_t fetch(std::vector<float>& theta) const {
    theta.resize(static_cast<size_t>(appo_param_count(&desc_)));
    int64_t v = -1;
    check(appo_params_get(h_, theta.data(), &v));
    return v;
  }

  // save_checkpoint / load_checkpoint (policy.hpp:545-605): APPOCKP1 file
  void save_checkpoint(const std::string& path) const {
    check(appo_checkpoint_save(h_, path.c_str()));
  }
  void load_checkpoint(const std::string& path) const {
    check(appo_checkpoint_load(h_, path.c_str()));
  }

 private:
  appo_model_desc desc_{};
  appo_ctx* h_ = nullptr;
};

// Device slot FIFO (ready queue / free list, trajstore.hpp:293-331).
class SlotQueue {
 public:
  SlotQueue(int device, int32_t n_slots, int32_t capacity = 0, double timeout_s = 2.0) {
    check(appo_slotq_create(device, n_slots, capacity, timeout_s, &q_));
  }
  ~SlotQueue() { appo_slotq_destroy(q_); }
  SlotQueue(const SlotQueue&) = delete;
  SlotQueue& operator=(const SlotQueue&) = delete;
  appo_slotq* get() const { return q_; }
  void push(const Context& c, const int32_t* d_ids, int n) const {
    check(appo_slotq_push(c.get(), q_, d_ids, n));
  }
  void push_range(const Context& c, int32_t first, int n) const {
    check(appo_slotq_push_range(c.get(), q_, first, n));
  }
  void pop(const Context& c, int32_t* d_out, int n) const { check(appo_slotq_pop(c.get(), q_, d_out, n)); }
  // assemble_minibatch + LearnerUnit::step without the host seeing slot ids
  void learner_submit(const Context& c, const void* d_region, uint64_t slot_bytes,
                      const SlotQueue* free_q, int n_traj, const appo_hparams& hp) const {
    check(appo_learner_submit_queued(c.get(), d_region, slot_bytes, q_,
                                     free_q ? free_q->get() : nullptr, n_traj, &hp));
  }

 private:
  appo_slotq* q_ = nullptr;
};

// PbtController (runner.hpp:169-252) over learner contexts; copy_weights is
// appo_params_copy between the contexts (device to device).
class PbtController {
 public:
  PbtController(const appo_pbt_config& cfg, std::vector<Context*> learners, uint64_t rng_seed,
                const std::vector<appo_agent_meta>* init = nullptr)
      : learners_(learners.size()) {
    for (size_t i = 0; i < learners.size(); ++i) learners_[i] = learners[i]->get();
    check(appo_pbt_create(&cfg, static_cast<int>(learners.size()), rng_seed,
                          init ? init->data() : nullptr, &p_));
  }
  ~PbtController() { appo_pbt_destroy(p_); }
  PbtController(const PbtController&) = delete;
  PbtController& operator=(const PbtController&) = delete;
  void record(uint32_t policy, double value) const { check(appo_pbt_record(p_, policy, value)); }
  // PbtController::tick: the events of a PBT step, or nothing before the boundary
  std::vector<appo_pbt_event> tick(int64_t frames) {
    std::vector<appo_pbt_event> ev(static_cast<size_t>(appo_pbt_max_events(p_)));
    int n = 0, fired = 0;
    check(appo_pbt_tick(p_, frames, appo_pbt_copy_contexts, learners_.data(), ev.data(),
                        static_cast<int>(ev.size()), &n, &fired));
    ev.resize(fired ? static_cast<size_t>(n) : 0);
    return ev;
  }
  appo_agent_meta agent(int i) const {
    appo_agent_meta a{};
    check(appo_pbt_get_agent(p_, i, &a));
    return a;
  }

 private:
  std::vector<appo_ctx*> learners_;
  appo_pbt* p_ = nullptr;
};

inline appo_hparams default_hparams() {
  appo_hparams hp{};
  hp.lr = 1e-4f; hp.beta1 = 0.9f; hp.beta2 = 0.999f; hp.eps = 1e-6f; hp.grad_clip = 4.0f;
  hp.entropy_coef = 0.003f; hp.value_coef = 0.5f; hp.clip_low = 1.0f / 1.1f; hp.clip_high = 1.1f;
  hp.rho_bar = 1.0f; hp.c_bar = 1.0f; hp.gamma = 0.99f; hp.gae_lambda = 0.95f;
  hp.adv_source = 0; hp.normalize_adv = 0;
  return hp;
}

}  // namespace appo_b200
