// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Compiles the UNMODIFIED reference headers where they lie
// (/root/reference/proj/include, header-only C++20) into oracle/_ref/libappo_ref.so
// and exposes the hot-path functions with a C ABI so the tests can
//   (1) pin the oracle restatement (oracle/appo_oracle.c) against the real
//       reference, and
//   (2) generate the golden vectors committed under tests/golden/.
// bench.py --impl reference also times these functions as the reference CPU
// path.  No reference source is copied into this repository; this file only
// includes the headers and forwards arguments.
#include <chrono>
#include <cstring>
#include <sstream>
#include <random>
#include <vector>

#include "appo/offpolicy.hpp"
#include "appo/population.hpp"
#include "appo/policy.hpp"
#include "appo/trajstore.hpp"

using namespace appo;

namespace {
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ContractError&) {
    return 1;
  } catch (const ConfigError&) {
    return 2;
  } catch (const NumericError&) {
    return 3;
  } catch (...) {
    return 4;
  }
}
}  // namespace

extern "C" {

// offpolicy.hpp:61 vtrace
int ref_vtrace(int T, const double* r, const double* v, double boot, const double* tl,
               const double* bl, const std::uint8_t* d, double rho_bar, double c_bar, double gamma,
               double* v_out, double* pg_out, double* rho_out, double* c_out) {
  return guarded([&] {
    auto o = vtrace({r, (size_t)T}, {v, (size_t)T}, boot, {tl, (size_t)T}, {bl, (size_t)T},
                    {d, (size_t)T}, VTraceConfig{rho_bar, c_bar, gamma});
    std::memcpy(v_out, o.v.data(), sizeof(double) * T);
    std::memcpy(pg_out, o.pg_adv.data(), sizeof(double) * T);
    if (rho_out) std::memcpy(rho_out, o.rho.data(), sizeof(double) * T);
    if (c_out) std::memcpy(c_out, o.c.data(), sizeof(double) * T);
  });
}

// Batched [n_traj x T] driver used for CPU-baseline timing; trajectories
// [lo, hi) only, so the caller can partition across threads.
int ref_vtrace_range(int lo, int hi, int T, const double* r, const double* v, const double* boot,
                     const double* tl, const double* bl, const std::uint8_t* d, double rho_bar,
                     double c_bar, double gamma, double* v_out, double* pg_out) {
  return guarded([&] {
    for (int i = lo; i < hi; ++i) {
      const size_t o = (size_t)i * T;
      auto out = vtrace({r + o, (size_t)T}, {v + o, (size_t)T}, boot[i], {tl + o, (size_t)T},
                        {bl + o, (size_t)T}, {d + o, (size_t)T},
                        VTraceConfig{rho_bar, c_bar, gamma});
      std::memcpy(v_out + o, out.v.data(), sizeof(double) * T);
      std::memcpy(pg_out + o, out.pg_adv.data(), sizeof(double) * T);
    }
  });
}

// offpolicy.hpp:104 nstep_returns
void ref_nstep_returns(int T, const double* r, double boot, const std::uint8_t* d, double gamma,
                       double* ret) {
  auto o = nstep_returns({r, (size_t)T}, boot, {d, (size_t)T}, gamma);
  std::memcpy(ret, o.data(), sizeof(double) * T);
}

// offpolicy.hpp:117 / :124
double ref_ppo_objective(double ratio, double adv, double lo, double hi) {
  ClipConfig c{lo, hi};
  return ppo_clip_objective(ratio, adv, c);
}
double ref_ppo_dratio(double ratio, double adv, double lo, double hi) {
  ClipConfig c{lo, hi};
  return ppo_clip_dratio(ratio, adv, c);
}
double ref_importance_ratio(double t, double b) { return importance_ratio(t, b); }

// offpolicy.hpp:146 total_loss ; out = policy, value, entropy, total
int ref_total_loss(int n, const double* ratios, const double* adv, const double* values,
                   const double* vt, const double* ent, double lo, double hi, double value_coef,
                   double entropy_coef, double* out4) {
  return guarded([&] {
    LossConfig cfg;
    cfg.clip = ClipConfig{lo, hi};
    cfg.value_coef = value_coef;
    cfg.entropy_coef = entropy_coef;
    auto o = total_loss({ratios, (size_t)n}, {adv, (size_t)n}, {values, (size_t)n},
                        {vt, (size_t)n}, {ent, (size_t)n}, cfg);
    out4[0] = o.policy;
    out4[1] = o.value;
    out4[2] = o.entropy;
    out4[3] = o.total;
  });
}

// policy.hpp:214 softmax_heads / :262 log_prob_and_entropy, single head {n}
void ref_softmax(int n, const double* logits, double* probs) {
  ActionHeadsSpec h;
  h.sizes = {n};
  softmax_heads(h, {logits, (size_t)n}, {probs, (size_t)n});
}
int ref_log_prob_entropy(int n, const double* logits, int action, double* logp, double* ent) {
  return guarded([&] {
    ActionHeadsSpec h;
    h.sizes = {n};
    auto [lp, e] = log_prob_and_entropy(h, {logits, (size_t)n}, FactoredAction{action});
    *logp = lp;
    *ent = e;
  });
}

// policy.hpp:262 log_prob_and_entropy over factored heads {sizes[0..n_heads)}:
// B rows of logits [B][logits_dim] and actions [B][n_heads]
int ref_log_prob_entropy_heads(int n_heads, const int* sizes, int B, const double* logits,
                               const int* actions, double* logp, double* ent) {
  return guarded([&] {
    ActionHeadsSpec h;
    h.sizes.assign(sizes, sizes + n_heads);
    const int ld = h.logits_dim();
    for (int b = 0; b < B; ++b) {
      FactoredAction a(actions + (size_t)b * n_heads, actions + (size_t)(b + 1) * n_heads);
      auto [lp, e] = log_prob_and_entropy(h, {logits + (size_t)b * ld, (size_t)ld}, a);
      logp[b] = lp;
      ent[b] = e;
    }
  });
}

// policy.hpp:232 sample_action, `count` draws from one mt19937_64(seed)
void ref_sample_actions(int n, const double* logits, std::uint64_t seed, int count, int* actions,
                        double* logps) {
  ActionHeadsSpec h;
  h.sizes = {n};
  std::mt19937_64 rng(seed);
  for (int i = 0; i < count; ++i) {
    auto [a, lp] = sample_action(h, {logits, (size_t)n}, rng);
    actions[i] = a[0];
    logps[i] = lp;
  }
}

// policy.hpp:431 optimizer_step on a raw vector (shape-free: a ModelShape
// whose n_params() equals n is not needed because optimizer_step only uses
// theta/m/v sizes).
int ref_optimizer_step(long n, double* theta, double* m, double* v, const double* g, long* t,
                       double lr, double b1, double b2, double eps, double clip) {
  return guarded([&] {
    PolicyParams p;
    p.theta.assign(theta, theta + n);
    p.adam.m.assign(m, m + n);
    p.adam.v.assign(v, v + n);
    p.adam.t = *t;
    AdamConfig cfg;
    cfg.lr = lr;
    cfg.beta1 = b1;
    cfg.beta2 = b2;
    cfg.eps = eps;
    cfg.grad_clip = clip;
    optimizer_step(p, {g, (size_t)n}, cfg);
    std::memcpy(theta, p.theta.data(), sizeof(double) * n);
    std::memcpy(m, p.adam.m.data(), sizeof(double) * n);
    std::memcpy(v, p.adam.v.data(), sizeof(double) * n);
    *t = p.adam.t;
  });
}

// trajstore.hpp:62 traj_layout::Offsets (reference f64 element types)
void ref_slot_offsets(std::uint32_t T, std::uint32_t obs_dim, std::uint32_t hidden_dim,
                      std::uint32_t n_heads, std::uint64_t* out) {
  TrajectoryShape s{T, obs_dim, hidden_dim, n_heads};
  traj_layout::Offsets o(s);
  const std::size_t v[10] = {o.obs,      o.hidden,   o.actions,  o.rewards,     o.logp,
                             o.dones,    o.versions, o.boot_obs, o.boot_hidden, o.total};
  for (int i = 0; i < 10; ++i) out[i] = v[i];
}

// acceptance.cpp:42-56 / test_offpolicy.cpp:20-34 instance generator,
// reproduced bit-for-bit by driving the same std distributions from the
// same engine.  Writes T values per array; `state` carries the engine.
void* ref_rng_new(std::uint64_t seed) { return new std::mt19937_64(seed); }
void ref_rng_free(void* p) { delete static_cast<std::mt19937_64*>(p); }
void ref_random_instance(void* state, int T, double done_prob, double* r, double* v, double* tl,
                         double* bl, std::uint8_t* d, double* boot) {
  auto& rng = *static_cast<std::mt19937_64*>(state);
  std::uniform_real_distribution<double> ur(-1.0, 1.0);
  std::uniform_real_distribution<double> lp(-2.5, -0.1);
  std::bernoulli_distribution bd(done_prob);
  for (int t = 0; t < T; ++t) {
    r[t] = ur(rng);
    v[t] = ur(rng);
    tl[t] = lp(rng);
    bl[t] = lp(rng);
    d[t] = bd(rng) ? 1 : 0;
  }
  *boot = ur(rng);
}

std::uint64_t ref_splitmix64(std::uint64_t x) { return splitmix64(x); }
std::uint64_t ref_derive_seed(std::uint64_t s, std::uint64_t k) { return derive_seed(s, k); }
std::uint64_t ref_fnv1a64(const void* p, std::size_t n) { return fnv1a64(p, n); }

// policy.hpp:545-564 save_checkpoint of an init_params MLP (format-parity
// fixture: the library's APPOCKP1 reader must read the reference's own files);
// returns n_params, or -1 on error.  theta / m / v / version / t are set to
// recognisable values first.
long long ref_save_checkpoint_mlp(const char* path, int obs_dim, int trunk_hidden,
                                  const int* heads, int n_heads, std::uint64_t seed,
                                  long long version, long long t) {
  long long n = -1;
  guarded([&] {
    ModelShape s;
    s.obs_dim = obs_dim;
    s.trunk_hidden = trunk_hidden;
    s.heads.sizes.assign(heads, heads + n_heads);
    PolicyParams p = init_params(s, seed);
    for (std::size_t i = 0; i < p.theta.size(); ++i) {
      p.adam.m[i] = 0.5 * p.theta[i];
      p.adam.v[i] = p.theta[i] * p.theta[i];
    }
    p.version = version;
    p.adam.t = t;
    save_checkpoint(path, p);
    n = (long long)p.theta.size();
  });
  return n;
}
std::uint64_t ref_spec_hash_mlp(int obs_dim, int hidden_dim, int trunk_hidden, const int* heads,
                                int n_heads) {
  ModelShape s;
  s.obs_dim = obs_dim;
  s.hidden_dim = hidden_dim;
  s.trunk_hidden = trunk_hidden;
  s.heads.sizes.assign(heads, heads + n_heads);
  return s.spec_hash();
}

// compute_gradients (policy.hpp:302-428) with injected logits and values: for
// each sample an MLP whose head / value weights are zero and whose biases ARE
// the sample's logits and value (obs_dim 1, trunk 1), run on a batch of one,
// so the head-bias gradient is exactly the reference's dlogits row and the
// value-bias gradient its dL/dV (policy.hpp:349-372,357).  Rows are scaled by
// 1/n (the batch mean, policy.hpp:318); loss4 = {policy, value, entropy,
// total} and *mean_ratio are the batch means of the per-sample results.
int ref_ppo_grads_injected(int n, int A, const double* logits, const double* values,
                           const int* actions, const double* blogp, const double* adv,
                           const double* vt, double lo, double hi, double value_coef,
                           double entropy_coef, double* dlogits, double* dv, double* loss4,
                           double* mean_ratio) {
  return guarded([&] {
    ModelShape s;
    s.obs_dim = 1;
    s.trunk_hidden = 1;
    s.heads.sizes = {A};
    ParamLayout L(s);
    PolicyParams p;
    p.shape = s;
    LossConfig cfg;
    cfg.clip = ClipConfig{lo, hi};
    cfg.value_coef = value_coef;
    cfg.entropy_coef = entropy_coef;
    double acc[5] = {0, 0, 0, 0, 0};
    for (int i = 0; i < n; ++i) {
      p.theta.assign(L.total, 0.0);
      for (int k = 0; k < A; ++k) p.theta[L.bh + k] = logits[(size_t)i * A + k];
      p.theta[L.bv] = values[i];
      SampleBatch b;
      b.batch = 1;
      b.obs = {0.0};
      b.actions = {actions[i]};
      b.behavior_logp = {blogp[i]};
      b.advantages = {adv[i]};
      b.v_targets = {vt[i]};
      GradientResult g = compute_gradients(p, b, cfg);
      for (int k = 0; k < A; ++k) dlogits[(size_t)i * A + k] = g.grad[L.bh + k] / n;
      dv[i] = g.grad[L.bv] / n;
      acc[0] += g.loss.policy;
      acc[1] += g.loss.value;
      acc[2] += g.loss.entropy;
      acc[4] += g.mean_ratio;
    }
    loss4[0] = acc[0] / n;
    loss4[1] = acc[1] / n;
    loss4[2] = acc[2] / n;
    loss4[3] = loss4[0] + loss4[1] - entropy_coef * loss4[2];
    *mean_ratio = acc[4] / n;
  });
}

// The reference's own learner math at the Doom input (SURVEY §8(d) CPU plan):
// its MLP stand-in (ModelShape{obs_dim, 0, trunk, {A}}, policy.hpp:39-59) timed
// through forward_batch (policy.hpp:165-200), compute_gradients (:302-428) and
// optimizer_step (:431-455) on one thread, steady_clock, best of `reps`.
// out[0] = forward s/sample, out[1] = compute_gradients s/sample,
// out[2] = optimizer_step s/call, out[3] = n_params.
int ref_mlp_stand_in_time(int obs_dim, int trunk, int A, int B, int reps, double* out) {
  return guarded([&] {
    ModelShape s;
    s.obs_dim = obs_dim;
    s.trunk_hidden = trunk;
    s.heads.sizes = {A};
    PolicyParams p = init_params(s, 1);
    std::mt19937_64 rng(3);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    SampleBatch b;
    b.batch = B;
    b.obs.resize(static_cast<std::size_t>(B) * obs_dim);
    for (auto& x : b.obs) x = u(rng);
    for (int i = 0; i < B; ++i) {
      b.actions.push_back(static_cast<std::int32_t>(rng() % A));
      b.behavior_logp.push_back(-std::log(static_cast<double>(A)));
      b.advantages.push_back(u(rng) - 0.5);
      b.v_targets.push_back(u(rng) - 0.5);
    }
    LossConfig cfg;
    AdamConfig adam;
    double best[3] = {1e30, 1e30, 1e30};
    for (int r = 0; r < reps; ++r) {
      ForwardCache cache;
      auto t0 = std::chrono::steady_clock::now();
      forward_batch(p, b.obs, B, cache);
      auto t1 = std::chrono::steady_clock::now();
      GradientResult g = compute_gradients(p, b, cfg);
      auto t2 = std::chrono::steady_clock::now();
      optimizer_step(p, g.grad, adam);
      auto t3 = std::chrono::steady_clock::now();
      best[0] = std::min(best[0], std::chrono::duration<double>(t1 - t0).count() / B);
      best[1] = std::min(best[1], std::chrono::duration<double>(t2 - t1).count() / B);
      best[2] = std::min(best[2], std::chrono::duration<double>(t3 - t2).count());
    }
    out[0] = best[0];
    out[1] = best[1];
    out[2] = best[2];
    out[3] = static_cast<double>(p.theta.size());
  });
}

// pbt_step (population.hpp:131-186) over `periods` periods of the synthetic
// score schedule of acceptance.cpp's PBT criterion (P agents, reward weights
// {1.0, 0.2, -0.5}, every third period compressed below the threshold);
// writes the CSV decision log (with header) and returns its length, or -1
// when cap is too small.  threshold < 0: no exchange gate.
long ref_pbt_log(int P, std::uint64_t seed, int periods, double threshold, char* buf,
                 std::size_t cap) {
  PopulationConfig cfg;
  cfg.P = static_cast<std::uint32_t>(P);
  if (threshold >= 0.0) cfg.exchange_threshold = threshold;
  std::mt19937_64 rng(seed);
  std::vector<AgentMeta> agents(P);
  for (int i = 0; i < P; ++i) {
    agents[i].policy_id = static_cast<std::uint32_t>(i);
    agents[i].reward_weights = {1.0, 0.2, -0.5};
  }
  std::vector<PbtEvent> all;
  for (int period = 0; period < periods; ++period) {
    std::vector<std::optional<double>> scores(P);
    for (int i = 0; i < P; ++i) {
      const double base = ((i * 13 + period * 7) % 23) / 23.0;
      scores[i] = (period % 3 == 2) ? 0.5 + 0.2 * base : base;
    }
    auto ev = pbt_step(agents, scores, cfg, rng, period * 5000000LL,
                       [](std::uint32_t, std::uint32_t) {});
    all.insert(all.end(), ev.begin(), ev.end());
  }
  std::ostringstream log;
  log << "frame,agent,event,field,old,new\n";
  for (const auto& e : all)
    log << e.frame << ',' << e.agent << ',' << e.event << ',' << e.field << ',' << e.old_value
        << ',' << e.new_value << "\n";
  const std::string t = log.str();
  if (t.size() + 1 > cap) return -1;
  std::memcpy(buf, t.c_str(), t.size() + 1);
  return static_cast<long>(t.size());
}

// dump_trajectory (trajstore.hpp:335-359) of one slot filled through the
// reference's own TrajectorySlotView::begin / write_step / set_bootstrap
// (trajstore.hpp:100-215) from the given arrays; n_heads = 1.  Returns the
// guarded status (the write_step contracts apply).
int ref_dump_trajectory(std::uint32_t T, std::uint32_t obs_dim, std::uint32_t hidden_dim,
                        const double* obs, const double* hidden, const std::int32_t* actions,
                        const double* rewards, const double* logp, const std::uint8_t* dones,
                        const std::int64_t* versions, const double* boot_obs,
                        const double* boot_hidden, std::uint32_t env, std::uint32_t worker,
                        std::uint32_t policy, const char* path) {
  return guarded([&] {
    TrajectoryStore store(TrajectoryShape{T, obs_dim, hidden_dim, 1}, 1);
    auto v = store.view(0);
    v.begin(env, worker, policy, 0);
    for (std::uint32_t t = 0; t < T; ++t) {
      StepRecord rec;
      rec.obs.assign(obs + std::size_t{t} * obs_dim, obs + std::size_t{t + 1} * obs_dim);
      rec.hidden.assign(hidden + std::size_t{t} * hidden_dim,
                        hidden + std::size_t{t + 1} * hidden_dim);
      rec.action = {actions[t]};
      rec.reward = rewards[t];
      rec.behavior_logp = logp[t];
      rec.done = dones[t] != 0;
      rec.policy_version = versions[t];
      v.write_step(t, rec);
    }
    v.set_bootstrap(std::span<const double>(boot_obs, obs_dim),
                    std::span<const double>(boot_hidden, hidden_dim));
    dump_trajectory(v, path);
  });
}

}  // extern "C"
