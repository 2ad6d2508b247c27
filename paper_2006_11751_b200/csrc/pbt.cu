// Population-based training controller over per-GPU learners: the PBT step
// (population.hpp:131-186) and the PbtController around it (runner.hpp:169-252:
// per-policy score windows, period boundaries, hyper-parameter hand-back).
// Host code -- a few hundred scalar decisions every pbt_period frames; the
// weight exchange it triggers is a device-to-device copy (appo_params_copy,
// peer copy over NVLink between GPUs).
//
// Bit-compatibility with the reference: the decision stream comes from the
// same std::mt19937_64 draws in the same order (one uniform_real draw per
// mutable field of the bottom cohort, one coin per applied mutation, one
// index per exchange), so a run seeded like the reference reproduces its
// decision log byte for byte (acceptance.cpp:573-662 freezes that log's hash).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "appo_common.cuh"

using namespace appo_b200;

#define TRY_OK(x)                  \
  do {                             \
    const int _st = (x);           \
    if (_st != APPO_OK) return _st; \
  } while (0)

struct appo_pbt {
  appo_pbt_config cfg{};
  std::mt19937_64 rng;
  std::vector<appo_agent_meta> agents;
  std::vector<std::deque<double>> windows;
  int64_t next_boundary = 0;
};

namespace {

constexpr const char* kEventNames[3] = {"mutate", "exchange", "skip-threshold"};

int validate(const appo_pbt_config& c) {
  auto frac = [](double f) { return f >= 0.0 && f <= 1.0; };
  APPO_REQUIRE(frac(c.mutate_fraction) && frac(c.mutation_rate) && frac(c.replace_fraction),
               APPO_ERR_CONFIG, "population fractions must lie in [0,1]");
  APPO_REQUIRE(c.mutation_factor > 1.0, APPO_ERR_CONFIG, "mutation factor must exceed 1");
  return APPO_OK;
}

// Mutable hyper-parameters in the reference's field order
// (AgentMeta::mutable_fields, population.hpp:48-57).
int mutable_fields(appo_agent_meta& a, double** vals, std::string* names) {
  int n = 0;
  vals[n] = &a.learning_rate; names[n++] = "learning_rate";
  vals[n] = &a.entropy_coef; names[n++] = "entropy_coef";
  vals[n] = &a.adam_beta1; names[n++] = "adam_beta1";
  for (int i = 0; i < a.n_reward_weights; ++i) {
    vals[n] = &a.reward_weights[i];
    names[n++] = "reward_weight_" + std::to_string(i);
  }
  return n;
}

appo_pbt_event make_event(int64_t frame, uint32_t agent, int kind, const std::string& field,
                          double old_v, double new_v) {
  appo_pbt_event e{};
  e.frame = frame;
  e.agent = agent;
  e.event = kind;
  std::snprintf(e.field, sizeof(e.field), "%s", field.c_str());
  e.old_value = old_v;
  e.new_value = new_v;
  return e;
}

struct CopyCb {
  appo_pbt_copy_fn fn;
  void* user;
};

// population.hpp:131-186: rank (best first, ties by policy id), mutate the
// bottom floor(mutate_fraction*P), replace the worst floor(replace_fraction*P)
// from the top ceil(replace_fraction*P) unless within exchange_threshold of
// the best.  Unscored agents sit the step out.
int pbt_step_impl(appo_pbt* s, const double* scores, const uint8_t* has, int64_t frame,
                  CopyCb cb, std::vector<appo_pbt_event>& ev) {
  TRY_OK(validate(s->cfg));
  const uint32_t P = (uint32_t)s->agents.size();
  std::vector<uint32_t> ranked;
  for (uint32_t i = 0; i < P; ++i)
    if (has[i]) ranked.push_back(i);
  std::sort(ranked.begin(), ranked.end(), [&](uint32_t a, uint32_t b) {
    if (scores[a] != scores[b]) return scores[a] > scores[b];
    return s->agents[a].policy_id < s->agents[b].policy_id;
  });
  if (ranked.empty()) return APPO_OK;
  const double n = (double)ranked.size();
  const size_t n_mutate = (size_t)std::floor(s->cfg.mutate_fraction * n);
  const size_t n_replace = (size_t)std::floor(s->cfg.replace_fraction * n);
  const size_t n_top = (size_t)std::ceil(s->cfg.replace_fraction * n);
  const double best = scores[ranked.front()];

  std::uniform_real_distribution<double> unit(0.0, 1.0);
  for (size_t r = ranked.size() - n_mutate; r < ranked.size(); ++r) {
    appo_agent_meta& a = s->agents[ranked[r]];
    double* vals[3 + APPO_PBT_MAX_REWARD_WEIGHTS];
    std::string names[3 + APPO_PBT_MAX_REWARD_WEIGHTS];
    const int nf = mutable_fields(a, vals, names);
    for (int f = 0; f < nf; ++f) {
      if (unit(s->rng) >= s->cfg.mutation_rate) continue;
      bool up = (s->rng() & 1) == 0;
      // adam_beta1 must stay below 1: reflect an up-move that would cross it
      if (f == 2 && up && *vals[f] * s->cfg.mutation_factor >= 1.0) up = false;
      const double before = *vals[f];
      *vals[f] = up ? before * s->cfg.mutation_factor : before / s->cfg.mutation_factor;
      ev.push_back(make_event(frame, a.policy_id, 0, names[f], before, *vals[f]));
    }
  }
  for (size_t r = ranked.size() - n_replace; r < ranked.size(); ++r) {
    appo_agent_meta& a = s->agents[ranked[r]];
    const double sc = scores[ranked[r]];
    if (s->cfg.has_exchange_threshold && best - sc < s->cfg.exchange_threshold) {
      ev.push_back(make_event(frame, a.policy_id, 2, "score", sc, best));
      continue;
    }
    const uint32_t src_rank = (uint32_t)(s->rng() % n_top);
    const appo_agent_meta src = s->agents[ranked[src_rank]];
    // replace_fraction > 0.5 lets the top cohort overlap the replaced one, so
    // src may be dst: the reference's copy_weights is then a harmless
    // self-copy and the exchange is still logged -- no callback here
    if (cb.fn && src.policy_id != a.policy_id) {
      const int st = cb.fn(cb.user, a.policy_id, src.policy_id);
      if (st != APPO_OK) return st;
    }
    const uint32_t dst_id = a.policy_id;
    a = src;
    a.policy_id = dst_id;
    ev.push_back(make_event(frame, dst_id, 1, "weights", (double)src.policy_id, (double)dst_id));
  }
  return APPO_OK;
}

int emit(const std::vector<appo_pbt_event>& ev, appo_pbt_event* out, int max_ev, int* n_ev) {
  if (n_ev) *n_ev = (int)ev.size();
  if (out) {
    APPO_REQUIRE((int)ev.size() <= max_ev, APPO_ERR_CONTRACT, "pbt: event buffer too small");
    std::copy(ev.begin(), ev.end(), out);
  }
  return APPO_OK;
}

}  // namespace

extern "C" {

int appo_pbt_create(const appo_pbt_config* cfg, int P, uint64_t rng_seed,
                    const appo_agent_meta* init, appo_pbt** out) {
  APPO_REQUIRE(cfg && out && P >= 1, APPO_ERR_CONTRACT, "pbt_create: bad arguments");
  *out = nullptr;
  TRY_OK(validate(*cfg));
  APPO_REQUIRE(cfg->window >= 1, APPO_ERR_CONFIG, "pbt_create: score window must be >= 1");
  auto* s = new appo_pbt;
  s->cfg = *cfg;
  s->rng.seed(rng_seed);
  s->agents.resize(P);
  for (int i = 0; i < P; ++i) {
    appo_agent_meta a{};
    if (init) {
      a = init[i];
    } else {
      a.learning_rate = 1e-4;
      a.entropy_coef = 0.003;
      a.adam_beta1 = 0.9;
    }
    a.policy_id = (uint32_t)i;
    if (a.n_reward_weights < 0 || a.n_reward_weights > APPO_PBT_MAX_REWARD_WEIGHTS) {
      delete s;
      set_error("pbt_create: n_reward_weights outside [0, APPO_PBT_MAX_REWARD_WEIGHTS]");
      return APPO_ERR_CONTRACT;
    }
    s->agents[i] = a;
  }
  s->windows.resize(P);
  s->next_boundary = cfg->pbt_period;
  *out = s;
  return APPO_OK;
}

int appo_pbt_destroy(appo_pbt* s) {
  delete s;
  return APPO_OK;
}

uint64_t appo_pbt_controller_seed(uint64_t pipeline_seed) {
  return host_derive_seed(pipeline_seed, 0x9B7);  // runner.hpp:172
}

int appo_pbt_record(appo_pbt* s, uint32_t policy, double value) {
  APPO_REQUIRE(s != nullptr, APPO_ERR_CONTRACT, "pbt: null controller");
  if (policy >= s->windows.size()) return APPO_OK;  // foreign policy ids are ignored
  auto& w = s->windows[policy];
  w.push_back(value);
  if ((int64_t)w.size() > s->cfg.window) w.pop_front();
  return APPO_OK;
}

int appo_pbt_score(appo_pbt* s, uint32_t policy, double* score, int* has) {
  APPO_REQUIRE(s && policy < s->windows.size(), APPO_ERR_CONTRACT, "pbt_score: bad policy");
  const auto& w = s->windows[policy];
  double sum = 0.0;
  for (double v : w) sum += v;
  if (has) *has = w.empty() ? 0 : 1;
  if (score) *score = w.empty() ? 0.0 : sum / (double)w.size();
  return APPO_OK;
}

int appo_pbt_step(appo_pbt* s, const double* scores, const uint8_t* has_score, int64_t frame,
                  appo_pbt_copy_fn copy_weights, void* user, appo_pbt_event* events,
                  int max_events, int* n_events) {
  APPO_REQUIRE(s && scores && has_score, APPO_ERR_CONTRACT, "pbt_step: bad arguments");
  std::vector<appo_pbt_event> ev;
  const int st = pbt_step_impl(s, scores, has_score, frame, CopyCb{copy_weights, user}, ev);
  if (st != APPO_OK) return st;
  return emit(ev, events, max_events, n_events);
}

int appo_pbt_tick(appo_pbt* s, int64_t frames, appo_pbt_copy_fn copy_weights, void* user,
                  appo_pbt_event* events, int max_events, int* n_events, int* fired) {
  APPO_REQUIRE(s != nullptr, APPO_ERR_CONTRACT, "pbt: null controller");
  if (fired) *fired = 0;
  if (n_events) *n_events = 0;
  if (s->agents.size() < 2 || s->cfg.pbt_period <= 0 || frames < s->next_boundary)
    return APPO_OK;
  s->next_boundary += s->cfg.pbt_period;
  const size_t P = s->agents.size();
  std::vector<double> sc(P);
  std::vector<uint8_t> has(P);
  for (size_t i = 0; i < P; ++i) {
    int h = 0;
    appo_pbt_score(s, (uint32_t)i, &sc[i], &h);
    has[i] = (uint8_t)h;
  }
  if (fired) *fired = 1;
  return appo_pbt_step(s, sc.data(), has.data(), frames, copy_weights, user, events, max_events,
                       n_events);
}

int appo_pbt_get_agent(appo_pbt* s, int i, appo_agent_meta* out) {
  APPO_REQUIRE(s && out && i >= 0 && i < (int)s->agents.size(), APPO_ERR_CONTRACT,
               "pbt_get_agent: bad index");
  *out = s->agents[i];
  return APPO_OK;
}

int appo_pbt_max_events(appo_pbt* s) {
  if (!s) return 0;
  int mx = 0;
  for (const auto& a : s->agents) mx = std::max(mx, 3 + a.n_reward_weights);
  return (int)s->agents.size() * (mx + 1);
}

// append_pbt_events_csv (population.hpp:110-118): "frame,agent,event,field,old,new"
// with the iostream default number format.
int appo_pbt_format_events(const appo_pbt_event* ev, int n, int header, char* buf, uint64_t cap,
                           uint64_t* len) {
  APPO_REQUIRE(n >= 0 && (n == 0 || ev), APPO_ERR_CONTRACT, "pbt_format_events: bad arguments");
  std::ostringstream o;
  if (header) o << "frame,agent,event,field,old,new\n";
  for (int i = 0; i < n; ++i) {
    APPO_REQUIRE(ev[i].event >= 0 && ev[i].event <= 2, APPO_ERR_CONTRACT,
                 "pbt_format_events: unknown event kind");
    o << ev[i].frame << ',' << ev[i].agent << ',' << kEventNames[ev[i].event] << ','
      << ev[i].field << ',' << ev[i].old_value << ',' << ev[i].new_value << '\n';
  }
  const std::string t = o.str();
  if (len) *len = t.size();
  if (buf) {
    APPO_REQUIRE(t.size() < cap, APPO_ERR_CONTRACT, "pbt_format_events: buffer too small");
    std::memcpy(buf, t.c_str(), t.size() + 1);
  }
  return APPO_OK;
}

// copy_weights over an array of learner contexts: user = appo_ctx*[P]
int appo_pbt_copy_contexts(void* user, uint32_t dst, uint32_t src) {
  appo_ctx** learners = static_cast<appo_ctx**>(user);
  if (dst == src || learners[dst] == learners[src]) return APPO_OK;  // self-copy: no-op
  return appo_params_copy(learners[dst], learners[src]);
}

}  // extern "C"
