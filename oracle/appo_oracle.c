/*
 * appo_oracle.c -- CPU restatement (fp64) of the APPO hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2006_11751_b200/,
 * include/) links or calls this file.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg load it, and only as the
 * checker or the timed CPU baseline, never as the measured product path.
 *
 * Every function cites the reference file:line it restates.  Reference =
 * /root/reference/proj/include/appo/*.hpp (header-only C++20).
 *
 * Parity status:
 *   - vtrace / nstep / ppo clip / total_loss / heads / sampling semantics /
 *     Adam+clip / slot layout: PINNED -- checked against the reference compiled
 *     here (oracle/_ref, built by oracle/Makefile) and against golden vectors
 *     generated from it (tests/golden/).
 *   - convnet_simple encoder, GRU-512, BPTT, GAE(lambda<1), u8/255 input,
 *     the counter-based sampler RNG, and the synthetic observation generator:
 *     the reference has no code for these.  They
 *     are "parity unpinned" against the reference; the restatement here is
 *     cross-checked against torch fp64 autograd in tests/test_oracle_torch.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_CONTRACT 1
#define ORC_CONFIG 2
#define ORC_NUMERIC 3

/* ------------------------------------------------------------------ hashing */

/* common.hpp:53-58 */
uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* common.hpp:60-62 */
uint64_t orc_derive_seed(uint64_t seed, uint64_t stream) {
  return orc_splitmix64(seed ^ orc_splitmix64(stream + 1));
}

/* common.hpp:66-74 */
uint64_t orc_fnv1a64(const void* data, size_t n) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 1469598103934665603ULL;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ULL;
  }
  return h;
}

/* Counter-based uniform in [0,1) used by the device sampler (the reference
 * draws from std::mt19937_64, policy.hpp:239; a stateful engine cannot be
 * shared by 16k concurrent envs, so the product keys one draw per (env, step)).
 * 53 high bits of splitmix64(key ^ splitmix64(counter)). */
double orc_uniform(uint64_t key, uint64_t counter) {
  uint64_t h = orc_splitmix64(key ^ orc_splitmix64(counter));
  return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

/* -------------------------------------------------------------- off-policy */

static int finite(double x) { return isfinite(x); }

/* offpolicy.hpp:50-54 */
double orc_importance_ratio(double target_logp, double behavior_logp) {
  double d = target_logp - behavior_logp;
  if (d < -20.0) d = -20.0;
  if (d > 20.0) d = 20.0;
  return exp(d);
}

/* offpolicy.hpp:23-27 */
int orc_vtrace_validate(double rho_bar, double c_bar, double gamma) {
  if (!(rho_bar >= c_bar && c_bar > 0.0)) return ORC_CONFIG;
  if (!(gamma > 0.0 && gamma <= 1.0)) return ORC_CONFIG;
  return ORC_OK;
}

/* offpolicy.hpp:61-100: backward recursion over one trajectory. */
int orc_vtrace(int T, const double* rewards, const double* values, double bootstrap,
               const double* tlogp, const double* blogp, const uint8_t* dones, double rho_bar,
               double c_bar, double gamma, double* v_out, double* pg_out, double* rho_out,
               double* c_out) {
  int st = orc_vtrace_validate(rho_bar, c_bar, gamma);
  if (st) return st;
  for (int t = 0; t < T; ++t)
    if (!finite(rewards[t]) || !finite(values[t]) || !finite(tlogp[t]) || !finite(blogp[t]))
      return ORC_NUMERIC;
  if (!finite(bootstrap)) return ORC_NUMERIC;
  double v_next = bootstrap, value_next = bootstrap;
  for (int i = T - 1; i >= 0; --i) {
    const double ratio = orc_importance_ratio(tlogp[i], blogp[i]);
    const double rho = ratio < rho_bar ? ratio : rho_bar;
    const double c = ratio < c_bar ? ratio : c_bar;
    const double disc = dones[i] ? 0.0 : gamma;
    const double delta = rho * (rewards[i] + disc * value_next - values[i]);
    const double v = values[i] + delta + disc * c * (v_next - value_next);
    v_out[i] = v;
    pg_out[i] = rho * (rewards[i] + disc * v_next - values[i]);
    if (rho_out) rho_out[i] = rho;
    if (c_out) c_out[i] = c;
    v_next = v;
    value_next = values[i];
  }
  return ORC_OK;
}

/* Batched form over [n_traj x T] row-major (the learner gather order
 * s = i*T + t, orchestrator.hpp:781-795). */
int orc_vtrace_batch(int n_traj, int T, const double* rewards, const double* values,
                     const double* boot, const double* tlogp, const double* blogp,
                     const uint8_t* dones, double rho_bar, double c_bar, double gamma, double* v,
                     double* pg, double* rho, double* c) {
  for (int i = 0; i < n_traj; ++i) {
    const size_t o = (size_t)i * T;
    int st = orc_vtrace(T, rewards + o, values + o, boot[i], tlogp + o, blogp + o, dones + o,
                        rho_bar, c_bar, gamma, v + o, pg + o, rho ? rho + o : 0, c ? c + o : 0);
    if (st) return st;
  }
  return ORC_OK;
}

/* offpolicy.hpp:104-114 */
void orc_nstep_returns(int T, const double* rewards, double bootstrap, const uint8_t* dones,
                       double gamma, double* ret) {
  double acc = bootstrap;
  for (int i = T - 1; i >= 0; --i) {
    const double disc = dones[i] ? 0.0 : gamma;
    acc = rewards[i] + disc * acc;
    ret[i] = acc;
  }
}

/* GAE (not in the reference, SPEC.md:358 marks it out of scope there; it is in
 * the north star).  A_t = delta_t + gamma*lambda*(1-done_t)*A_{t+1},
 * delta_t = r_t + gamma*(1-done_t)*V_{t+1} - V_t, V_T := bootstrap;
 * ret_t = A_t + V_t.  With lambda = 1 A_t telescopes to nstep_returns - V
 * (the reference's NStep advantage, orchestrator.hpp:831-833). */
void orc_gae(int T, const double* rewards, const double* values, double bootstrap,
             const uint8_t* dones, double gamma, double lambda, double* adv, double* ret) {
  double a_next = 0.0, value_next = bootstrap;
  for (int i = T - 1; i >= 0; --i) {
    const double disc = dones[i] ? 0.0 : gamma;
    const double delta = rewards[i] + disc * value_next - values[i];
    const double a = delta + disc * lambda * a_next;
    adv[i] = a;
    if (ret) ret[i] = a + values[i];
    a_next = a;
    value_next = values[i];
  }
}

/* offpolicy.hpp:117-120 */
double orc_ppo_objective(double ratio, double adv, double lo, double hi) {
  double cl = ratio < lo ? lo : (ratio > hi ? hi : ratio);
  double a = ratio * adv, b = cl * adv;
  return a < b ? a : b;
}

/* offpolicy.hpp:124-128: unclipped branch wins ties */
double orc_ppo_dratio(double ratio, double adv, double lo, double hi) {
  double cl = ratio < lo ? lo : (ratio > hi ? hi : ratio);
  return (ratio * adv <= cl * adv) ? adv : 0.0;
}

/* offpolicy.hpp:146-168; out = {policy, value, entropy, total} */
int orc_total_loss(int n, const double* ratios, const double* adv, const double* values,
                   const double* vt, const double* ent, double lo, double hi, double value_coef,
                   double entropy_coef, double* out4) {
  double p = 0, v = 0, e = 0;
  for (int i = 0; i < n; ++i) {
    p -= orc_ppo_objective(ratios[i], adv[i], lo, hi);
    double ve = values[i] - vt[i];
    v += ve * ve;
    e += ent[i];
  }
  if (n > 0) {
    p /= n;
    v = value_coef * v / n;
    e /= n;
  }
  out4[0] = p;
  out4[1] = v;
  out4[2] = e;
  out4[3] = p + v - entropy_coef * e;
  return finite(out4[3]) ? ORC_OK : ORC_NUMERIC;
}

/* ------------------------------------------------------------------ heads */

/* policy.hpp:214-228, one head */
void orc_softmax(int n, const double* logits, double* probs) {
  double mx = logits[0];
  for (int i = 1; i < n; ++i) mx = logits[i] > mx ? logits[i] : mx;
  double z = 0;
  for (int i = 0; i < n; ++i) {
    probs[i] = exp(logits[i] - mx);
    z += probs[i];
  }
  for (int i = 0; i < n; ++i) probs[i] /= z;
}

/* policy.hpp:232-258 for heads {n}: inverse CDF with first i where u < cum,
 * fallback n-1; logp = log(max(p, 1e-300)). */
int orc_sample(int n, const double* logits, double u, double* logp) {
  double probs[64];
  orc_softmax(n, logits, probs);
  double cum = 0;
  int chosen = n - 1;
  for (int i = 0; i < n; ++i) {
    cum += probs[i];
    if (u < cum) {
      chosen = i;
      break;
    }
  }
  double p = probs[chosen] > 1e-300 ? probs[chosen] : 1e-300;
  *logp = log(p);
  return chosen;
}

/* policy.hpp:262-281 for heads {n} */
int orc_logp_entropy(int n, const double* logits, int action, double* logp, double* entropy) {
  if (action < 0 || action >= n) return ORC_CONTRACT;
  double probs[64];
  orc_softmax(n, logits, probs);
  double p = probs[action] > 1e-300 ? probs[action] : 1e-300;
  *logp = log(p);
  double h = 0;
  for (int i = 0; i < n; ++i)
    if (probs[i] > 0) h -= probs[i] * log(probs[i]);
  *entropy = h;
  return ORC_OK;
}

/* -------------------------------------------------------------- optimizer */

/* policy.hpp:431-455: finite check, global-norm clip, Adam, t += 1. */
int orc_adam_step(long n, double* theta, double* m, double* v, const double* g, long* t,
                  double lr, double b1, double b2, double eps, double clip) {
  double sq = 0;
  for (long i = 0; i < n; ++i) {
    if (!finite(g[i])) return ORC_NUMERIC;
    sq += g[i] * g[i];
  }
  const double norm = sqrt(sq);
  double scale = 1.0;
  if (clip > 0.0 && norm > clip) scale = clip / norm;
  *t += 1;
  const double bc1 = 1.0 - pow(b1, (double)*t);
  const double bc2 = 1.0 - pow(b2, (double)*t);
  for (long i = 0; i < n; ++i) {
    const double gi = g[i] * scale;
    m[i] = b1 * m[i] + (1.0 - b1) * gi;
    v[i] = b2 * v[i] + (1.0 - b2) * gi * gi;
    theta[i] -= lr * (m[i] / bc1) / (sqrt(v[i] / bc2) + eps);
  }
  return ORC_OK;
}

/* --------------------------------------------------------- slot layout v2 */

/* trajstore.hpp:60-87 Offsets algorithm (64-byte header, align8 arrays in the
 * reference order), with the device element types: obs u8, hidden f32,
 * actions i32, rewards f32, logp f32, dones u8, versions i64, boot_obs u8,
 * boot_hidden f32.  elem_* are byte sizes so the reference's f64 layout is the
 * same function with (8, 8, 8, 8). out[10] = obs, hidden, actions, rewards,
 * logp, dones, versions, boot_obs, boot_hidden, total. */
static size_t a8(size_t x) { return (x + 7) & ~(size_t)7; }
void orc_slot_offsets(uint32_t T, uint32_t obs_dim, uint32_t hidden_dim, uint32_t n_heads,
                      int obs_elem, int hid_elem, int rew_elem, int logp_elem, uint64_t* out) {
  size_t o = 64;
  out[0] = o; o += a8((size_t)T * obs_dim * obs_elem);
  out[1] = o; o += a8((size_t)T * hidden_dim * hid_elem);
  out[2] = o; o += a8((size_t)T * n_heads * 4);
  out[3] = o; o += a8((size_t)T * rew_elem);
  out[4] = o; o += a8((size_t)T * logp_elem);
  out[5] = o; o += a8((size_t)T * 1);
  out[6] = o; o += a8((size_t)T * 8);
  out[7] = o; o += a8((size_t)obs_dim * obs_elem);
  out[8] = o; o += a8((size_t)hidden_dim * hid_elem);
  out[9] = o;
}

/* ------------------------------------------------- synthetic env generator */

/* Restates SyntheticLatencyEnv (envs.hpp:103-158) for u8 pixels: the keyed
 * hash of make_obs (envs.hpp:143-151) is evaluated once per 8 pixels and its
 * 8 bytes become 8 consecutive u8 pixels; reward schedule envs.hpp:127, done
 * at episode_len envs.hpp:128.  env_seed = derive_seed(seed, (env << 24) ^
 * episode) as in RolloutWorker::reset_env (orchestrator.hpp:403-404). */
void orc_gen_obs(uint64_t env_seed, uint32_t step, long obs_dim, uint8_t* out) {
  for (long i = 0; i < obs_dim; ++i) {
    uint64_t h = orc_splitmix64(env_seed ^ ((uint64_t)step << 20) ^ (uint64_t)(i >> 3));
    out[i] = (uint8_t)(h >> (8 * (i & 7)));
  }
}
double orc_gen_reward(uint64_t env_seed, uint32_t step_after) {
  return 0.1 * (double)((step_after + env_seed % 7) % 11) - 0.5;
}

/* ------------------------------------------------------------------ model */
/*
 * convnet_simple (Sample Factory; not in the reference -> parity unpinned):
 *   x = obs/255, obs u8 CHW [C][H][W]
 *   conv1 C->32 k8 s4, ELU ; conv2 32->64 k4 s2, ELU ; conv3 64->128 k3 s2, ELU
 *   fc (128*H3*W3) -> 512, ELU ; GRU(512, 512) PyTorch gate order (r, z, n)
 *   logits = Wpi h' + bpi (A actions) ; value = wv . h' + bv
 * Parameter contract (flat, in this order):
 *   c1w [32][C][8][8]  c1b[32]          (PyTorch OIHW: conv1 reads CHW obs)
 *   c2w [64][4][4][32] c2b[64]          (O,kh,kw,I: activations are HWC)
 *   c3w [128][3][3][64] c3b[128]
 *   fcw [512][H3*W3*128] fcb[512]       (input flattened h, w, c)
 *   w_ih [1536][512] w_hh [1536][512] b_ih[1536] b_hh[1536]
 *   wpi [A][512] bpi[A] wv[512] bv[1]
 */
typedef struct {
  int C, H, W, A;
  int H1, W1, H2, W2, H3, W3;
  long off_c1w, off_c1b, off_c2w, off_c2b, off_c3w, off_c3b, off_fcw, off_fcb, off_wih, off_whh,
      off_bih, off_bhh, off_wpi, off_bpi, off_wv, off_bv, total;
} orc_model;

#define NH 512
#define NG (3 * NH)
#define F3 128

void orc_model_make(int C, int H, int W, int A, orc_model* m) {
  m->C = C; m->H = H; m->W = W; m->A = A;
  m->H1 = (H - 8) / 4 + 1; m->W1 = (W - 8) / 4 + 1;
  m->H2 = (m->H1 - 4) / 2 + 1; m->W2 = (m->W1 - 4) / 2 + 1;
  m->H3 = (m->H2 - 3) / 2 + 1; m->W3 = (m->W2 - 3) / 2 + 1;
  long o = 0;
  m->off_c1w = o; o += 32L * C * 64;
  m->off_c1b = o; o += 32;
  m->off_c2w = o; o += 64L * 16 * 32;
  m->off_c2b = o; o += 64;
  m->off_c3w = o; o += 128L * 9 * 64;
  m->off_c3b = o; o += 128;
  m->off_fcw = o; o += (long)NH * m->H3 * m->W3 * F3;
  m->off_fcb = o; o += NH;
  m->off_wih = o; o += (long)NG * NH;
  m->off_whh = o; o += (long)NG * NH;
  m->off_bih = o; o += NG;
  m->off_bhh = o; o += NG;
  m->off_wpi = o; o += (long)A * NH;
  m->off_bpi = o; o += A;
  m->off_wv = o; o += NH;
  m->off_bv = o; o += 1;
  m->total = o;
}

long orc_model_param_count(int C, int H, int W, int A) {
  orc_model m;
  orc_model_make(C, H, W, A, &m);
  return m.total;
}

/* Scaled-uniform (Glorot) init in the style of init_params (policy.hpp:110-131):
 * a = gain*sqrt(6/(rows+cols)), gain 1.0 on trunk/core, 0.01 on policy and
 * value heads, biases 0.  Draws come from orc_uniform keyed per tensor (the
 * reference uses mt19937_64, policy.hpp:117). */
static void fill_uniform(double* p, long rows, long cols, double gain, uint64_t key) {
  const double a = gain * sqrt(6.0 / (double)(rows + cols));
  for (long i = 0; i < rows * cols; ++i) p[i] = (2.0 * orc_uniform(key, (uint64_t)i) - 1.0) * a;
}
void orc_model_init(int C, int H, int W, int A, uint64_t seed, double* theta) {
  orc_model m;
  orc_model_make(C, H, W, A, &m);
  memset(theta, 0, sizeof(double) * m.total);
  uint64_t k = orc_derive_seed(seed, 0xA11CE);
  fill_uniform(theta + m.off_c1w, 32, (long)C * 64, 1.0, k + 1);
  fill_uniform(theta + m.off_c2w, 64, 16 * 32, 1.0, k + 2);
  fill_uniform(theta + m.off_c3w, 128, 9 * 64, 1.0, k + 3);
  fill_uniform(theta + m.off_fcw, NH, (long)m.H3 * m.W3 * F3, 1.0, k + 4);
  fill_uniform(theta + m.off_wih, NG, NH, 1.0, k + 5);
  fill_uniform(theta + m.off_whh, NG, NH, 1.0, k + 6);
  fill_uniform(theta + m.off_wpi, m.A, NH, 0.01, k + 7);
  fill_uniform(theta + m.off_wv, 1, NH, 0.01, k + 8);
}

static double elu(double x) { return x > 0 ? x : expm1(x); }
static double delu_from_out(double y) { return y > 0 ? 1.0 : y + 1.0; } /* d elu = exp(x) = y+1 */
static double sigm(double x) { return 1.0 / (1.0 + exp(-x)); }

/* Activations of one sample through the encoder (kept for backward). */
typedef struct {
  double* a1; /* [H1][W1][32] post-ELU */
  double* a2; /* [H2][W2][64] */
  double* a3; /* [H3][W3][128] */
  double* fc; /* [512] post-ELU */
} enc_cache;

static void encoder_fwd(const orc_model* m, const double* th, const uint8_t* obs, enc_cache* c) {
  const int C = m->C, H = m->H, W = m->W;
  (void)H;
  for (int y = 0; y < m->H1; ++y)
    for (int x = 0; x < m->W1; ++x)
      for (int o = 0; o < 32; ++o) {
        double acc = th[m->off_c1b + o];
        const double* w = th + m->off_c1w + (long)o * C * 64;
        for (int ci = 0; ci < C; ++ci)
          for (int kh = 0; kh < 8; ++kh)
            for (int kw = 0; kw < 8; ++kw)
              acc += w[(ci * 8 + kh) * 8 + kw] *
                     ((double)obs[((long)ci * m->H + y * 4 + kh) * W + x * 4 + kw] / 255.0);
        c->a1[((long)y * m->W1 + x) * 32 + o] = elu(acc);
      }
  for (int y = 0; y < m->H2; ++y)
    for (int x = 0; x < m->W2; ++x)
      for (int o = 0; o < 64; ++o) {
        double acc = th[m->off_c2b + o];
        const double* w = th + m->off_c2w + (long)o * 16 * 32;
        for (int kh = 0; kh < 4; ++kh)
          for (int kw = 0; kw < 4; ++kw)
            for (int ci = 0; ci < 32; ++ci)
              acc += w[(kh * 4 + kw) * 32 + ci] *
                     c->a1[((long)(y * 2 + kh) * m->W1 + x * 2 + kw) * 32 + ci];
        c->a2[((long)y * m->W2 + x) * 64 + o] = elu(acc);
      }
  for (int y = 0; y < m->H3; ++y)
    for (int x = 0; x < m->W3; ++x)
      for (int o = 0; o < 128; ++o) {
        double acc = th[m->off_c3b + o];
        const double* w = th + m->off_c3w + (long)o * 9 * 64;
        for (int kh = 0; kh < 3; ++kh)
          for (int kw = 0; kw < 3; ++kw)
            for (int ci = 0; ci < 64; ++ci)
              acc += w[(kh * 3 + kw) * 64 + ci] *
                     c->a2[((long)(y * 2 + kh) * m->W2 + x * 2 + kw) * 64 + ci];
        c->a3[((long)y * m->W3 + x) * 128 + o] = elu(acc);
      }
  const long nf = (long)m->H3 * m->W3 * F3;
  for (int j = 0; j < NH; ++j) {
    double acc = th[m->off_fcb + j];
    const double* w = th + m->off_fcw + (long)j * nf;
    for (long k = 0; k < nf; ++k) acc += w[k] * c->a3[k];
    c->fc[j] = elu(acc);
  }
}

/* GRU cell, PyTorch convention.  Saves r, z, n, ghn (= W_hn h + b_hn). */
static void gru_fwd(const orc_model* m, const double* th, const double* x, const double* h,
                    double* hout, double* r, double* z, double* n, double* ghn) {
  for (int j = 0; j < NH; ++j) {
    double gi[3], gh[3];
    for (int g = 0; g < 3; ++g) {
      const long row = (long)g * NH + j;
      double a = th[m->off_bih + row], b = th[m->off_bhh + row];
      const double* wi = th + m->off_wih + row * NH;
      const double* wh = th + m->off_whh + row * NH;
      for (int k = 0; k < NH; ++k) {
        a += wi[k] * x[k];
        b += wh[k] * h[k];
      }
      gi[g] = a;
      gh[g] = b;
    }
    const double rr = sigm(gi[0] + gh[0]);
    const double zz = sigm(gi[1] + gh[1]);
    const double nn = tanh(gi[2] + rr * gh[2]);
    r[j] = rr; z[j] = zz; n[j] = nn; ghn[j] = gh[2];
    hout[j] = (1.0 - zz) * nn + zz * h[j];
  }
}

static void heads_fwd(const orc_model* m, const double* th, const double* h, double* logits,
                      double* value) {
  for (int a = 0; a < m->A; ++a) {
    double acc = th[m->off_bpi + a];
    for (int k = 0; k < NH; ++k) acc += th[m->off_wpi + (long)a * NH + k] * h[k];
    logits[a] = acc;
  }
  double v = th[m->off_bv];
  for (int k = 0; k < NH; ++k) v += th[m->off_wv + k] * h[k];
  *value = v;
}

static void enc_alloc(const orc_model* m, enc_cache* c) {
  c->a1 = (double*)malloc(sizeof(double) * m->H1 * m->W1 * 32);
  c->a2 = (double*)malloc(sizeof(double) * m->H2 * m->W2 * 64);
  c->a3 = (double*)malloc(sizeof(double) * m->H3 * m->W3 * 128);
  c->fc = (double*)malloc(sizeof(double) * NH);
}
static void enc_free(enc_cache* c) { free(c->a1); free(c->a2); free(c->a3); free(c->fc); }

/* Batched inference for B envs: replaces forward_batch + sample_action
 * (policy.hpp:165-258, caller orchestrator.hpp:643-656).  Writes h_out,
 * logits [B][A], values [B]; if u != NULL also samples actions/logp with the
 * given uniforms (one per env). */
void orc_policy_forward(int C, int H, int W, int A, const double* th, int B, const uint8_t* obs,
                        const double* h_in, double* h_out, double* logits, double* values,
                        const double* u, int32_t* actions, double* logp) {
  orc_model m;
  orc_model_make(C, H, W, A, &m);
  enc_cache c;
  enc_alloc(&m, &c);
  double r[NH], z[NH], n[NH], ghn[NH];
  const long od = (long)C * H * W;
  for (int b = 0; b < B; ++b) {
    encoder_fwd(&m, th, obs + b * od, &c);
    gru_fwd(&m, th, c.fc, h_in + (long)b * NH, h_out + (long)b * NH, r, z, n, ghn);
    heads_fwd(&m, th, h_out + (long)b * NH, logits + (long)b * A, values + b);
    if (u) {
      double lp;
      actions[b] = orc_sample(A, logits + (long)b * A, u[b], &lp);
      logp[b] = lp;
    }
  }
  enc_free(&c);
}

/* Encoder backward for one sample: given d(fc post-ELU), accumulate grads. */
static void encoder_bwd(const orc_model* m, const double* th, const uint8_t* obs,
                        const enc_cache* c, const double* dfc, double* g) {
  const int C = m->C, W = m->W;
  const long nf = (long)m->H3 * m->W3 * F3;
  double* dz = (double*)malloc(sizeof(double) * NH);
  double* da3 = (double*)calloc(nf, sizeof(double));
  double* da2 = (double*)calloc((long)m->H2 * m->W2 * 64, sizeof(double));
  double* da1 = (double*)calloc((long)m->H1 * m->W1 * 32, sizeof(double));
  for (int j = 0; j < NH; ++j) dz[j] = dfc[j] * delu_from_out(c->fc[j]);
  for (int j = 0; j < NH; ++j) {
    if (dz[j] == 0) continue;
    const double* w = th + m->off_fcw + (long)j * nf;
    double* gw = g + m->off_fcw + (long)j * nf;
    for (long k = 0; k < nf; ++k) {
      gw[k] += dz[j] * c->a3[k];
      da3[k] += dz[j] * w[k];
    }
    g[m->off_fcb + j] += dz[j];
  }
  /* conv3 */
  for (int y = 0; y < m->H3; ++y)
    for (int x = 0; x < m->W3; ++x)
      for (int o = 0; o < 128; ++o) {
        const long oi = ((long)y * m->W3 + x) * 128 + o;
        const double d = da3[oi] * delu_from_out(c->a3[oi]);
        if (d == 0) continue;
        g[m->off_c3b + o] += d;
        const double* w = th + m->off_c3w + (long)o * 9 * 64;
        double* gw = g + m->off_c3w + (long)o * 9 * 64;
        for (int kh = 0; kh < 3; ++kh)
          for (int kw = 0; kw < 3; ++kw)
            for (int ci = 0; ci < 64; ++ci) {
              const long ii = ((long)(y * 2 + kh) * m->W2 + x * 2 + kw) * 64 + ci;
              gw[(kh * 3 + kw) * 64 + ci] += d * c->a2[ii];
              da2[ii] += d * w[(kh * 3 + kw) * 64 + ci];
            }
      }
  /* conv2 */
  for (int y = 0; y < m->H2; ++y)
    for (int x = 0; x < m->W2; ++x)
      for (int o = 0; o < 64; ++o) {
        const long oi = ((long)y * m->W2 + x) * 64 + o;
        const double d = da2[oi] * delu_from_out(c->a2[oi]);
        if (d == 0) continue;
        g[m->off_c2b + o] += d;
        const double* w = th + m->off_c2w + (long)o * 16 * 32;
        double* gw = g + m->off_c2w + (long)o * 16 * 32;
        for (int kh = 0; kh < 4; ++kh)
          for (int kw = 0; kw < 4; ++kw)
            for (int ci = 0; ci < 32; ++ci) {
              const long ii = ((long)(y * 2 + kh) * m->W1 + x * 2 + kw) * 32 + ci;
              gw[(kh * 4 + kw) * 32 + ci] += d * c->a1[ii];
              da1[ii] += d * w[(kh * 4 + kw) * 32 + ci];
            }
      }
  /* conv1 (no input gradient) */
  for (int y = 0; y < m->H1; ++y)
    for (int x = 0; x < m->W1; ++x)
      for (int o = 0; o < 32; ++o) {
        const long oi = ((long)y * m->W1 + x) * 32 + o;
        const double d = da1[oi] * delu_from_out(c->a1[oi]);
        if (d == 0) continue;
        g[m->off_c1b + o] += d;
        double* gw = g + m->off_c1w + (long)o * C * 64;
        for (int ci = 0; ci < C; ++ci)
          for (int kh = 0; kh < 8; ++kh)
            for (int kw = 0; kw < 8; ++kw)
              gw[(ci * 8 + kh) * 8 + kw] +=
                  d * ((double)obs[((long)ci * m->H + y * 4 + kh) * W + x * 4 + kw] / 255.0);
      }
  free(dz); free(da3); free(da2); free(da1);
}

/*
 * One APPO learner step over n_traj trajectories of length T, restating
 * LearnerUnit::step (orchestrator.hpp:760-868) for the recurrent model:
 *   forward on all T*n_traj obs + bootstrap obs with the current params, the
 *   GRU unrolled from the stored h0 with h_{t+1} = h'_t * (1 - done_t)
 *   (hidden reset after done, orchestrator.hpp:402,545-547);
 *   target logp / entropy (policy.hpp:262-281); vtrace per trajectory
 *   (offpolicy.hpp:61-100); advantage = pg_adv (adv_source 0), nstep - V (1,
 *   orchestrator.hpp:831-833) or GAE(lambda) (2); optional normalisation
 *   (orchestrator.hpp:838-845); exact gradient of the loss with adv and v
 *   targets constant (policy.hpp:299-428), back-propagated through the GRU
 *   over the T-step window (BPTT) and the encoder; then Adam + clip
 *   (policy.hpp:431-455) when do_adam.
 * Inputs: obs [n_traj][T+1][C*H*W] (index T = bootstrap obs), h0 [n_traj][512],
 *   actions [n_traj*T], blogp, rewards, dones.
 * Outputs: grad [P] (zeroed here), stats[8] = {policy, value, entropy, total,
 *   mean_ratio, unused...}, optional v_targets/adv/values/tlogp [n_traj*T].
 */
int orc_learner_step(int C, int H, int W, int A, double* theta, double* adam_m, double* adam_v,
                     long* adam_t, int n_traj, int T, const uint8_t* obs, const double* h0,
                     const int32_t* actions, const double* blogp, const double* rewards,
                     const uint8_t* dones, const double* hp, int do_adam, double* grad,
                     double* stats, double* out_vt, double* out_adv, double* out_values,
                     double* out_tlogp) {
  /* hp: 0 lr, 1 beta1, 2 beta2, 3 eps, 4 grad_clip, 5 entropy_coef,
   *     6 value_coef, 7 clip_low, 8 clip_high, 9 rho_bar, 10 c_bar, 11 gamma,
   *     12 adv_source, 13 normalize, 14 gae_lambda */
  orc_model m;
  orc_model_make(C, H, W, A, &m);
  const long P = m.total, od = (long)C * H * W;
  const int B = n_traj * T;
  int st = orc_vtrace_validate(hp[9], hp[10], hp[11]);
  if (st) return st;
  for (int s = 0; s < B; ++s)
    if (actions[s] < 0 || actions[s] >= A) return ORC_CONTRACT;

  enc_cache* ec = (enc_cache*)malloc(sizeof(enc_cache) * n_traj * (T + 1));
  double* hs = (double*)malloc(sizeof(double) * n_traj * (T + 2) * NH);   /* h_t inputs */
  double* hc = (double*)malloc(sizeof(double) * n_traj * (T + 1) * NH);   /* core outputs */
  double* gr = (double*)malloc(sizeof(double) * n_traj * (T + 1) * NH);
  double* gz = (double*)malloc(sizeof(double) * n_traj * (T + 1) * NH);
  double* gn = (double*)malloc(sizeof(double) * n_traj * (T + 1) * NH);
  double* gh = (double*)malloc(sizeof(double) * n_traj * (T + 1) * NH);
  double* logits = (double*)malloc(sizeof(double) * n_traj * (T + 1) * A);
  double* values = (double*)malloc(sizeof(double) * n_traj * (T + 1));
  double* tl = (double*)malloc(sizeof(double) * B);
  double* ent = (double*)malloc(sizeof(double) * B);
  double* vt = (double*)malloc(sizeof(double) * B);
  double* pg = (double*)malloc(sizeof(double) * B);
  double* adv = (double*)malloc(sizeof(double) * B);
  double* boot = (double*)malloc(sizeof(double) * n_traj);
  double* vals = (double*)malloc(sizeof(double) * B);

  for (int i = 0; i < n_traj; ++i) {
    memcpy(hs + (long)i * (T + 2) * NH, h0 + (long)i * NH, sizeof(double) * NH);
    for (int t = 0; t <= T; ++t) {
      const long k = (long)i * (T + 1) + t;
      enc_alloc(&m, &ec[k]);
      encoder_fwd(&m, theta, obs + k * od, &ec[k]);
      const double* hin = hs + ((long)i * (T + 2) + t) * NH;
      double* hnext = hs + ((long)i * (T + 2) + t + 1) * NH;
      gru_fwd(&m, theta, ec[k].fc, hin, hc + k * NH, gr + k * NH, gz + k * NH, gn + k * NH,
              gh + k * NH);
      const double keep = (t < T && dones[(long)i * T + t]) ? 0.0 : 1.0;
      for (int j = 0; j < NH; ++j) hnext[j] = hc[k * NH + j] * keep;
      heads_fwd(&m, theta, hc + k * NH, logits + k * A, values + k);
    }
  }
  for (int i = 0; i < n_traj; ++i) {
    boot[i] = values[(long)i * (T + 1) + T];
    for (int t = 0; t < T; ++t) {
      const long k = (long)i * (T + 1) + t, s = (long)i * T + t;
      orc_logp_entropy(A, logits + k * A, actions[s], &tl[s], &ent[s]);
      vals[s] = values[k];
    }
  }
  for (int i = 0; i < n_traj; ++i) {
    const long o = (long)i * T;
    st = orc_vtrace(T, rewards + o, vals + o, boot[i], tl + o, blogp + o, dones + o, hp[9],
                    hp[10], hp[11], vt + o, pg + o, 0, 0);
    if (st) goto done;
    const int src = (int)hp[12];
    if (src == 0) {
      memcpy(adv + o, pg + o, sizeof(double) * T);
    } else if (src == 1) {
      orc_nstep_returns(T, rewards + o, boot[i], dones + o, hp[11], adv + o);
      for (int t = 0; t < T; ++t) adv[o + t] -= vals[o + t];
    } else {
      orc_gae(T, rewards + o, vals + o, boot[i], dones + o, hp[11], hp[14], adv + o, 0);
    }
  }
  if (hp[13] != 0.0) {
    double mean = 0, sq = 0;
    for (int s = 0; s < B; ++s) mean += adv[s];
    mean /= B;
    for (int s = 0; s < B; ++s) sq += (adv[s] - mean) * (adv[s] - mean);
    const double sd = sqrt(sq / B) + 1e-8;
    for (int s = 0; s < B; ++s) adv[s] = (adv[s] - mean) / sd;
  }

  /* loss + dlogits / dvalue (policy.hpp:323-375) */
  memset(grad, 0, sizeof(double) * P);
  {
    const double invB = 1.0 / B, ec_ = hp[5], vc = hp[6], lo = hp[7], hi = hp[8];
    double pol = 0, vl = 0, es = 0, rs = 0;
    double* dhc = (double*)calloc((size_t)n_traj * (T + 1) * NH, sizeof(double));
    for (int i = 0; i < n_traj; ++i)
      for (int t = 0; t < T; ++t) {
        const long k = (long)i * (T + 1) + t, s = (long)i * T + t;
        double probs[64], dlog[64];
        orc_softmax(A, logits + k * A, probs);
        const double ratio = orc_importance_ratio(tl[s], blogp[s]);
        const double dsur = orc_ppo_dratio(ratio, adv[s], lo, hi);
        const double dL_dlogp = -invB * dsur * ratio;
        pol -= orc_ppo_objective(ratio, adv[s], lo, hi);
        es += ent[s];
        rs += ratio;
        const double verr = vals[s] - vt[s];
        vl += verr * verr;
        const double dV = vc * invB * 2.0 * verr;
        for (int a = 0; a < A; ++a) {
          const double pk = probs[a];
          const double dlp = (a == actions[s] ? 1.0 : 0.0) - pk;
          const double dH = pk > 0 ? -pk * (log(pk) + ent[s]) : 0.0;
          dlog[a] = dL_dlogp * dlp - ec_ * invB * dH;
        }
        const double* h = hc + k * NH;
        double* dh = dhc + k * NH;
        for (int a = 0; a < A; ++a) {
          double* gw = grad + m.off_wpi + (long)a * NH;
          const double* w = theta + m.off_wpi + (long)a * NH;
          for (int j = 0; j < NH; ++j) {
            gw[j] += dlog[a] * h[j];
            dh[j] += dlog[a] * w[j];
          }
          grad[m.off_bpi + a] += dlog[a];
        }
        for (int j = 0; j < NH; ++j) {
          grad[m.off_wv + j] += dV * h[j];
          dh[j] += dV * theta[m.off_wv + j];
        }
        grad[m.off_bv] += dV;
      }
    stats[0] = pol * invB;
    stats[1] = vc * vl * invB;
    stats[2] = es * invB;
    stats[3] = stats[0] + stats[1] - ec_ * stats[2];
    stats[4] = rs * invB;

    /* BPTT through the GRU, reverse over t; bootstrap step gets no gradient */
    double* dnext = (double*)malloc(sizeof(double) * NH);
    double* dgi = (double*)malloc(sizeof(double) * NG);
    double* dgh = (double*)malloc(sizeof(double) * NG);
    double* dx = (double*)malloc(sizeof(double) * NH);
    for (int i = 0; i < n_traj; ++i) {
      memset(dnext, 0, sizeof(double) * NH);
      for (int t = T - 1; t >= 0; --t) {
        const long k = (long)i * (T + 1) + t;
        const double keep = dones[(long)i * T + t] ? 0.0 : 1.0;
        const double* hin = hs + ((long)i * (T + 2) + t) * NH;
        double dh[NH];
        for (int j = 0; j < NH; ++j) dh[j] = dhc[k * NH + j] + keep * dnext[j];
        for (int j = 0; j < NH; ++j) {
          const double r = gr[k * NH + j], z = gz[k * NH + j], n = gn[k * NH + j];
          const double dn = dh[j] * (1.0 - z);
          const double dzz = dh[j] * (hin[j] - n);
          const double dan = dn * (1.0 - n * n);
          const double dr = dan * gh[k * NH + j];
          dgi[j] = dr * r * (1.0 - r);
          dgi[NH + j] = dzz * z * (1.0 - z);
          dgi[2 * NH + j] = dan;
          dgh[j] = dgi[j];
          dgh[NH + j] = dgi[NH + j];
          dgh[2 * NH + j] = dan * r;
          dnext[j] = dh[j] * z;
        }
        memset(dx, 0, sizeof(double) * NH);
        for (int row = 0; row < NG; ++row) {
          const double* wi = theta + m.off_wih + (long)row * NH;
          const double* wh = theta + m.off_whh + (long)row * NH;
          double* gwi = grad + m.off_wih + (long)row * NH;
          double* gwh = grad + m.off_whh + (long)row * NH;
          const double a = dgi[row], b = dgh[row];
          for (int j = 0; j < NH; ++j) {
            gwi[j] += a * ec[k].fc[j];
            gwh[j] += b * hin[j];
            dx[j] += a * wi[j];
            dnext[j] += b * wh[j];
          }
          grad[m.off_bih + row] += a;
          grad[m.off_bhh + row] += b;
        }
        encoder_bwd(&m, theta, obs + k * od, &ec[k], dx, grad);
      }
    }
    free(dnext); free(dgi); free(dgh); free(dx); free(dhc);
  }
  for (long p = 0; p < P; ++p)
    if (!finite(grad[p])) { st = ORC_NUMERIC; goto done; }
  if (!finite(stats[3])) { st = ORC_NUMERIC; goto done; }
  if (out_vt) memcpy(out_vt, vt, sizeof(double) * B);
  if (out_adv) memcpy(out_adv, adv, sizeof(double) * B);
  if (out_values) memcpy(out_values, vals, sizeof(double) * B);
  if (out_tlogp) memcpy(out_tlogp, tl, sizeof(double) * B);
  if (do_adam)
    st = orc_adam_step(P, theta, adam_m, adam_v, grad, adam_t, hp[0], hp[1], hp[2], hp[3], hp[4]);
done:
  for (int k = 0; k < n_traj * (T + 1); ++k) enc_free(&ec[k]);
  free(ec); free(hs); free(hc); free(gr); free(gz); free(gn); free(gh); free(logits);
  free(values); free(tl); free(ent); free(vt); free(pg); free(adv); free(boot); free(vals);
  return st;
}
