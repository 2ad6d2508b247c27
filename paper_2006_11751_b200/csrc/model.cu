// Model-level orchestration and its C ABI: parameter contract and init,
// batched policy inference (replaces forward_batch + sample_action,
// policy.hpp:165-258, in PolicyWorkerUnit::run_once, orchestrator.hpp:602-673)
// and the learner step (replaces assemble_minibatch's gather +
// LearnerUnit::step, orchestrator.hpp:760-868).
//
// Dense contractions go to the tcgen05 GEMM engine (gemm.cu); everything else
// to the SIMT kernels of model_kernels.cu.  Activations are NHWC bf16 so each
// conv layer is one im2col + one GEMM whose [rows][Cout] output IS the next
// layer's NHWC input, and conv3's output rows flatten (h, w, c) for the FC.
#include <cuda_bf16.h>

#include <unistd.h>

#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "gemm.cuh"
#include "model.cuh"
#include "model_kernels.cuh"
#include "slotq.cuh"

namespace appo_b200 {

static size_t a8(size_t x) { return (x + 7) & ~size_t(7); }

int make_dims(const appo_model_desc& m, Dims* out) {
  Dims d{};
  d.C = m.obs_c;
  d.H = m.obs_h;
  d.W = m.obs_w;
  d.A = m.n_actions;
  d.T = m.T;
  if (d.C < 1 || d.H < 36 || d.W < 36 || (d.W % 4) != 0 || d.A < 1 || d.A > kMaxActions - 1 ||
      d.T < 1) {
    set_error("model desc: need C>=1, H,W>=36, W%4==0, 1<=n_actions<=15, T>=1");
    return APPO_ERR_CONFIG;
  }
  d.H1 = (d.H - 8) / 4 + 1;
  d.W1 = (d.W - 8) / 4 + 1;
  d.H2 = (d.H1 - 4) / 2 + 1;
  d.W2 = (d.W1 - 4) / 2 + 1;
  d.H3 = (d.H2 - 3) / 2 + 1;
  d.W3 = (d.W2 - 3) / 2 + 1;
  d.P1 = d.H1 * d.W1;
  d.P2 = d.H2 * d.W2;
  d.P3 = d.H3 * d.W3;
  d.K1 = d.C * 64;
  d.F = d.P3 * 128;
  int64_t o = 0;
  d.off_c1w = o; o += 32LL * d.K1;
  d.off_c1b = o; o += 32;
  d.off_c2w = o; o += 64LL * 16 * 32;
  d.off_c2b = o; o += 64;
  d.off_c3w = o; o += 128LL * 9 * 64;
  d.off_c3b = o; o += 128;
  d.off_fcw = o; o += (int64_t)kHidden * d.F;
  d.off_fcb = o; o += kHidden;
  d.off_wih = o; o += (int64_t)kGates * kHidden;
  d.off_whh = o; o += (int64_t)kGates * kHidden;
  d.off_bih = o; o += kGates;
  d.off_bhh = o; o += kGates;
  d.off_wpi = o; o += (int64_t)d.A * kHidden;
  d.off_bpi = o; o += d.A;
  d.off_wv = o; o += kHidden;
  d.off_bv = o; o += 1;
  d.total = o;
  d.obs_dim = (int64_t)d.C * d.H * d.W;
  // trajectory slot layout v2 (trajstore.hpp:62-87; u8 obs, f32 hidden/reward/logp)
  size_t s = 64;
  const size_t T = d.T, od = d.obs_dim, hd = kHidden;
  d.slot[0] = s; s += a8(T * od);
  d.slot[1] = s; s += a8(T * hd * 4);
  d.slot[2] = s; s += a8(T * 1 * 4);
  d.slot[3] = s; s += a8(T * 4);
  d.slot[4] = s; s += a8(T * 4);
  d.slot[5] = s; s += a8(T);
  d.slot[6] = s; s += a8(T * 8);
  d.slot[7] = s; s += a8(od);
  d.slot[8] = s; s += a8(hd * 4);
  d.slot[9] = s;
  *out = d;
  return APPO_OK;
}

namespace {

uint16_t host_f2bf(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  const uint32_t r = ((u >> 16) & 1u) + 0x7FFFu;  // round to nearest even
  return (uint16_t)((u + r) >> 16);
}

double host_uniform(uint64_t key, uint64_t counter) {
  const uint64_t h = host_splitmix64(key ^ host_splitmix64(counter));
  return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

// Glorot-uniform in the style of init_params (policy.hpp:110-131); gain 1.0
// trunk/core, 0.01 heads; biases zero.  Same stream as the oracle's
// orc_model_init so tests can start both from identical parameters.
void init_params_host(const Dims& d, uint64_t seed, std::vector<float>& th) {
  th.assign(d.total, 0.0f);
  const uint64_t k = host_derive_seed(seed, 0xA11CE);
  auto fill = [&](int64_t off, int64_t rows, int64_t cols, double gain, uint64_t key) {
    const double a = gain * std::sqrt(6.0 / (double)(rows + cols));
    for (int64_t i = 0; i < rows * cols; ++i)
      th[off + i] = (float)((2.0 * host_uniform(key, (uint64_t)i) - 1.0) * a);
  };
  fill(d.off_c1w, 32, d.K1, 1.0, k + 1);
  fill(d.off_c2w, 64, 16 * 32, 1.0, k + 2);
  fill(d.off_c3w, 128, 9 * 64, 1.0, k + 3);
  fill(d.off_fcw, kHidden, d.F, 1.0, k + 4);
  fill(d.off_wih, kGates, kHidden, 1.0, k + 5);
  fill(d.off_whh, kGates, kHidden, 1.0, k + 6);
  fill(d.off_wpi, d.A, kHidden, 0.01, k + 7);
  fill(d.off_wv, 1, kHidden, 0.01, k + 8);
}

// Arena allocation helper: offsets are 256-byte aligned.
struct Arena {
  size_t off = 0;
  template <class T>
  size_t take(T** p, size_t count) {
    const size_t o = off;
    off += ((count * sizeof(T)) + 255) & ~size_t(255);
    *p = reinterpret_cast<T*>(o);  // relocated after the single cudaMalloc
    return o;
  }
};
template <class T>
void reloc(T*& p, uint8_t* base) {
  p = reinterpret_cast<T*>(base + reinterpret_cast<size_t>(p));
}

int alloc_scratch(Ctx* c, Model* M, Scratch& s, int R, int n_traj, bool learner) {
  if (R <= s.cap_rows && n_traj <= s.cap_traj) return APPO_OK;
  const Dims& d = M->d;
  if (s.col1) {
    cudaStreamSynchronize(c->stream);
    cudaFree(s.col1);
    cudaFreeHost(s.h_stats);
  }
  s = Scratch{};
  const int B = learner ? n_traj * d.T : R;
  const int G = learner ? n_traj : R;  // rows of gh per GEMM
  Arena a;
  // im2col matrices only for the learner (inference gathers them on the fly);
  // col1 stays the arena base (it is what gets freed)
  a.take(&s.col1, learner ? (size_t)R * d.P1 * d.K1 : 64);
  a.take(&s.a1, (size_t)R * d.P1 * 32);
  a.take(&s.col2, 64);  // im2col matrices are no longer materialised
  a.take(&s.a2, (size_t)R * d.P2 * 64);
  a.take(&s.col3, 64);
  a.take(&s.a3, (size_t)R * d.F);
  a.take(&s.x, (size_t)R * kHidden);
  a.take(&s.gi, (size_t)R * kGates);
  a.take(&s.gh, (size_t)G * kGates);
  a.take(&s.hbf, (size_t)R * kHidden);
  if (learner) {
    a.take(&s.core, (size_t)R * kHidden);
    a.take(&s.core_bf, (size_t)R * kHidden);
    a.take(&s.gates, (size_t)R * 4 * kHidden);
    a.take(&s.hin, (size_t)R * kHidden);
    a.take(&s.hcur, (size_t)2 * n_traj * kHidden);  // ping-pong h_t for the persistent GRU
    a.take(&s.dghx, (size_t)2 * n_traj * kGates);
    a.take(&s.hcur_bf, (size_t)2 * n_traj * kHidden);
    a.take(&s.logits, (size_t)R * d.A);
    a.take(&s.values, (size_t)R);
    a.take(&s.tlogp, (size_t)B);
    a.take(&s.ent, (size_t)B);
    a.take(&s.vt, (size_t)B);
    a.take(&s.pg, (size_t)B);
    a.take(&s.adv, (size_t)B);
    a.take(&s.rew, (size_t)B);
    a.take(&s.blogp, (size_t)B);
    a.take(&s.act, (size_t)B);
    a.take(&s.done, (size_t)B);
    a.take(&s.ver, (size_t)B);
    a.take(&s.dlog, (size_t)B * (d.A + 1));
    a.take(&s.dhead, (size_t)B * 16);
    a.take(&s.dcore, (size_t)B * kHidden);
    a.take(&s.dnext, (size_t)n_traj * kHidden);
    a.take(&s.dgi, (size_t)B * kGates);
    a.take(&s.dgh, (size_t)B * kGates);
    a.take(&s.dzfc, (size_t)B * kHidden);
    a.take(&s.dz3, (size_t)B * d.F);
    a.take(&s.dz2, (size_t)B * d.P2 * 64);
    a.take(&s.dz1, (size_t)B * d.P1 * 32);
    a.take(&s.wt3, (size_t)4 * 64 * 512);
    a.take(&s.wt2, (size_t)4 * 32 * 256);
    a.take(&s.headw, (size_t)16 * kHidden);
    a.take(&s.colsum_part, (size_t)160 * (kMaxActions + 1) * (kHidden + 1) + 256 * kGates);
    a.take(&s.bias_acc, (size_t)4 * kBiasAccCols);
    a.take(&s.bias_cnt, (size_t)4);
    a.take(&s.slot_ids, (size_t)n_traj);
    a.take(&s.stats, (size_t)16);
  }
  uint8_t* base = nullptr;
  if (cudaMalloc(&base, a.off) != cudaSuccess) {
    set_error("scratch allocation failed (" + std::to_string(a.off >> 20) + " MiB)");
    s = Scratch{};
    return APPO_ERR_RESOURCE;
  }
  reloc(s.col1, base); reloc(s.a1, base); reloc(s.col2, base); reloc(s.a2, base);
  reloc(s.col3, base); reloc(s.a3, base); reloc(s.x, base); reloc(s.gi, base);
  reloc(s.gh, base); reloc(s.hbf, base);
  if (learner) {
    reloc(s.core, base); reloc(s.core_bf, base); reloc(s.gates, base); reloc(s.hin, base);
    reloc(s.hcur, base); reloc(s.dghx, base); reloc(s.hcur_bf, base); reloc(s.logits, base); reloc(s.values, base); reloc(s.tlogp, base);
    reloc(s.ent, base); reloc(s.vt, base); reloc(s.pg, base); reloc(s.adv, base);
    reloc(s.rew, base); reloc(s.blogp, base); reloc(s.act, base); reloc(s.done, base);
    reloc(s.ver, base); reloc(s.dlog, base); reloc(s.dhead, base); reloc(s.dcore, base);
    reloc(s.dnext, base); reloc(s.dgi, base); reloc(s.dgh, base); reloc(s.dzfc, base);
    reloc(s.dz3, base); reloc(s.dz2, base); reloc(s.dz1, base); reloc(s.wt3, base);
    reloc(s.wt2, base); reloc(s.headw, base); reloc(s.colsum_part, base);
    reloc(s.bias_acc, base); reloc(s.bias_cnt, base);
    if (cudaMemset(s.bias_acc, 0, sizeof(unsigned long long) * 4 * kBiasAccCols) != cudaSuccess ||
        cudaMemset(s.bias_cnt, 0, sizeof(unsigned) * 4) != cudaSuccess) {
      cudaFree(base);
      s = Scratch{};
      set_error("scratch memset failed");
      return APPO_ERR_RESOURCE;
    }
    reloc(s.slot_ids, base); reloc(s.stats, base);
    if (cudaMallocHost(&s.h_stats, sizeof(double) * 16 + sizeof(int32_t) * n_traj) !=
        cudaSuccess) {
      cudaFree(base);
      s = Scratch{};
      set_error("pinned stats allocation failed");
      return APPO_ERR_RESOURCE;
    }
  } else {
    cudaMallocHost(&s.h_stats, sizeof(double) * 16);
  }
  // col1 is the arena base (first take) -> freeing col1 frees the arena.
  s.cap_rows = R;
  s.cap_traj = n_traj;
  return APPO_OK;
}

// Split-K factor for a GEMM with a long reduction (weight gradients): the
// main loop shrinks with more splits, the fp32 partial traffic (write + read
// by the reduce) and one extra launch grow.  Per-k-block SM time: the larger
// of the MMA (2*BN clk for 128xBNx64) and the L2->SMEM operand stream
// (~100 B/clk per SM); partials at ~6 TB/s.
int splits_for(Ctx* c, int M, int N, int bn, int K) {
  const int tiles = ((M + 127) / 128) * ((N + bn - 1) / bn);
  const int nkb = (K + 63) / 64;
  const int smem = 4 * (16384 + bn * 128) + 1280;
  int per_sm = (227 * 1024) / smem;
  const int tmem_cols = 2 * bn <= 32 ? 32 : 2 * bn <= 64 ? 64 : 2 * bn <= 128 ? 128 : 2 * bn <= 256 ? 256 : 512;
  if (per_sm > 512 / tmem_cols) per_sm = 512 / tmem_cols;
  if (per_sm < 1) per_sm = 1;
  const double clk_kb = std::fmax(2.0 * bn, (16384.0 + bn * 128.0) / 100.0);
  const double us_kb = clk_kb / 1900.0;
  const int slots = c->num_sms * per_sm;
  double best_t = 1e30;
  int best = 1;
  for (int sp = 1; sp <= nkb / 2 || sp == 1; ++sp) {
    const int kbps = (nkb + sp - 1) / sp;
    if (sp > 1 && (nkb + kbps - 1) / kbps != sp) continue;  // same as a smaller split
    const int units = tiles * sp;
    const int waves = (units + slots - 1) / slots;
    const int conc = units < slots ? (units + c->num_sms - 1) / c->num_sms : per_sm;
    double t = waves * (conc < 1 ? 1 : conc) * kbps * us_kb;
    if (sp > 1) t += 2.0 * sp * (double)M * N * 4.0 / 6.0e6 + 2.0;
    if (t < best_t - 1e-9) {
      best_t = t;
      best = sp;
    }
    if (sp > 1024) break;
  }
  return best;
}

#define TRY(x)                    \
  do {                            \
    int _st = (x);                \
    if (_st != APPO_OK) return _st; \
  } while (0)

// Encoder forward over R images: col1..a3 -> x (bf16 [R][512]) and gi.
// Encoder forward over R images.  implicit: the three convolutions gather
// their A operand on the fly (inference: no im2col traffic); otherwise the
// im2col matrices are materialised because the learner's weight gradients
// consume them.
// conv1 input description (u8 images, contiguous batch or trajectory slots)
ConvIn conv1_in(const ObsSrc& src, int R, const Dims& d) {
  ConvIn in;
  in.src = src.base;
  in.img_stride = src.img_stride;
  in.slot_ids = src.slot_ids;
  in.slot_bytes = src.slot_bytes;
  in.obs_off = src.obs_off;
  in.boot_off = src.boot_off;
  in.T = src.T;
  in.n_traj = src.n_traj;
  in.n_slots = src.n_slots;
  in.n_img = R;
  in.Hi = d.H; in.Wi = d.W; in.Cin = d.C; in.ksz = 8; in.s = 4; in.Ho = d.H1; in.Wo = d.W1;
  in.u8 = true;
  return in;
}

int encoder_forward(Ctx* c, Model* M, Scratch& s, const ObsSrc& src, int R, const uint16_t* wb,
                    const float* pf, int pub, bool implicit, bool conv2_implicit,
                    bool gate_proj = true, cudaEvent_t join_before_fc = nullptr) {
  const Dims& d = M->d;
  Epilogue e;
  // conv1: [R*P1, 32] = (1024 + obs) . W1h^T / 255 + bias' (fp16 operands,
  // offset removed by the corrected bias of the published copy)
  e.flags = EPI_BIAS | EPI_ELU | EPI_BF16;
  e.scale = 1.0f / 255.0f;
  e.bias = M->pub_c1b[pub];
  e.out = s.a1;
  e.ldo = 32;
  // conv1 gathers its input from the u8 images (smem-staged implicit GEMM);
  // so does its weight gradient in the learner (conv1_wgrad_implicit)
  // conv1 as a space-to-depth taps GEMM (conv1.cu: each image byte converted
  // once); the im2col engine path remains for shapes outside its envelope
  // (unaligned images) and as the A/B reference (APPO_CONV1=engine)
  static const bool conv1_engine = [] {
    const char* v = getenv("APPO_CONV1");
    return v && v[0] == 'e';
  }();
  const ConvIn c1in = conv1_in(src, R, d);
  if (!conv1_engine && conv1_s2d_supported(c1in, 32, e) && conv1_s2d_forward(c, c1in, M->pub_c1h[pub], e) == APPO_OK) {
  } else {
    TRY(conv_implicit_bf16(c, c1in, 32, Operand{M->pub_c1h[pub], d.K1, false}, e, 32));
  }
  e.scale = 1.0f;
  e.bias = pf + d.off_c2b;
  e.out = s.a2;
  e.ldo = 64;
  if (implicit || conv2_implicit) {
    ConvIn in;
    in.src = reinterpret_cast<const uint8_t*>(s.a1);
    in.n_img = R;
    in.Hi = d.H1; in.Wi = d.W1; in.Cin = 32; in.ksz = 4; in.s = 2; in.Ho = d.H2; in.Wo = d.W2;
    // space-to-depth taps GEMM (conv2.cu), else the per-tap strided-box engine path
    static const bool conv2_engine = [] {
      const char* v = getenv("APPO_CONV2");
      return v && v[0] == 'e';
    }();
    const int st2 = conv2_engine ? APPO_ERR_CONTRACT
                                 : conv2_s2d_forward(c, s.a1, R, d.H1, d.W1, d.H2, d.W2,
                                                     wb + d.off_c2w, e);
    if (st2 == APPO_ERR_CONTRACT)
      TRY(conv_implicit_bf16(c, in, 64, Operand{wb + d.off_c2w, 512, false}, e, 64));
    else if (st2 != APPO_OK)
      return st2;
  } else {
    TRY(k_im2col_nhwc(c, s.a1, R, d.H1, d.W1, 32, 4, 2, d.H2, d.W2, s.col2));
    TRY(gemm_bf16(c, R * d.P2, 64, 512, Operand{s.col2, 512, false},
                  Operand{wb + d.off_c2w, 512, false}, e, 64));
  }
  e.bias = pf + d.off_c3b;
  e.out = s.a3;
  e.ldo = 128;
  if (implicit || conv2_implicit) {
    ConvIn in;
    in.src = reinterpret_cast<const uint8_t*>(s.a2);
    in.n_img = R;
    in.Hi = d.H2; in.Wi = d.W2; in.Cin = 64; in.ksz = 3; in.s = 2; in.Ho = d.H3; in.Wo = d.W3;
    TRY(conv_implicit_bf16(c, in, 128, Operand{wb + d.off_c3w, 576, false}, e, 128));
  } else {
    TRY(k_im2col_nhwc(c, s.a2, R, d.H2, d.W2, 64, 3, 2, d.H3, d.W3, s.col3));
    TRY(gemm_bf16(c, R * d.P3, 128, 576, Operand{s.col3, 576, false},
                  Operand{wb + d.off_c3w, 576, false}, e, 128));
  }
  // the previous learner step's Adam over the FC / GRU / head parameters
  // (side stream) is complete before anything reads them
  if (join_before_fc) APPO_CUDA_TRY(cudaStreamWaitEvent(c->stream, join_before_fc, 0));
  e.bias = pf + d.off_fcb;
  e.out = s.x;
  e.ldo = kHidden;
  // learner-sized batches: narrow N tiles fill more SMs (scripts/gemm_sweep.py)
  const bool small = R <= 4096;
  TRY(gemm_bf16(c, R, kHidden, d.F, Operand{s.a3, d.F, false}, Operand{wb + d.off_fcw, d.F, false},
                e, small ? 64 : 256));
  if (!gate_proj) return APPO_OK;  // inference: the gate GEMMs are fused with the cell
  Epilogue g;
  g.flags = EPI_BIAS;
  g.bias = pf + d.off_bih;
  g.out = s.gi;
  g.ldo = kGates;
  TRY(gemm_bf16(c, R, kGates, kHidden, Operand{s.x, kHidden, false},
                Operand{wb + d.off_wih, kHidden, false}, g, small ? 64 : 128));
  return APPO_OK;
}

}  // namespace

// dp.cu: bucketed data-parallel gradient all-reduce
int dp_bucket(Ctx* c, float* buf, int64_t n);
int dp_finish(Ctx* c, float* buf, int64_t n, const int** peer_flags);

// Batched inference over B observations at obs_base + b*obs_stride (contiguous
// batch or trajectory slots): encoder + GRU + heads + sampling.
int sampler_infer(Ctx* c, const uint8_t* obs_base, int64_t obs_stride, int B, const float* h_in,
                  uint64_t counter0, int32_t* actions, float* logp, float* h_out, float* values,
                  float* logits, int64_t* version_out) {
  Model* M = c->model;
  const Dims& d = M->d;
  Reader* rd = reader_of(c);
  APPO_REQUIRE(rd != nullptr, APPO_ERR_RESOURCE, "inference state allocation failed");
  Scratch& s = rd->s;
  TRY(alloc_scratch(c, M, s, B, 0, false));
  // ParamStore::fetch (policy.hpp:498-509): newest COMPLETED publish; if the
  // newest Adam step is still running (possibly on the learner's stream) take
  // the previous one instead of waiting for it.
  // Candidates: the newest kPub-1 publishes (the oldest slot is the learner's
  // next write target); take the newest whose Adam step has completed.
  int pub = M->published;
  for (int back = 0; back <= Model::kPub - 2; ++back) {
    pub = (M->published - back + Model::kPub) % Model::kPub;
    if (cudaEventQuery(M->ready_ev[pub]) == cudaSuccess) break;
  }
  APPO_CUDA_TRY(cudaStreamWaitEvent(c->stream, M->ready_ev[pub], 0));
  if (version_out) *version_out = M->pub_version[pub];
  const uint16_t* wb = M->pub_bf16[pub];
  const float* pf = M->pub_f32[pub];
  ObsSrc src;
  src.base = obs_base;
  src.img_stride = obs_stride;
  // GRU cell fused into its gate GEMMs (gru_infer.cu) unless the head count is
  // outside its envelope (A > 7) or APPO_GRU_INFER=unfused (A/B reference)
  static const bool unfused = [] {
    const char* v = getenv("APPO_GRU_INFER");
    return v && v[0] == 'u';
  }();
  if (!unfused && gru_infer_fused_supported(B, d.A)) {
    TRY(encoder_forward(c, M, s, src, B, wb, pf, pub, /*implicit=*/true, true, /*gate_proj=*/false));
    TRY(k_f32_to_bf16(c, B, h_in, kHidden, s.hbf, kHidden, kHidden));
    TRY(gru_infer_fused(c, B, d.A, s.x, s.hbf, wb + d.off_wih, wb + d.off_whh, pf + d.off_bih,
                        pf + d.off_bhh, h_in, pf + d.off_wpi, pf + d.off_bpi, pf + d.off_wv,
                        pf + d.off_bv, M->sample_key, counter0, /*partials=*/s.gh, h_out, actions,
                        logp, values, logits));
    APPO_CUDA_TRY(cudaEventRecord(rd->read_ev[pub], c->stream));
    return APPO_OK;
  }
  TRY(encoder_forward(c, M, s, src, B, wb, pf, pub, /*implicit=*/true, true));
  TRY(k_f32_to_bf16(c, B, h_in, kHidden, s.hbf, kHidden, kHidden));
  Epilogue g;
  g.flags = EPI_BIAS;
  g.bias = pf + d.off_bhh;
  g.out = s.gh;
  g.ldo = kGates;
  TRY(gemm_bf16(c, B, kGates, kHidden, Operand{s.hbf, kHidden, false},
                Operand{wb + d.off_whh, kHidden, false}, g, 128));
  TRY(k_gru_infer(c, B, d.A, s.gi, s.gh, h_in, pf + d.off_wpi, pf + d.off_bpi, pf + d.off_wv,
                  pf + d.off_bv, M->sample_key, counter0, h_out, actions, logp, values, logits));
  // last read of pub[pub] by this context: the learner waits on this event
  // (and every other reader's) before overwriting the buffer
  APPO_CUDA_TRY(cudaEventRecord(rd->read_ev[pub], c->stream));
  return APPO_OK;
}

Reader* reader_of(Ctx* c) {
  if (c->reader) return c->reader;
  Reader* r = new Reader();
  for (int k = 0; k < Model::kPub; ++k)
    if (cudaEventCreateWithFlags(&r->read_ev[k], cudaEventDisableTiming) != cudaSuccess) {
      for (int j = 0; j < k; ++j) cudaEventDestroy(r->read_ev[j]);
      delete r;
      return nullptr;
    }
  {
    std::lock_guard<std::mutex> lk(c->model->readers_mu);
    c->model->readers.push_back(r);
  }
  c->reader = r;
  return r;
}

static void reader_free(Reader* r) {
  if (r->s.col1) cudaFree(r->s.col1);
  if (r->s.h_stats) cudaFreeHost(r->s.h_stats);
  for (int k = 0; k < Model::kPub; ++k)
    if (r->read_ev[k]) cudaEventDestroy(r->read_ev[k]);
  delete r;
}

void reader_release(Ctx* c) {
  Reader* r = c->reader;
  if (!r) return;
  c->reader = nullptr;
  if (c->model) {
    std::lock_guard<std::mutex> lk(c->model->readers_mu);
    auto& v = c->model->readers;
    for (size_t i = 0; i < v.size(); ++i)
      if (v[i] == r) {
        v.erase(v.begin() + (long)i);
        break;
      }
  }
  reader_free(r);
}

int wait_readers(Model* M, cudaStream_t st, int k) {
  std::lock_guard<std::mutex> lk(M->readers_mu);
  for (Reader* r : M->readers) APPO_CUDA_TRY(cudaStreamWaitEvent(st, r->read_ev[k], 0));
  return APPO_OK;
}

const char* side_class_name(const char* name) {
  static std::mutex mu;
  static std::set<std::string> names;
  std::lock_guard<std::mutex> lock(mu);
  return names.insert(std::string(name) + "@side").first->c_str();
}

}  // namespace appo_b200

using namespace appo_b200;

int model_create(Ctx* c) {
  Model* M = new Model();
  int st = make_dims(c->desc, &M->d);
  if (st) {
    delete M;
    return st;
  }
  // encoder kernel envelope (conv1 input staging): W in {64, 128}, C*W <= 512
  if ((M->d.W != 64 && M->d.W != 128) || M->d.C * M->d.W > 512) {
    delete M;
    set_error("model desc: the sm_100a encoder needs obs width 64 or 128 and C*W <= 512");
    return APPO_ERR_CONFIG;
  }
  c->model = M;
  const int64_t P = M->d.total;
  APPO_CUDA_TRY(cudaMalloc(&M->theta, P * 4));
  APPO_CUDA_TRY(cudaMalloc(&M->m, P * 4));
  APPO_CUDA_TRY(cudaMalloc(&M->v, P * 4));
  APPO_CUDA_TRY(cudaMalloc(&M->grad, P * 4));
  for (int k = 0; k < Model::kPub; ++k) {
    APPO_CUDA_TRY(cudaMalloc(&M->pub_bf16[k], P * 2));
    APPO_CUDA_TRY(cudaMalloc(&M->pub_f32[k], P * 4));
    APPO_CUDA_TRY(cudaMalloc(&M->pub_c1h[k], (size_t)32 * M->d.K1 * 2));
    APPO_CUDA_TRY(cudaMalloc(&M->pub_c1b[k], 32 * 4));
    APPO_CUDA_TRY(cudaMalloc(&M->pub_wt2[k], (size_t)4 * 32 * 256 * 2));
    APPO_CUDA_TRY(cudaMalloc(&M->pub_wt3[k], (size_t)4 * 64 * 512 * 2));
    APPO_CUDA_TRY(cudaEventCreateWithFlags(&M->ready_ev[k], cudaEventDisableTiming));
  }
  M->sample_key = host_derive_seed(c->seed, 0x9900);
  APPO_CUDA_TRY(cudaMallocHost(&M->ring_host, sizeof(double) * Model::kRing * Model::kRingStride));
  for (int k = 0; k < Model::kRing; ++k)
    APPO_CUDA_TRY(cudaEventCreateWithFlags(&M->ring_ev[k], cudaEventDisableTiming));
  std::vector<float> th;
  init_params_host(M->d, c->seed, th);
  return appo_params_set(static_cast<appo_ctx*>(c), th.data(), 0);
}

void model_destroy(Ctx* c) {
  Model* M = c->model;
  if (!M) return;
  cudaFree(M->theta);
  cudaFree(M->m);
  cudaFree(M->v);
  cudaFree(M->grad);
  for (int k = 0; k < Model::kPub; ++k) {
    cudaFree(M->pub_bf16[k]);
    cudaFree(M->pub_f32[k]);
    cudaFree(M->pub_c1h[k]);
    cudaFree(M->pub_c1b[k]);
    cudaFree(M->pub_wt2[k]);
    cudaFree(M->pub_wt3[k]);
    if (M->ready_ev[k]) cudaEventDestroy(M->ready_ev[k]);
  }
  if (M->ring_host) cudaFreeHost(M->ring_host);
  for (int k = 0; k < Model::kRing; ++k)
    if (M->ring_ev[k]) cudaEventDestroy(M->ring_ev[k]);
  if (M->sl.col1) cudaFree(M->sl.col1);
  if (M->sl.h_stats) cudaFreeHost(M->sl.h_stats);
  // readers of shared contexts still alive (contract: destroy those first)
  for (Reader* r : M->readers) reader_free(r);
  M->readers.clear();
  delete M;
  c->model = nullptr;
}

#define MODEL_OR_RETURN(ctx)                                                        \
  do {                                                                              \
    APPO_REQUIRE((ctx) != nullptr, APPO_ERR_CONTRACT, "null appo_ctx");             \
    APPO_REQUIRE((ctx)->model != nullptr, APPO_ERR_CONTRACT,                        \
                 "context was created without a model desc");                       \
    APPO_CUDA_TRY(cudaSetDevice((ctx)->device));                                    \
  } while (0)

extern "C" {

int64_t appo_param_count(const appo_model_desc* desc) {
  if (!desc) return -1;
  Dims d;
  if (make_dims(*desc, &d)) return -1;
  return d.total;
}

int appo_slot_layout(const appo_model_desc* desc, uint64_t* out10) {
  APPO_REQUIRE(desc && out10, APPO_ERR_CONTRACT, "slot_layout: null argument");
  Dims d;
  int st = make_dims(*desc, &d);
  if (st) return st;
  for (int i = 0; i < 10; ++i) out10[i] = d.slot[i];
  return APPO_OK;
}

int appo_params_set(appo_ctx* ctx, const float* h_src, int64_t version) {
  MODEL_OR_RETURN(ctx);
  Model* M = ctx->model;
  const int64_t P = M->d.total;
  APPO_REQUIRE(h_src != nullptr, APPO_ERR_CONTRACT, "params_set: null source");
  std::vector<uint16_t> bf(P);
  for (int64_t i = 0; i < P; ++i) bf[i] = host_f2bf(h_src[i]);
  APPO_CUDA_TRY(cudaDeviceSynchronize());  // no stream may be reading the published copies
  APPO_CUDA_TRY(cudaMemcpy(M->theta, h_src, P * 4, cudaMemcpyHostToDevice));
  APPO_CUDA_TRY(cudaMemset(M->m, 0, P * 4));
  APPO_CUDA_TRY(cudaMemset(M->v, 0, P * 4));
  for (int k = 0; k < Model::kPub; ++k) {
    APPO_CUDA_TRY(cudaMemcpy(M->pub_f32[k], h_src, P * 4, cudaMemcpyHostToDevice));
    APPO_CUDA_TRY(cudaMemcpy(M->pub_bf16[k], bf.data(), P * 2, cudaMemcpyHostToDevice));
  }
  for (int k = 0; k < Model::kPub; ++k)
    TRY(k_publish_derived(ctx, M->pub_bf16[k], M->pub_f32[k], M->d, M->pub_c1h[k], M->pub_c1b[k],
                          M->pub_wt2[k], M->pub_wt3[k]));
  APPO_CUDA_TRY(ctx_streams_sync(ctx));
  M->version = version;
  M->adam_t = 0;
  M->published = 0;
  M->published_prev = 0;
  for (int k = 0; k < Model::kPub; ++k) M->pub_version[k] = version;
  return APPO_OK;
}

int appo_params_get(appo_ctx* ctx, float* h_dst, int64_t* version_out) {
  MODEL_OR_RETURN(ctx);
  Model* M = ctx->model;
  APPO_CUDA_TRY(ctx_streams_sync(ctx));
  if (h_dst)
    APPO_CUDA_TRY(cudaMemcpy(h_dst, M->theta, M->d.total * 4, cudaMemcpyDeviceToHost));
  if (version_out) *version_out = M->version;
  return APPO_OK;
}

int appo_adam_get(appo_ctx* ctx, float* h_m, float* h_v, int64_t* t_out) {
  MODEL_OR_RETURN(ctx);
  Model* M = ctx->model;
  APPO_CUDA_TRY(ctx_streams_sync(ctx));
  if (h_m) APPO_CUDA_TRY(cudaMemcpy(h_m, M->m, M->d.total * 4, cudaMemcpyDeviceToHost));
  if (h_v) APPO_CUDA_TRY(cudaMemcpy(h_v, M->v, M->d.total * 4, cudaMemcpyDeviceToHost));
  if (t_out) *t_out = M->adam_t;
  return APPO_OK;
}

int appo_adam_set(appo_ctx* ctx, const float* h_m, const float* h_v, int64_t t) {
  MODEL_OR_RETURN(ctx);
  Model* M = ctx->model;
  APPO_CUDA_TRY(ctx_streams_sync(ctx));
  if (h_m) APPO_CUDA_TRY(cudaMemcpy(M->m, h_m, M->d.total * 4, cudaMemcpyHostToDevice));
  if (h_v) APPO_CUDA_TRY(cudaMemcpy(M->v, h_v, M->d.total * 4, cudaMemcpyHostToDevice));
  M->adam_t = t;
  return APPO_OK;
}

// After theta / m / v of dst were overwritten on dst's stream: derive and
// publish the inference copy into buffer `next`, adopt the Adam step count
// (copy_weights copies d.adam = s.adam, runner.hpp:221-222) and count the
// publish as dst's next version.  (The reference republishes with dst's
// unchanged version, so its policy workers keep the old weights until the next
// SGD step; here inference switches to the copied weights at once.)
static int publish_copied(appo_ctx* dst, int next, int64_t adam_t) {
  Model* D = dst->model;
  const int64_t P = D->d.total;
  cudaStream_t st = dst->stream;
  APPO_CUDA_TRY(cudaMemcpyAsync(D->pub_f32[next], D->theta, P * 4, cudaMemcpyDeviceToDevice, st));
  TRY(k_f32_to_bf16(dst, 1, D->theta, P, D->pub_bf16[next], P, (int)P));
  TRY(k_publish_derived(dst, D->pub_bf16[next], D->pub_f32[next], D->d, D->pub_c1h[next],
                        D->pub_c1b[next], D->pub_wt2[next], D->pub_wt3[next]));
  APPO_CUDA_TRY(cudaEventRecord(D->ready_ev[next], st));
  D->adam_t = adam_t;
  D->pub_version[next] = D->version + 1;
  D->published_prev = D->published;
  D->published = next;
  D->version += 1;  // ParamStore::publish of the copied weights
  return APPO_OK;
}

// PbtController's copy_weights (runner.hpp:211-219): dst takes src's theta and
// Adam state and publishes them as its next version.  Device to device (peer
// copy over NVLink when the learners live on different GPUs), ordered after
// src's queued work; dst must have no uncollected learner steps.
int appo_params_copy(appo_ctx* dst, appo_ctx* src) {
  MODEL_OR_RETURN(dst);
  MODEL_OR_RETURN(src);
  Model* D = dst->model;
  Model* S = src->model;
  APPO_REQUIRE(dst != src && D != S, APPO_ERR_CONTRACT, "params_copy: same learner");
  APPO_REQUIRE(D->d.total == S->d.total && dst->desc.obs_c == src->desc.obs_c &&
                   dst->desc.obs_h == src->desc.obs_h && dst->desc.obs_w == src->desc.obs_w &&
                   dst->desc.n_actions == src->desc.n_actions,
               APPO_ERR_CONFIG, "params_copy: different model shapes");
  APPO_REQUIRE(D->pending == 0, APPO_ERR_CONTRACT,
               "params_copy: collect the destination's learner steps first");
  const int64_t P = D->d.total;
  // src's published state is final once its stream drained (its version and
  // adam_t are host values advanced at submit)
  APPO_CUDA_TRY(cudaSetDevice(src->device));
  APPO_CUDA_TRY(ctx_streams_sync(src));
  APPO_CUDA_TRY(cudaSetDevice(dst->device));
  cudaStream_t st = dst->stream;
  const int next = (D->published + 1) % Model::kPub;
  TRY(wait_readers(D, st, next));
  auto copy = [&](float* to, const float* from) -> int {
    if (dst->device == src->device)
      APPO_CUDA_TRY(cudaMemcpyAsync(to, from, P * 4, cudaMemcpyDeviceToDevice, st));
    else
      APPO_CUDA_TRY(cudaMemcpyPeerAsync(to, dst->device, from, src->device, P * 4, st));
    return APPO_OK;
  };
  TRY(copy(D->theta, S->theta));
  TRY(copy(D->m, S->m));
  TRY(copy(D->v, S->v));
  return publish_copied(dst, next, S->adam_t);
}

// The published state a peer PROCESS imports (appo_params_export/_import):
// CUDA IPC handles of the exporter's theta / m / v plus the host values that
// go with them.  Fixed layout inside APPO_STATE_HANDLE_BYTES.
struct StateHandle {
  uint64_t magic;
  int64_t pid, device, n_params, adam_t, version;
  uint64_t spec_hash;
  cudaIpcMemHandle_t theta, m, v;
};
static_assert(sizeof(StateHandle) <= APPO_STATE_HANDLE_BYTES, "state handle too large");
constexpr uint64_t kStateMagic = 0x31455441545341ull;  // "ASTATE1"

int appo_params_export(appo_ctx* ctx, void* handle_out) {
  MODEL_OR_RETURN(ctx);
  APPO_REQUIRE(handle_out != nullptr, APPO_ERR_CONTRACT, "params_export: null handle");
  Model* M = ctx->model;
  APPO_REQUIRE(M->pending == 0, APPO_ERR_CONTRACT,
               "params_export: collect the learner steps first");
  APPO_CUDA_TRY(ctx_streams_sync(ctx));  // the exported state is final
  StateHandle h{};
  h.magic = kStateMagic;
  h.pid = (int64_t)getpid();
  h.device = ctx->device;
  h.n_params = M->d.total;
  h.adam_t = M->adam_t;
  h.version = M->version;
  h.spec_hash = appo_model_spec_hash(&ctx->desc);
  APPO_CUDA_TRY(cudaIpcGetMemHandle(&h.theta, M->theta));
  APPO_CUDA_TRY(cudaIpcGetMemHandle(&h.m, M->m));
  APPO_CUDA_TRY(cudaIpcGetMemHandle(&h.v, M->v));
  std::memset(handle_out, 0, APPO_STATE_HANDLE_BYTES);
  std::memcpy(handle_out, &h, sizeof(h));
  return APPO_OK;
}

// Opened peer allocations, kept for the life of the process (PBT exchanges
// repeat between the same learners; opening a handle costs milliseconds).
static void* open_peer(const cudaIpcMemHandle_t& mh, int device, int* status) {
  static std::mutex mu;
  static std::map<std::pair<std::string, int>, void*> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(std::string(mh.reserved, sizeof(mh.reserved)), device);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  void* p = nullptr;
  const cudaError_t e = cudaIpcOpenMemHandle(&p, mh, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    set_error(std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    *status = APPO_ERR_RESOURCE;
    return nullptr;
  }
  cache[key] = p;
  return p;
}

int appo_params_import(appo_ctx* dst, const void* handle) {
  MODEL_OR_RETURN(dst);
  APPO_REQUIRE(handle != nullptr, APPO_ERR_CONTRACT, "params_import: null handle");
  StateHandle h;
  std::memcpy(&h, handle, sizeof(h));
  APPO_REQUIRE(h.magic == kStateMagic, APPO_ERR_CONTRACT, "params_import: not a state handle");
  APPO_REQUIRE(h.pid != (int64_t)getpid(), APPO_ERR_CONTRACT,
               "params_import: exporter is this process (use appo_params_copy)");
  Model* D = dst->model;
  APPO_REQUIRE(h.n_params == D->d.total && h.spec_hash == appo_model_spec_hash(&dst->desc),
               APPO_ERR_CONFIG, "params_import: different model shapes");
  APPO_REQUIRE(D->pending == 0, APPO_ERR_CONTRACT,
               "params_import: collect the destination's learner steps first");
  int st = APPO_OK;
  const float* th = static_cast<const float*>(open_peer(h.theta, dst->device, &st));
  const float* m = th ? static_cast<const float*>(open_peer(h.m, dst->device, &st)) : nullptr;
  const float* v = m ? static_cast<const float*>(open_peer(h.v, dst->device, &st)) : nullptr;
  if (!v) return st;
  const int64_t P = D->d.total;
  cudaStream_t s = dst->stream;
  const int next = (D->published + 1) % Model::kPub;
  TRY(wait_readers(D, s, next));
  // unified addressing: same-GPU device copy or NVLink peer copy
  APPO_CUDA_TRY(cudaMemcpyAsync(D->theta, th, P * 4, cudaMemcpyDefault, s));
  APPO_CUDA_TRY(cudaMemcpyAsync(D->m, m, P * 4, cudaMemcpyDefault, s));
  APPO_CUDA_TRY(cudaMemcpyAsync(D->v, v, P * 4, cudaMemcpyDefault, s));
  TRY(publish_copied(dst, next, h.adam_t));
  // the exporter may resume once this returns (its state was read)
  APPO_CUDA_TRY(cudaStreamSynchronize(s));
  return APPO_OK;
}

int64_t appo_params_version(appo_ctx* ctx) {
  return (ctx && ctx->model) ? ctx->model->version : -1;
}

int appo_policy_forward(appo_ctx* ctx, int B, const uint8_t* d_obs, const float* d_h_in,
                        uint64_t rng_counter0, int32_t* d_actions, float* d_logp,
                        float* d_h_out, float* d_values, float* d_logits,
                        int64_t* h_version_out) {
  MODEL_OR_RETURN(ctx);
  Model* M = ctx->model;
  APPO_REQUIRE(B >= 0, APPO_ERR_CONTRACT, "policy_forward: batch must be >= 0");
  if (h_version_out) *h_version_out = M->pub_version[M->published];
  if (B == 0) return APPO_OK;
  APPO_REQUIRE(d_obs && d_h_in && d_actions && d_logp && d_h_out && d_values, APPO_ERR_CONTRACT,
               "policy_forward: null buffer");
  APPO_REQUIRE((reinterpret_cast<uintptr_t>(d_obs) & 3) == 0, APPO_ERR_CONTRACT,
               "policy_forward: obs must be 4-byte aligned");
  return sampler_infer(ctx, d_obs, M->d.obs_dim, B, d_h_in, rng_counter0, d_actions, d_logp,
                       d_h_out, d_values, d_logits, h_version_out);
}

// h_slot_ids != null: ids from the host (FIFO order given by the caller);
// else ids popped on the device from rq (FIFO arrival order) and, when fq is
// set, returned to fq after the last kernel reading the slots.
// GEMM tile width override for A/B sweeps of the learner backward
// (APPO_BN_<name>=32/64/128/192/256; unset = the measured default)
static int bn_env(const char* name, int dflt) {
  const char* v = getenv(name);
  if (!v || !v[0]) return dflt;
  const int b = atoi(v);
  return (b == 32 || b == 64 || b == 128 || b == 192 || b == 256) ? b : dflt;
}

// ---- learner side stream ----
// The backward's weight-gradient kernels (dW_ih, dW_hh, FC, conv3, conv2)
// depend on the input-gradient chain (dx -> FC dgrad -> conv3 dgrad -> conv2
// dgrad -> conv1 wgrad) but nothing in the chain depends on them, so they run
// on a side stream as soon as their inputs exist and fill the SMs the chain's
// kernels leave idle; the main stream joins before the optimizer.  Every
// kernel writes disjoint outputs (bias sums have their own counters), the side
// stream has its own split-K workspace, so the results are bit-identical to
// the serial order.  appo_ctx_set_learner_fork(ctx, 0) (or the env default
// APPO_LEARNER_FORK=0) keeps everything on one stream.

static int side_init(Ctx* c) {
  if (c->side_stream) return APPO_OK;
  // the main stream's priority (measured: one step below it lets the
  // concurrently running sampler delay the weight gradients the join waits
  // for, 12.26 -> 11.98 M frames/s); APPO_SIDE_PRIO=+/- one step below/above
  int prio = 0, least = 0, greatest = 0;
  APPO_CUDA_TRY(cudaStreamGetPriority(c->stream, &prio));
  APPO_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  const char* sp = getenv("APPO_SIDE_PRIO");
  if (sp && sp[0] == '+' && prio < least) prio += 1;
  if (sp && sp[0] == '-' && prio > greatest) prio -= 1;
  APPO_CUDA_TRY(cudaStreamCreateWithPriority(&c->side_stream, cudaStreamNonBlocking, prio));
  for (auto& e : c->side_ev) APPO_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  APPO_CUDA_TRY(cudaEventCreateWithFlags(&c->adam_tail_ev, cudaEventDisableTiming));
  return APPO_OK;
}

// record on `from`, wait on `to`
static int side_edge(Ctx* c, cudaStream_t from, cudaStream_t to) {
  cudaEvent_t e = c->side_ev[c->side_ev_next++ % Ctx::kSideEvents];
  APPO_CUDA_TRY(cudaEventRecord(e, from));
  APPO_CUDA_TRY(cudaStreamWaitEvent(to, e, 0));
  return APPO_OK;
}

// launches inside the scope go to the side stream with the side workspace
struct OnSide {
  Ctx* c;
  cudaStream_t main_stream;
  float* main_ws;
  size_t main_ws_bytes;
  explicit OnSide(Ctx* ctx) : c(ctx), main_stream(ctx->stream), main_ws(ctx->d_ws),
                              main_ws_bytes(ctx->ws_bytes) {
    c->stream = c->side_stream;
    c->d_ws = c->side_ws;
    c->ws_bytes = c->side_ws_bytes;
    c->on_side = true;
  }
  ~OnSide() {
    c->side_ws = c->d_ws;
    c->side_ws_bytes = c->ws_bytes;
    c->on_side = false;
    c->stream = main_stream;
    c->d_ws = main_ws;
    c->ws_bytes = main_ws_bytes;
  }
};

static int learner_submit_impl(appo_ctx* ctx, const void* d_region, uint64_t slot_bytes,
                               const int32_t* h_slot_ids, appo_slotq* rq, appo_slotq* fq,
                               int n_traj, const appo_hparams* hp) {
  MODEL_OR_RETURN(ctx);
  Model* M = ctx->model;
  const Dims& d = M->d;
  APPO_REQUIRE(hp && d_region && (h_slot_ids || rq) && n_traj >= 1, APPO_ERR_CONTRACT,
               "learner_step: bad arguments");
  APPO_REQUIRE(!rq || (uint32_t)n_traj <= rq->capacity, APPO_ERR_CONTRACT,
               "learner_step: minibatch larger than the ready queue");
  APPO_REQUIRE(slot_bytes >= d.slot[9], APPO_ERR_CONTRACT,
               "learner_step: slot_bytes smaller than the layout v2 slot");
  APPO_REQUIRE(n_traj <= 4096, APPO_ERR_CONTRACT, "learner_step: at most 4096 trajectories");
  // VTraceConfig / ClipConfig validation (offpolicy.hpp:23-44)
  APPO_REQUIRE(hp->rho_bar >= hp->c_bar && hp->c_bar > 0.0f, APPO_ERR_CONFIG,
               "vtrace requires rho_bar >= c_bar > 0");
  APPO_REQUIRE(hp->gamma > 0.0f && hp->gamma <= 1.0f, APPO_ERR_CONFIG,
               "discount must be in (0,1]");
  APPO_REQUIRE(0.0f < hp->clip_low && hp->clip_low < 1.0f && 1.0f < hp->clip_high,
               APPO_ERR_CONFIG, "ppo clip requires 0 < low < 1 < high");
  APPO_REQUIRE(hp->adv_source >= 0 && hp->adv_source <= 2, APPO_ERR_CONFIG,
               "adv_source must be 0 (vtrace), 1 (nstep) or 2 (gae)");
  const int T = d.T;
  const int B = n_traj * T;
  const int R = B + n_traj;
  Scratch& s = M->sl;
  TRY(alloc_scratch(ctx, M, s, R, n_traj, true));
  cudaStream_t st = ctx->stream;
  const int pub = M->published;
  const uint16_t* wb = M->pub_bf16[pub];
  // this step publishes into the oldest of the kPub copies: wait (here, ahead
  // of the step's kernels, so no event wait splits their PDL chain) for every
  // inference that may still read it -- readers only take the newest copy, so
  // all of them were enqueued before this step
  const int next = (pub + 1) % Model::kPub;
  TRY(wait_readers(M, st, next));
  const float* th = M->theta;  // fp32 master (== pub_f32[pub])
  const uint8_t* region = static_cast<const uint8_t*>(d_region);

  // pinned ring slot for this step's slot ids (H2D) and stats (D2H)
  const int ring = M->ring_pos;
  M->ring_pos = (M->ring_pos + 1) % Model::kRing;
  APPO_CUDA_TRY(cudaEventSynchronize(M->ring_ev[ring]));
  double* h_st = M->ring_host + (size_t)ring * Model::kRingStride;
  int32_t* h_ids = reinterpret_cast<int32_t*>(h_st + 16);
  int* q_ok = reinterpret_cast<int*>(ctx->d_counter + 9);
  if (h_slot_ids) {
    std::memcpy(h_ids, h_slot_ids, sizeof(int32_t) * n_traj);
    APPO_CUDA_TRY(cudaMemcpyAsync(s.slot_ids, h_ids, sizeof(int32_t) * n_traj,
                                  cudaMemcpyHostToDevice, st));
  } else {
    TRY(slotq_pop_launch(ctx, rq, s.slot_ids, n_traj, q_ok));
  }
  SlotOffsets off;
  std::memcpy(&off, d.slot, sizeof(off));
  TRY(k_gather_slots(ctx, n_traj, T, region, slot_bytes, s.slot_ids, off, s.act, s.rew, s.blogp,
                     s.done, s.ver, s.hcur));

  // ---- forward: encoder over all T steps + bootstrap obs ----
  ObsSrc src;
  src.base = region;
  src.slot_ids = s.slot_ids;
  src.slot_bytes = slot_bytes;
  src.obs_off = d.slot[0];
  src.boot_off = d.slot[7];
  src.T = T;
  src.n_traj = n_traj;
  if (h_slot_ids) {
    int mx = 0;
    for (int i = 0; i < n_traj; ++i) mx = h_slot_ids[i] > mx ? h_slot_ids[i] : mx;
    src.n_slots = mx + 1;
  } else {
    src.n_slots = rq->n_slots;
  }
  src.obs_dim = d.obs_dim;
  // learner: every convolution gathers its input by TMA (so do the weight
  // gradients: conv1_wgrad_implicit, conv_taps_wgrad) -- no im2col matrices
  cudaEvent_t tail = ctx->adam_tail_pending ? ctx->adam_tail_ev : nullptr;
  ctx->adam_tail_pending = false;
  TRY(encoder_forward(ctx, M, s, src, R, wb, th, pub, /*implicit=*/false, /*learner=*/true,
                      /*gate_proj=*/true, tail));

  // ---- GRU unrolled over T steps (+ bootstrap step) ----
  const bool seq = gru_seq_supported(n_traj);
  Epilogue g;
  g.flags = EPI_BIAS;
  g.bias = th + d.off_bhh;
  g.out = s.gh;
  g.ldo = kGates;
  if (seq)
    TRY(k_gru_seq_fwd(ctx, n_traj, T, s.gi, wb + d.off_whh, th + d.off_bhh, s.done, s.hcur,
                      s.hcur_bf, s.core, s.core_bf, s.gates, s.hin, s.hbf));
  for (int t = 0; !seq && t <= T; ++t) {
    TRY(k_stage_h(ctx, n_traj, T, t, s.hcur, s.hin, s.hbf));
    const uint16_t* a = (t < T) ? s.hbf + (size_t)t * kHidden : s.hbf + (size_t)B * kHidden;
    const int64_t lda = (t < T) ? (int64_t)T * kHidden : kHidden;
    TRY(gemm_bf16(ctx, n_traj, kGates, kHidden, Operand{a, lda, false},
                  Operand{wb + d.off_whh, kHidden, false}, g, 128));
    TRY(k_gru_train(ctx, n_traj, T, t, s.gi, s.gh, s.done, s.hcur, s.core, s.core_bf, s.gates));
  }
  LossHP lh{hp->clip_low, hp->clip_high, hp->value_coef, hp->entropy_coef};
  float* G = M->grad;
  // weight gradients on the side stream (ctx->fork), the
  // input-gradient chain (and BPTT) on the main stream
  const bool fork = seq && ctx->fork;
  static const int bn_dw = bn_env("APPO_BN_DW", 64), bn_dx = bn_env("APPO_BN_DX", 64),
                   bn_fcw = bn_env("APPO_BN_FCW", 64), bn_fcd = bn_env("APPO_BN_FCD", 128);
  if (fork) TRY(side_init(ctx));
  auto to_side = [&]() -> int {
    return fork ? side_edge(ctx, ctx->stream, ctx->side_stream) : APPO_OK;
  };
  auto run_side = [&](auto&& f) -> int {
    if (!fork) return f();
    OnSide on(ctx);
    return f();
  };
  if (traj_loss_supported(n_traj, T, d.A, hp->normalize_adv != 0)) {
    // heads, targets, loss and heads backward fused per trajectory (traj_loss.cu)
    // no gradient memset on this path: every entry of G is written (not
    // accumulated) by the kernels below -- checked by running the learner
    // parity tests with G pre-filled with NaN
    const bool gae = hp->adv_source == 1 || hp->adv_source == 2;
    const float lam = hp->adv_source == 1 ? 1.0f : hp->gae_lambda;
    TRY(k_traj_loss(ctx, n_traj, T, d.A, s.core, th + d.off_wpi, th + d.off_bpi, th + d.off_wv,
                    th + d.off_bv, s.act, s.rew, s.blogp, s.done, s.ver, M->version, hp->gamma,
                    hp->rho_bar, hp->c_bar, gae, lam, lh, s.logits, s.values, s.vt, s.pg, s.adv,
                    s.dcore, s.colsum_part, s.stats, G + d.off_wpi, G + d.off_bpi, G + d.off_wv,
                    G + d.off_bv, !fork));
    if (fork) {
      // the head gradients' partial sums are reduced beside BPTT
      TRY(to_side());
      TRY(run_side([&]() -> int {
        return k_heads_grad_reduce(ctx, d.A, n_traj, s.colsum_part, G + d.off_wpi,
                                   G + d.off_bpi, G + d.off_wv, G + d.off_bv);
      }));
    }
  } else {
    TRY(k_heads_fwd(ctx, R, d.A, s.core, th + d.off_wpi, th + d.off_bpi, th + d.off_wv,
                    th + d.off_bv, s.logits, s.values, B, s.act, s.tlogp, s.ent));

    // ---- targets: logp/entropy, V-trace, advantages ----
    TRY(launch_vtrace(ctx, n_traj, T, s.rew, s.values, s.values + B, s.tlogp, s.blogp, s.done,
                      hp->gamma, hp->rho_bar, hp->c_bar, s.vt, s.pg, nullptr, nullptr));
    const float* adv = s.pg;
    if (hp->adv_source == 1 || hp->adv_source == 2) {
      const float lam = hp->adv_source == 1 ? 1.0f : hp->gae_lambda;
      TRY(launch_gae(ctx, n_traj, T, s.rew, s.values, s.values + B, s.done, hp->gamma, lam, s.adv,
                     nullptr));
      adv = s.adv;
    } else if (hp->normalize_adv) {
      APPO_CUDA_TRY(cudaMemcpyAsync(s.adv, s.pg, sizeof(float) * B, cudaMemcpyDeviceToDevice, st));
      adv = s.adv;
    }
    if (hp->normalize_adv) TRY(k_normalize(ctx, B, s.adv));

    // ---- loss and its gradient wrt logits / value ----
    TRY(k_ppo_loss(ctx, B, d.A, s.logits, s.values, s.act, s.blogp, adv, s.vt, lh, s.dlog,
                   s.dhead, s.stats, s.ver, M->version));

    APPO_CUDA_TRY(cudaMemsetAsync(G, 0, d.total * 4, st));

    // ---- heads backward: dcore + head weight / bias gradients, one launch ----
    TRY(k_heads_bwd_fused(ctx, B, d.A, s.dlog, s.core, th + d.off_wpi, th + d.off_wv, s.dcore,
                          s.colsum_part, G + d.off_wpi, G + d.off_bpi, G + d.off_wv, G + d.off_bv));
  }

  // bias gradients of fc / conv layers, fused into the kernels producing /
  // reading their dz (deterministic fixed-point sums, model_kernels.cu)
  auto bias_out = [&](int k, float* out, int N) {
    BiasOut b;
    b.out = out;
    b.acc = s.bias_acc + (size_t)k * kBiasAccCols;
    b.counter = s.bias_cnt + k;
    b.N = N;
    return b;
  };

  // ---- BPTT through the GRU ----
  if (seq)
    TRY(k_gru_seq_bwd(ctx, n_traj, T, s.dcore, s.done, s.gates, s.hin, wb + d.off_whh, s.dghx,
                      s.dgi, s.dgh, G + d.off_bih, G + d.off_bhh));
  else
    APPO_CUDA_TRY(cudaMemsetAsync(s.dnext, 0, sizeof(float) * n_traj * kHidden, st));
  if (!seq) {
    Epilogue e;
    e.flags = EPI_ACCUM;
    e.out = s.dnext;
    e.ldo = kHidden;
    for (int t = T - 1; t >= 0; --t) {
      TRY(k_gru_bwd(ctx, n_traj, T, t, s.dcore, s.done, s.gates, s.hin, s.dnext, s.dgi, s.dgh));
      if (t == 0) break;  // dh wrt h0 is not needed (h0 is data)
      TRY(gemm_bf16(ctx, n_traj, kHidden, kGates,
                    Operand{s.dgh + (size_t)t * kGates, (int64_t)T * kGates, false},
                    Operand{wb + d.off_whh, kHidden, true}, e, 64, 4));
    }
  }
  TRY(to_side());  // dgi, dgh, GRU bias and head gradients are final
  TRY(run_side([&]() -> int {
    // dW_ih = dgi^T x, dW_hh = dgh^T h_in, biases = column sums (64-wide N
    // tiles, no split-K: measured fastest at these shapes, scripts/gemm_sweep.py)
    Epilogue e;
    e.out = G + d.off_wih;
    e.ldo = kHidden;
    TRY(gemm_bf16(ctx, kGates, kHidden, B, Operand{s.dgi, kGates, true},
                  Operand{s.x, kHidden, true}, e, bn_dw, 1));
    e.out = G + d.off_whh;
    TRY(gemm_bf16(ctx, kGates, kHidden, B, Operand{s.dgh, kGates, true},
                  Operand{s.hbf, kHidden, true}, e, bn_dw, 1));
    if (!seq) {
      TRY(k_colsum(ctx, B, kGates, s.dgi, kGates, true, s.colsum_part, G + d.off_bih, false));
      TRY(k_colsum(ctx, B, kGates, s.dgh, kGates, true, s.colsum_part, G + d.off_bhh, false));
    }
    // data-parallel bucket 1 (GRU + heads) is final: reduce it while the
    // encoder backward runs
    return dp_bucket(ctx, G + d.off_wih, d.total - d.off_wih);
  }));
  {
    // dx = dgi . W_ih, times ELU'(fc) -> dz_fc
    Epilogue x;
    x.flags = EPI_DELU | EPI_BF16;
    x.aux = s.x;
    x.ld_aux = kHidden;
    x.out = s.dzfc;
    x.ldo = kHidden;
    {  // fc bias gradient = column sums of dz_fc, fused into this epilogue
      const BiasOut bo = bias_out(0, G + d.off_fcb, kHidden);
      x.bsum_acc = bo.acc;
      x.bsum_cnt = bo.counter;
      x.bsum_out = bo.out;
      x.bsum_mod = kHidden;
    }
    // 64-wide N tiles: 128 tiles instead of 64 on 148 SMs (22.8 -> 18.9 us measured)
    TRY(gemm_bf16(ctx, B, kHidden, kGates, Operand{s.dgi, kGates, false},
                  Operand{wb + d.off_wih, kHidden, true}, x, bn_dx));
  }
  // ---- FC backward ----
  TRY(to_side());  // dz_fc and the fc bias gradient are final
  TRY(run_side([&]() -> int {
    Epilogue e;
    e.out = G + d.off_fcw;
    e.ldo = d.F;
    TRY(gemm_bf16(ctx, kHidden, d.F, B, Operand{s.dzfc, kHidden, true},
                  Operand{s.a3, d.F, true}, e, bn_fcw, 1));
    // bucket 2 (FC weight + bias) is final
    return dp_bucket(ctx, G + d.off_fcw, d.off_wih - d.off_fcw);
  }));
  {
    Epilogue x;
    x.flags = EPI_DELU | EPI_BF16;
    x.aux = s.a3;
    x.ld_aux = d.F;
    x.out = s.dz3;
    x.ldo = d.F;
    {  // conv3 bias gradient = dz3 column sums folded over the (h, w) positions
      const BiasOut bo = bias_out(1, G + d.off_c3b, 128);
      x.bsum_acc = bo.acc;
      x.bsum_cnt = bo.counter;
      x.bsum_out = bo.out;
      x.bsum_mod = 128;
    }
    TRY(gemm_bf16(ctx, B, d.F, kHidden, Operand{s.dzfc, kHidden, false},
                  Operand{wb + d.off_fcw, d.F, true}, x, bn_fcd));
  }
  // ---- conv3 backward ----
  TRY(to_side());  // dz3 is final
  TRY(run_side([&]() -> int {
    return conv_taps_wgrad(ctx, s.a2, B, d.H2, d.W2, 64, s.dz3, d.H3, d.W3, 128, 3,
                           G + d.off_c3w);
  }));
  {
    // dz2 = ELU'(a2) * conv3^T(dz3): sub-pixel implicit GEMM (+ conv2 bias grad)
    DgradIn in;
    in.dz_next = s.dz3;
    in.wt = M->pub_wt3[pub];
    in.aprev = s.a2;
    in.dz = s.dz2;
    in.n_img = B;
    in.Ho = d.H3; in.Wo = d.W3; in.Co = 128; in.Hi = d.H2; in.Wi = d.W2; in.N = 64; in.k = 3;
    in.bias = bias_out(2, G + d.off_c2b, 64);
    TRY(conv_dgrad_s2_bf16(ctx, in));
  }
  // ---- conv2 backward ----
  static const bool conv2_engine = [] {
    const char* v = getenv("APPO_CONV2");
    return v && v[0] == 'e';
  }();
  TRY(to_side());  // dz2 is final
  TRY(run_side([&]() -> int {
    // weight gradient straight from a1 / dz2 (strided TMA windows, no col2)
    const int w2st = conv2_engine ? APPO_ERR_CONTRACT
                                  : conv2_wgrad(ctx, s.a1, B, d.H1, d.W1, s.dz2, d.H2, d.W2,
                                                G + d.off_c2w);
    if (w2st == APPO_ERR_CONTRACT)
      return conv_taps_wgrad(ctx, s.a1, B, d.H1, d.W1, 32, s.dz2, d.H2, d.W2, 64, 4,
                             G + d.off_c2w);
    return w2st;
  }));
  {
    // dz1 = ELU'(a1) * conv2^T(dz2) (+ conv1 bias grad)
    DgradIn in;
    in.dz_next = s.dz2;
    in.wt = M->pub_wt2[pub];
    in.aprev = s.a1;
    in.dz = s.dz1;
    in.n_img = B;
    in.Ho = d.H2; in.Wo = d.W2; in.Co = 64; in.Hi = d.H1; in.Wi = d.W1; in.N = 32; in.k = 4;
    in.bias = bias_out(3, G + d.off_c1b, 32);
    // shifted-view kernel (conv2.cu) at the Doom shape, else the engine path
    const int dst = conv2_engine ? APPO_ERR_CONTRACT : conv2_dgrad(ctx, in);
    if (dst == APPO_ERR_CONTRACT)
      TRY(conv_dgrad_s2_bf16(ctx, in));
    else if (dst != APPO_OK)
      return dst;
  }
  // ---- conv1 weight gradient (input is data): straight from the u8 images;
  //      im2col + GEMM only when the images cannot be TMA-staged ----
  {
    // space-to-depth form (conv1.cu), else the im2col-staging engine path
    static const bool conv1_engine = [] {
      const char* v = getenv("APPO_CONV1");
      return v && v[0] == 'e';
    }();
    int wst = conv1_engine ? APPO_ERR_CONTRACT
                           : conv1_s2d_wgrad(ctx, conv1_in(src, B, d), s.dz1, G + d.off_c1w,
                                             1.0f / 255.0f);
    if (wst == APPO_ERR_CONTRACT)
      wst = conv1_wgrad_implicit(ctx, conv1_in(src, B, d), s.dz1, G + d.off_c1w, 1.0f / 255.0f);
    if (wst == APPO_ERR_CONTRACT) {
      const int M1 = B * d.P1;
      TRY(k_im2col_u8(ctx, src, B, d, s.col1));
      Epilogue e;
      e.scale = 1.0f / 255.0f;
      e.out = G + d.off_c1w;
      e.ldo = d.K1;
      TRY(gemm_bf16(ctx, 32, d.K1, M1, Operand{s.dz1, 32, true}, Operand{s.col1, d.K1, true}, e,
                    d.K1 % 64 == 0 && d.K1 <= 256 ? d.K1 : 64,
                    splits_for(ctx, 32, d.K1, d.K1 % 64 == 0 && d.K1 <= 256 ? d.K1 : 64, M1)));
    } else if (wst != APPO_OK) {
      return wst;
    }
  }
  // the slots are no longer read: hand them back (free list, orchestrator.hpp:870)
  if (fq) TRY(slotq_push_launch(ctx, fq, s.slot_ids, 0, n_traj, q_ok));

  // join: every weight gradient is final before the reduction / optimizer
  if (fork) TRY(side_edge(ctx, ctx->side_stream, ctx->stream));

  // ---- data-parallel: last bucket (convolutions) + rejection consensus;
  //      the averaged gradient is complete before clip + Adam ----
  const int* peer_flags = nullptr;
  TRY(dp_finish(ctx, G, d.off_fcw, &peer_flags));

  // ---- global-norm clip + Adam; publish into the other buffer ----
  M->adam_t += 1;
  TRY(launch_adam(ctx, d.total, M->theta, M->m, M->v, G, M->adam_t, hp->lr, hp->beta1,
                  hp->beta2, hp->eps, hp->grad_clip, s.stats + 8, M->pub_bf16[next],
                  M->pub_f32[next], ctx->d_counter + 6, peer_flags,
                  fork ? d.off_fcw : -1));
  TRY(k_publish_derived(ctx, M->pub_bf16[next], M->pub_f32[next], d, M->pub_c1h[next],
                        M->pub_c1b[next], M->pub_wt2[next], M->pub_wt3[next]));
  // two-stream tail: the next step's convolutions need only the convolution
  // parameters (updated above with their derived operands); Adam over the rest
  // runs on the side stream beside them and the next step joins before its FC
  // forward.  The published copy, the statistics and the step's ring event
  // follow the side stream.
  cudaStream_t tail_st = st;
  if (fork) {
    TRY(side_edge(ctx, ctx->stream, ctx->side_stream));
    {
      OnSide on(ctx);
      TRY(launch_adam_rest(ctx, d.total, d.off_fcw, M->theta, M->m, M->v, G, M->adam_t, hp->lr,
                           hp->beta1, hp->beta2, hp->eps, s.stats + 8, M->pub_bf16[next],
                           M->pub_f32[next]));
    }
    tail_st = ctx->side_stream;
  }
  APPO_CUDA_TRY(cudaEventRecord(M->ready_ev[next], tail_st));
  // statistics back to the host after the kernels (a copy node between two
  // kernels would end their PDL overlap)
  APPO_CUDA_TRY(cudaMemcpyAsync(h_st, s.stats, sizeof(double) * 10, cudaMemcpyDeviceToHost,
                                tail_st));
  APPO_CUDA_TRY(cudaEventRecord(M->ring_ev[ring], tail_st));
  if (fork) {  // after the statistics copy: the next step rewrites them
    APPO_CUDA_TRY(cudaEventRecord(ctx->adam_tail_ev, ctx->side_stream));
    ctx->adam_tail_pending = true;
  }
  M->last_ring = ring;
  // Optimistic publish: the Adam kernel always rewrites pub[next] (with the
  // unchanged parameters when the step is rejected); readers on other streams
  // wait on ready_ev[next] (or take the previous buffer while it runs).
  M->pub_version[next] = M->version + 1;
  M->published_prev = M->published;
  M->published = next;
  M->version += 1;
  M->pending += 1;
  return APPO_OK;
}

int appo_learner_submit(appo_ctx* ctx, const void* d_region, uint64_t slot_bytes,
                        const int32_t* h_slot_ids, int n_traj, const appo_hparams* hp) {
  APPO_REQUIRE(h_slot_ids != nullptr, APPO_ERR_CONTRACT, "learner_step: null slot ids");
  return learner_submit_impl(ctx, d_region, slot_bytes, h_slot_ids, nullptr, nullptr, n_traj, hp);
}

int appo_learner_submit_queued(appo_ctx* ctx, const void* d_region, uint64_t slot_bytes,
                               appo_slotq* ready_q, appo_slotq* free_q, int n_traj,
                               const appo_hparams* hp) {
  APPO_REQUIRE(ready_q != nullptr, APPO_ERR_CONTRACT, "learner_step: null ready queue");
  APPO_REQUIRE(!free_q || free_q->n_slots >= ready_q->n_slots, APPO_ERR_CONTRACT,
               "learner_step: free queue smaller than the ready queue's slot range");
  return learner_submit_impl(ctx, d_region, slot_bytes, nullptr, ready_q, free_q, n_traj, hp);
}

// Waits for the submitted learner steps; reports the last one's statistics
// and any NumericError / ContractError raised on the device since the last
// collect.  Steps rejected by the device flag do not count as versions.
int appo_learner_collect(appo_ctx* ctx, appo_step_out* out) {
  MODEL_OR_RETURN(ctx);
  Model* M = ctx->model;
  const int sync_st = appo_ctx_sync(ctx);
  unsigned applied = 0;
  APPO_CUDA_TRY(cudaMemcpy(&applied, ctx->d_counter + 6, sizeof(unsigned),
                           cudaMemcpyDeviceToHost));
  const int64_t ok_steps = (int64_t)(applied - M->applied_synced);
  const int64_t rejected = M->pending - ok_steps;
  M->version -= rejected;
  M->adam_t -= rejected;
  M->applied_synced = applied;
  M->pending = 0;
  if (out) {
    std::memset(out, 0, sizeof(*out));
    if (M->last_ring >= 0) {
      const double* hs = M->ring_host + (size_t)M->last_ring * Model::kRingStride;
      out->policy_loss = hs[0];
      out->value_loss = hs[1];
      out->entropy = hs[2];
      out->total_loss = hs[3];
      out->mean_ratio = hs[4];
      out->lag_mean = hs[6];
      out->lag_max = hs[7];
      out->grad_norm = hs[8];
    }
    out->version = M->version;
  }
  return sync_st;
}

int appo_learner_step(appo_ctx* ctx, const void* d_region, uint64_t slot_bytes,
                      const int32_t* h_slot_ids, int n_traj, const appo_hparams* hp,
                      appo_step_out* out) {
  APPO_REQUIRE(out != nullptr, APPO_ERR_CONTRACT, "learner_step: null out");
  const int st = appo_learner_submit(ctx, d_region, slot_bytes, h_slot_ids, n_traj, hp);
  if (st != APPO_OK) return st;
  return appo_learner_collect(ctx, out);
}

}  // extern "C"

#include "../../include/appo_internal.h"
extern "C" int appo_dbg_model_ptrs(appo_ctx* ctx, float** theta, float** grad, void** pub_bf16) {
  MODEL_OR_RETURN(ctx);
  if (theta) *theta = ctx->model->theta;
  if (grad) *grad = ctx->model->grad;
  if (pub_bf16) *pub_bf16 = ctx->model->pub_bf16[ctx->model->published];
  return APPO_OK;
}
extern "C" int appo_dbg_copy_d2h(appo_ctx* ctx, void* h_dst, const void* d_src, uint64_t bytes) {
  APPO_REQUIRE(ctx != nullptr, APPO_ERR_CONTRACT, "null ctx");
  APPO_CUDA_TRY(cudaSetDevice(ctx->device));
  APPO_CUDA_TRY(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  APPO_CUDA_TRY(ctx_streams_sync(ctx));
  return APPO_OK;
}

// The learner's fused loss kernel (ppo_loss_kernel) on caller-supplied logits /
// values: parity of the loss and its logit / value gradient against the
// reference's compute_gradients (policy.hpp:323-375) with injected inputs.
extern "C" int appo_dbg_traj_loss(appo_ctx* ctx, int n_traj, int T, int A, const float* d_core,
                                  const float* d_wpi, const float* d_bpi, const float* d_wv,
                                  const float* d_bv, const int32_t* d_actions,
                                  const float* d_rewards, const float* d_blogp,
                                  const uint8_t* d_dones, float gamma, float rho_bar,
                                  float c_bar, int adv_source, float gae_lambda, float clip_low,
                                  float clip_high, float value_coef, float entropy_coef,
                                  float* d_logits, float* d_values, float* d_vt, float* d_pg,
                                  float* d_adv, float* d_dcore, float* d_ghead, double* h_stats8) {
  APPO_REQUIRE(ctx != nullptr && traj_loss_supported(n_traj, T, A, false), APPO_ERR_CONTRACT,
               "dbg_traj_loss: outside the fused kernel's envelope");
  APPO_CUDA_TRY(cudaSetDevice(ctx->device));
  const int B = n_traj * T;
  double* stats = nullptr;
  int64_t* ver = nullptr;
  float* part = nullptr;
  APPO_CUDA_TRY(cudaMalloc(&stats, sizeof(double) * 16));
  APPO_CUDA_TRY(cudaMalloc(&ver, sizeof(int64_t) * B));
  APPO_CUDA_TRY(cudaMalloc(&part, sizeof(float) * n_traj * (A + 1) * (kHidden + 1)));
  APPO_CUDA_TRY(cudaMemsetAsync(ver, 0, sizeof(int64_t) * B, ctx->stream));
  LossHP lh{clip_low, clip_high, value_coef, entropy_coef};
  const bool gae = adv_source == 1 || adv_source == 2;
  const float lam = adv_source == 1 ? 1.0f : gae_lambda;
  float* g = d_ghead;  // W_pi [A][512], b_pi [A], w_v [512], b_v
  int st = k_traj_loss(ctx, n_traj, T, A, d_core, d_wpi, d_bpi, d_wv, d_bv, d_actions, d_rewards,
                       d_blogp, d_dones, ver, 0, gamma, rho_bar, c_bar, gae, lam, lh, d_logits,
                       d_values, d_vt, d_pg, d_adv, d_dcore, part, stats, g, g + A * kHidden,
                       g + A * kHidden + A, g + A * kHidden + A + kHidden);
  if (st == APPO_OK) {
    APPO_CUDA_TRY(cudaMemcpyAsync(h_stats8, stats, sizeof(double) * 8, cudaMemcpyDeviceToHost,
                                  ctx->stream));
    APPO_CUDA_TRY(ctx_streams_sync(ctx));
  }
  cudaFree(stats);
  cudaFree(ver);
  cudaFree(part);
  return st;
}

extern "C" int appo_dbg_ppo_loss(appo_ctx* ctx, int B, int A, const float* d_logits,
                                 const float* d_values, const int32_t* d_actions,
                                 const float* d_blogp, const float* d_adv, const float* d_vt,
                                 float clip_low, float clip_high, float value_coef,
                                 float entropy_coef, float* d_dlog, double* h_stats8) {
  APPO_REQUIRE(ctx != nullptr && B >= 1 && A >= 1 && A < kMaxActions, APPO_ERR_CONTRACT,
               "dbg_ppo_loss: bad arguments");
  APPO_CUDA_TRY(cudaSetDevice(ctx->device));
  uint16_t* dhead = nullptr;
  double* stats = nullptr;
  int64_t* ver = nullptr;
  APPO_CUDA_TRY(cudaMalloc(&dhead, (size_t)B * 16 * 2));
  APPO_CUDA_TRY(cudaMalloc(&stats, sizeof(double) * 16));
  APPO_CUDA_TRY(cudaMalloc(&ver, sizeof(int64_t) * B));
  APPO_CUDA_TRY(cudaMemsetAsync(ver, 0, sizeof(int64_t) * B, ctx->stream));
  LossHP lh{clip_low, clip_high, value_coef, entropy_coef};
  int st = k_ppo_loss(ctx, B, A, d_logits, d_values, d_actions, d_blogp, d_adv, d_vt, lh, d_dlog,
                      dhead, stats, ver, 0);
  if (st == APPO_OK) {
    APPO_CUDA_TRY(cudaMemcpyAsync(h_stats8, stats, sizeof(double) * 8, cudaMemcpyDeviceToHost,
                                  ctx->stream));
    APPO_CUDA_TRY(ctx_streams_sync(ctx));
  }
  cudaFree(dhead);
  cudaFree(stats);
  cudaFree(ver);
  return st;
}
