// Model state owned by a context: convnet_simple + GRU-512 + categorical head
// (DESIGN.md §2), fp32 master parameters + Adam moments, the double-buffered
// published copy read by inference (bf16 for GEMM weights, fp32 for the small
// SIMT-consumed tensors), and activation scratch sized on demand.
#pragma once
#include <stdint.h>

#include <mutex>
#include <vector>

#include "appo_common.cuh"

namespace appo_b200 {

constexpr int kHidden = 512;
constexpr int kGates = 3 * kHidden;
constexpr int kBiasCopies = 16;                  // accumulator copies per bias vector
constexpr int kBiasAccCols = 512 * kBiasCopies;  // per bias vector (N <= 512)

struct Dims {
  int C, H, W, A, T;
  int H1, W1, P1, H2, W2, P2, H3, W3, P3;
  int K1;  // C*64
  int F;   // P3*128 (flatten)
  int64_t off_c1w, off_c1b, off_c2w, off_c2b, off_c3w, off_c3b, off_fcw, off_fcb, off_wih,
      off_whh, off_bih, off_bhh, off_wpi, off_bpi, off_wv, off_bv, total;
  int64_t obs_dim;
  uint64_t slot[10];  // layout v2 offsets
};

int make_dims(const appo_model_desc& d, Dims* out);

// Scratch for a forward / learner pass over R encoder rows.
struct Scratch {
  int cap_rows = 0;  // encoder rows (images)
  int cap_traj = 0;
  uint16_t *col1 = nullptr, *a1 = nullptr, *col2 = nullptr, *a2 = nullptr, *col3 = nullptr,
           *a3 = nullptr, *x = nullptr;  // bf16
  float* gi = nullptr;                   // [R][1536]
  float* gh = nullptr;                   // [R or n_traj][1536]
  uint16_t* hbf = nullptr;               // [R][512] bf16 h inputs
  // learner-only
  float *core = nullptr, *gates = nullptr, *hin = nullptr, *hcur = nullptr;  // fp32
  uint16_t* core_bf = nullptr;
  float *logits = nullptr, *values = nullptr;
  float *tlogp = nullptr, *ent = nullptr, *vt = nullptr, *pg = nullptr, *adv = nullptr;
  float *rew = nullptr, *blogp = nullptr;
  int32_t* act = nullptr;
  uint8_t* done = nullptr;
  int64_t* ver = nullptr;
  float* dlog = nullptr;        // [B][A+1] fp32
  uint16_t* dhead = nullptr;    // [B][16] bf16
  float* dcore = nullptr;       // [B][512]
  float* dnext = nullptr;       // [n_traj][512]
  uint16_t* dghx = nullptr;     // [2][n_traj][1536] bf16 BPTT exchange (persistent GRU)
  uint16_t* hcur_bf = nullptr;  // [2][n_traj][512] bf16 h_t exchange (persistent GRU)
  uint16_t *dgi = nullptr, *dgh = nullptr;  // [B][1536] bf16
  uint16_t *dzfc = nullptr, *dz3 = nullptr, *dz2 = nullptr, *dz1 = nullptr;
  uint16_t *wt3 = nullptr, *wt2 = nullptr;  // sub-pixel dgrad weight operands
  float* headw = nullptr;       // [16][512]
  float* colsum_part = nullptr; // partials for bias grads
  unsigned long long* bias_acc = nullptr;  // [4][kBiasAccCols] fixed-point bias-gradient sums
  unsigned* bias_cnt = nullptr;            // [4] last-block counters
  int32_t* slot_ids = nullptr;
  double* stats = nullptr;      // device stats block
  double* h_stats = nullptr;    // pinned
};

struct Reader;

struct Model {
  Dims d;
  float* theta = nullptr;  // fp32 master [P]
  float* m = nullptr;
  float* v = nullptr;
  float* grad = nullptr;
  // Published inference copies, kPub-buffered: the learner writes
  // pub[(published+1)%kPub] (after waiting on every reader context's read
  // event of that buffer, recorded by its last inference that read it,
  // possibly on another stream), then flips `published` -- the device-side
  // counterpart of ParamStore's seqlock (policy.hpp:457-519): inference never
  // observes a half-written version.
  static constexpr int kPub = 8;
  uint16_t* pub_bf16[kPub] = {};
  float* pub_f32[kPub] = {};
  // conv1 operands of the published copy: fp16 weights [32][K1] and the bias
  // with the fp16-input offset removed (b - 1024/255 * sum_k W), see gemm.cu
  uint16_t* pub_c1h[kPub] = {};
  float* pub_c1b[kPub] = {};
  // sub-pixel dgrad operands of conv2 / conv3 (k_publish_derived layout)
  uint16_t* pub_wt2[kPub] = {};
  uint16_t* pub_wt3[kPub] = {};
  cudaEvent_t ready_ev[kPub] = {};  // recorded after the Adam step that wrote pub[k]
  int64_t pub_version[kPub] = {};   // parameter version held by pub[k]
  int published = 0;                // newest submitted publish
  int published_prev = 0;           // the one before (complete when `published` is in flight)
  int64_t version = 0;
  int64_t adam_t = 0;
  uint64_t sample_key = 0;
  // asynchronous learner submissions (appo_learner_submit / _collect)
  static constexpr int kRing = 8;
  static constexpr int kRingStride = 16 + 4096 / 2;  // doubles: 16 stats + 4096 slot ids
  double* ring_host = nullptr;  // pinned [kRing][kRingStride]
  cudaEvent_t ring_ev[kRing] = {};
  int ring_pos = 0;
  int last_ring = -1;
  int64_t pending = 0;
  unsigned applied_synced = 0;
  Scratch sl;  // learner scratch
  // contexts running inference on this model (the owner and its
  // appo_ctx_create_shared contexts), each with its own scratch and read events
  std::mutex readers_mu;
  std::vector<Reader*> readers;
};

// Per-context inference state: activation scratch and, per published buffer,
// the event recorded after this context's last inference read of it.  Shared
// contexts run inference concurrently on their own streams, so none of this
// may be shared between them.
struct Reader {
  Scratch s;
  cudaEvent_t read_ev[Model::kPub] = {};
};

// Make `st` wait until no reader context still reads published buffer k.
int wait_readers(Model* M, cudaStream_t st, int k);
// The ctx's reader state (created and registered with its model on first use).
Reader* reader_of(Ctx* c);
// Unregister and free the ctx's reader state (appo_ctx_destroy).
void reader_release(Ctx* c);

}  // namespace appo_b200
