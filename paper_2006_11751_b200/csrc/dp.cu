// Data-parallel learner plumbing: an NCCL communicator owned by the context.
// appo_learner_step all-reduces (averages) the flat fp32 gradient over the
// ranks before the global-norm clip and Adam, so every replica applies the
// identical update and versions advance in lockstep.  The
// reference has no multi-GPU path; this replaces its single
// learner per policy (orchestrator.hpp:938-946) for one policy on N GPUs.
//
// The gradient is reduced in three buckets in reverse layer order, each
// launched on a side stream as soon as the backward pass has finished
// writing it, so the transfers overlap the rest of the backward:
//   1. GRU + heads  [off_wih, P)      after the GRU weight gradients
//   2. FC           [off_fcw, off_wih) after the FC backward
//   3. convolutions [0, off_fcw)       after conv1's weight gradient, grouped
//      with a max-reduction of the ranks' step-rejection flags, so a step one
//      rank rejects (queue timeout, bad action, non-finite input) is rejected
//      by every rank and the replicas never diverge.
// The learner stream joins the side stream before the global-norm clip.
//
// NCCL is resolved with dlopen at init time so the process uses the NCCL that
// torch.distributed already loaded (one libnccl.so.2 per process).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "appo_common.cuh"
#include "model.cuh"

namespace appo_b200 {
namespace {

struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
      api.commInitRank =
          reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
      api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
      api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
      api.getErrorString =
          reinterpret_cast<decltype(api.getErrorString)>(dlsym(h, "ncclGetErrorString"));
      api.groupStart = reinterpret_cast<decltype(api.groupStart)>(dlsym(h, "ncclGroupStart"));
      api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(dlsym(h, "ncclGroupEnd"));
      api.ok = api.getUniqueId && api.commInitRank && api.allReduce && api.commDestroy &&
               api.groupStart && api.groupEnd;
    }
  }
  return api;
}

}  // namespace

#define NCCL_TRY(expr)                                                       \
  do {                                                                       \
    ncclResult_t _r = (expr);                                                \
    if (_r != ncclSuccess) {                                                 \
      set_error(std::string(#expr ": ") + nccl().getErrorString(_r));        \
      return APPO_ERR_RESOURCE;                                              \
    }                                                                        \
  } while (0)

bool dp_active(const Ctx* c) { return c->dp_comm != nullptr; }

// Bucket k of the gradient is complete on the learner stream: average it
// over the ranks on the side stream (ordered after everything enqueued so far).
int dp_bucket(Ctx* c, float* buf, int64_t n) {
  if (!dp_active(c)) return APPO_OK;
  const int k = c->dp_ev_next++ % Ctx::kDpEvents;
  APPO_CUDA_TRY(cudaEventRecord(c->dp_ev[k], c->stream));
  APPO_CUDA_TRY(cudaStreamWaitEvent(c->dp_stream, c->dp_ev[k], 0));
  NCCL_TRY(nccl().allReduce(buf, buf, (size_t)n, ncclFloat32, ncclAvg,
                            static_cast<ncclComm_t>(c->dp_comm), c->dp_stream));
  return APPO_OK;
}

// Last bucket + the rejection-flag consensus, then the learner stream waits
// for every bucket.  *peer_flags receives the ranks' max-reduced flags (the
// optimizer folds them into this context's flags before deciding the step).
int dp_finish(Ctx* c, float* buf, int64_t n, const int** peer_flags) {
  *peer_flags = nullptr;
  if (!dp_active(c)) return APPO_OK;
  APPO_CUDA_TRY(cudaMemcpyAsync(c->d_dp_flags, c->d_flags, sizeof(int) * kNumFlags,
                                cudaMemcpyDeviceToDevice, c->stream));
  const int k = c->dp_ev_next++ % Ctx::kDpEvents;
  APPO_CUDA_TRY(cudaEventRecord(c->dp_ev[k], c->stream));
  APPO_CUDA_TRY(cudaStreamWaitEvent(c->dp_stream, c->dp_ev[k], 0));
  ncclComm_t comm = static_cast<ncclComm_t>(c->dp_comm);
  NCCL_TRY(nccl().groupStart());
  NCCL_TRY(nccl().allReduce(buf, buf, (size_t)n, ncclFloat32, ncclAvg, comm, c->dp_stream));
  NCCL_TRY(nccl().allReduce(c->d_dp_flags, c->d_dp_flags, kNumFlags, ncclInt32, ncclMax, comm,
                            c->dp_stream));
  NCCL_TRY(nccl().groupEnd());
  const int j = c->dp_ev_next++ % Ctx::kDpEvents;
  APPO_CUDA_TRY(cudaEventRecord(c->dp_ev[j], c->dp_stream));
  APPO_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->dp_ev[j], 0));
  *peer_flags = c->d_dp_flags;
  return APPO_OK;
}

void dp_destroy(Ctx* c) {
  if (c->dp_stream) cudaStreamSynchronize(c->dp_stream);
  if (c->dp_comm && nccl().ok) nccl().commDestroy(static_cast<ncclComm_t>(c->dp_comm));
  c->dp_comm = nullptr;
  for (auto& e : c->dp_ev)
    if (e) {
      cudaEventDestroy(e);
      e = nullptr;
    }
  if (c->dp_stream) cudaStreamDestroy(c->dp_stream);
  c->dp_stream = nullptr;
  if (c->d_dp_flags) cudaFree(c->d_dp_flags);
  c->d_dp_flags = nullptr;
}

}  // namespace appo_b200

using namespace appo_b200;

extern "C" {

APPO_API int appo_dp_unique_id(char* out128) {
  APPO_REQUIRE(out128 != nullptr, APPO_ERR_CONTRACT, "dp_unique_id: null buffer");
  APPO_REQUIRE(nccl().ok, APPO_ERR_RESOURCE, "NCCL not available (libnccl.so.2)");
  ncclUniqueId id;
  ncclResult_t r = nccl().getUniqueId(&id);
  APPO_REQUIRE(r == ncclSuccess, APPO_ERR_RESOURCE, "ncclGetUniqueId failed");
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, 128);
  return APPO_OK;
}

APPO_API int appo_dp_init(appo_ctx* ctx, int nranks, int rank, const char* id128) {
  APPO_REQUIRE(ctx && id128 && nranks >= 1 && rank >= 0 && rank < nranks, APPO_ERR_CONTRACT,
               "dp_init: bad arguments");
  APPO_REQUIRE(nccl().ok, APPO_ERR_RESOURCE, "NCCL not available (libnccl.so.2)");
  APPO_CUDA_TRY(cudaSetDevice(ctx->device));
  dp_destroy(ctx);
  ncclUniqueId id;
  std::memcpy(&id, id128, 128);
  ncclComm_t comm;
  ncclResult_t r = nccl().commInitRank(&comm, nranks, id, rank);
  APPO_REQUIRE(r == ncclSuccess, APPO_ERR_RESOURCE, "ncclCommInitRank failed");
  ctx->dp_comm = comm;
  ctx->dp_size = nranks;
  ctx->dp_rank = rank;
  int lo = 0, hi = 0;
  APPO_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  APPO_CUDA_TRY(cudaStreamCreateWithPriority(&ctx->dp_stream, cudaStreamNonBlocking, hi));
  for (auto& e : ctx->dp_ev) APPO_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  APPO_CUDA_TRY(cudaMalloc(&ctx->d_dp_flags, sizeof(int) * kNumFlags));
  return APPO_OK;
}

// The gradient buckets in the order the learner reduces them (reverse layer
// order), as (offset, count) pairs over the flat parameter vector.
APPO_API int appo_dp_bucket_plan(const appo_model_desc* desc, int64_t* out_pairs, int cap,
                                 int* n_out) {
  APPO_REQUIRE(desc && out_pairs && n_out, APPO_ERR_CONTRACT, "dp_bucket_plan: null argument");
  Dims d;
  const int st = make_dims(*desc, &d);
  if (st) return st;
  const int64_t plan[3][2] = {{d.off_wih, d.total - d.off_wih},
                              {d.off_fcw, d.off_wih - d.off_fcw},
                              {0, d.off_fcw}};
  APPO_REQUIRE(cap >= 3, APPO_ERR_CONTRACT, "dp_bucket_plan: need room for 3 buckets");
  for (int i = 0; i < 3; ++i) {
    out_pairs[2 * i] = plan[i][0];
    out_pairs[2 * i + 1] = plan[i][1];
  }
  *n_out = 3;
  return APPO_OK;
}

}  // extern "C"
