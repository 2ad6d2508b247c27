// Data-parallel learner plumbing: an NCCL communicator owned by the context.
// appo_learner_step all-reduces (averages) the flat fp32 gradient over the
// ranks before the global-norm clip and Adam, so every replica applies the
// identical update and versions advance in lockstep.  The
// reference has no multi-GPU path; this replaces its single
// learner per policy (orchestrator.hpp:938-946) for one policy on N GPUs.
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
      api.ok = api.getUniqueId && api.commInitRank && api.allReduce && api.commDestroy;
    }
  }
  return api;
}

}  // namespace

// Called by the learner step between backward and Adam.
int dp_allreduce_grad(Ctx* c, float* grad, int64_t n) {
  if (!c->dp_comm || c->dp_size <= 1) return APPO_OK;
  ncclResult_t r = nccl().allReduce(grad, grad, (size_t)n, ncclFloat32, ncclAvg,
                                    static_cast<ncclComm_t>(c->dp_comm), c->stream);
  if (r != ncclSuccess) {
    set_error(std::string("ncclAllReduce: ") + nccl().getErrorString(r));
    return APPO_ERR_RESOURCE;
  }
  return APPO_OK;
}

void dp_destroy(Ctx* c) {
  if (c->dp_comm && nccl().ok) nccl().commDestroy(static_cast<ncclComm_t>(c->dp_comm));
  c->dp_comm = nullptr;
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
  return APPO_OK;
}

}  // extern "C"
