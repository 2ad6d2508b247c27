// Device-resident slot queues: the ready queue between rollout writers and the
// learner, and the free list that returns consumed slots (trajstore.hpp:293-331
// assemble_minibatch over BoundedFifo ready_q, transport.hpp; release of the
// consumed slots at orchestrator.hpp:870).  The reference moves slot indices
// through host FIFOs and the learner thread blocks in pop_many; here the ids
// stay in HBM, producers enqueue from their own streams and the learner's pop
// is the first kernel of its step, so the host is off the learner's critical
// path and FIFO (arrival) order is kept.
//
// Layout: a bounded ring of `capacity` (power of two >= n_slots) entries, each
// an int32 id plus a u64 sequence word (Vyukov's bounded MPMC queue): entry at
// position p is free for the producer of ticket p when seq == p, holds a
// published id when seq == p + 1, and is handed back for ticket p + capacity by
// the consumer.  Producers reserve a contiguous ticket range with one atomic
// per push (ids of one push stay contiguous and in input order); there is one
// consumer per queue (the policy's learner, as in the reference), which waits
// until its whole minibatch is published before touching anything, so a
// timed-out pop leaves the queue exactly as it was.
#include "slotq.cuh"

#include <cuda.h>

#include <cstring>
#include <mutex>
#include <vector>

using namespace appo_b200;

#define SQ_CTX_OR_RETURN(ctx) \
  APPO_REQUIRE((ctx) != nullptr && (ctx)->d_flags != nullptr, APPO_ERR_CONTRACT, "null context")

namespace {

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void slotq_init_kernel(unsigned long long* seq, uint32_t cap) {
  APPO_PDL_ENTRY();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += gridDim.x * blockDim.x)
    seq[i] = i;
}

// One block: one reservation, ids written in input order.
__global__ void __launch_bounds__(1024)
    slotq_push_kernel(int32_t* __restrict__ ids, unsigned long long* __restrict__ seq,
                      unsigned long long* ctr, uint32_t mask, int n,
                      const int32_t* __restrict__ src, int32_t first, const int* ok,
                      int64_t timeout_ns, int* flags) {
  APPO_PDL_ENTRY();
  __shared__ unsigned long long base;
  if (ok && *ok == 0) return;
  if (threadIdx.x == 0) base = atomicAdd(ctr + 0, (unsigned long long)n);
  __syncthreads();
  const uint64_t t0 = global_ns();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned long long p = base + (unsigned long long)i;
    unsigned long long* sq = seq + (p & mask);
    // the entry is free once the consumer of ticket p - capacity handed it back
    // (always true when at most capacity ids circulate; bounded regardless)
    while (ld_acquire_u64(sq) != p) {
      if (global_ns() - t0 > (uint64_t)timeout_ns) {
        atomicOr(flags + kFlagQueue, 1);
        break;
      }
      __nanosleep(128);
    }
    ids[p & mask] = src ? src[i] : first + i;
    st_release_u64(sq, p + 1);
  }
}

// Single consumer, one block: wait until tickets [head, head + n) are all
// published, then take them (FIFO order) and hand the entries back.
__global__ void __launch_bounds__(1024)
    slotq_pop_kernel(int32_t* __restrict__ ids, unsigned long long* __restrict__ seq,
                     unsigned long long* ctr, uint32_t mask, uint32_t cap, int n, int32_t n_slots,
                     int32_t* __restrict__ out, int* ok, int64_t timeout_ns, int* flags) {
  APPO_PDL_ENTRY();
  __shared__ int timed_out;
  const unsigned long long head = *reinterpret_cast<volatile unsigned long long*>(ctr + 1);
  const uint64_t t0 = global_ns();
  if (threadIdx.x == 0) timed_out = 0;
  __syncthreads();
  for (;;) {
    int ready = 1;
    for (int i = threadIdx.x; i < n && ready; i += blockDim.x) {
      const unsigned long long p = head + (unsigned long long)i;
      ready = ld_acquire_u64(seq + (p & mask)) == p + 1;
    }
    if (__syncthreads_and(ready)) break;
    if (threadIdx.x == 0 && global_ns() - t0 > (uint64_t)timeout_ns) timed_out = 1;
    __syncthreads();
    if (timed_out) break;
    __nanosleep(256);
  }
  if (timed_out) {
    // nothing consumed: the step that follows runs on slot 0 and is rejected
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = 0;
    if (threadIdx.x == 0) {
      *ok = 0;
      atomicOr(flags + kFlagQueue, 1);
      atomicAdd(ctr + 2, 1ull);
    }
    return;
  }
  int bad = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned long long p = head + (unsigned long long)i;
    int32_t id = ids[p & mask];
    if (id < 0 || id >= n_slots) {  // a foreign id must not address outside the region
      bad = 1;
      id = 0;
    }
    out[i] = id;
    st_release_u64(seq + (p & mask), p + cap);
  }
  if (bad) atomicOr(flags + kFlagContract, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    *reinterpret_cast<volatile unsigned long long*>(ctr + 1) = head + (unsigned long long)n;
    *ok = 1;
  }
}

}  // namespace

namespace appo_b200 {

const void* kanchor_gemm();
const void* kanchor_gru();
const void* kanchor_model();
const void* kanchor_offpolicy();
const void* kanchor_optim();
const void* kanchor_sampler();
const void* kanchor_conv1();
const void* kanchor_conv2();
const void* kanchor_gru_infer();
const void* kanchor_traj_loss();

// CUDA lazy loading loads a kernel on its first launch, and that load may
// need a context-wide synchronisation; a consumer spinning on the device for
// a producer kernel that is not loaded yet would then wait for its own
// timeout.  Before any queue exists, every kernel of the library (all
// modules: one per translation unit, found through one anchor kernel each) is
// loaded explicitly.
int preload_library_kernels() {
  static uint64_t done = 0;  // one bit per device (each has its own context)
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  APPO_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 64 && (done >> dev) & 1) return APPO_OK;
  using GetModule = CUresult (*)(CUmodule*, CUfunction);
  using Count = CUresult (*)(unsigned*, CUmodule);
  using Enumerate = CUresult (*)(CUfunction*, unsigned, CUmodule);
  using Load = CUresult (*)(CUfunction);
  void* p[4] = {};
  const char* names[4] = {"cuFuncGetModule", "cuModuleGetFunctionCount",
                          "cuModuleEnumerateFunctions", "cuFuncLoad"};
  for (int i = 0; i < 4; ++i) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(names[i], &p[i], cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p[i]) {
      set_error(std::string("slot queue: driver entry point unavailable: ") + names[i]);
      return APPO_ERR_RESOURCE;
    }
  }
  const void* anchors[] = {kanchor_gemm(),      kanchor_gru(),   kanchor_model(),
                           kanchor_offpolicy(), kanchor_optim(), kanchor_sampler(),
                           kanchor_conv1(),     kanchor_conv2(), kanchor_gru_infer(),
                           kanchor_traj_loss(),
                           reinterpret_cast<const void*>(&slotq_push_kernel)};
  for (const void* a : anchors) {
    cudaFunction_t f = nullptr;
    APPO_CUDA_TRY(cudaGetFuncBySymbol(&f, a));
    CUmodule mod = nullptr;
    if (reinterpret_cast<GetModule>(p[0])(&mod, reinterpret_cast<CUfunction>(f)) != CUDA_SUCCESS) {
      set_error("slot queue: cuFuncGetModule failed");
      return APPO_ERR_RESOURCE;
    }
    unsigned n = 0;
    if (reinterpret_cast<Count>(p[1])(&n, mod) != CUDA_SUCCESS) {
      set_error("slot queue: cuModuleGetFunctionCount failed");
      return APPO_ERR_RESOURCE;
    }
    std::vector<CUfunction> fs(n);
    if (n && reinterpret_cast<Enumerate>(p[2])(fs.data(), n, mod) != CUDA_SUCCESS) {
      set_error("slot queue: cuModuleEnumerateFunctions failed");
      return APPO_ERR_RESOURCE;
    }
    for (CUfunction fn : fs)
      if (reinterpret_cast<Load>(p[3])(fn) != CUDA_SUCCESS) {
        set_error("slot queue: cuFuncLoad failed");
        return APPO_ERR_RESOURCE;
      }
  }
  if (dev < 64) done |= 1ull << dev;
  return APPO_OK;
}

int slotq_push_launch(Ctx* c, appo_slotq* q, const int32_t* d_ids, int32_t first_id, int n,
                      const int* d_ok) {
  if (n == 0) return APPO_OK;
  APPO_LAUNCH(c, slotq_push_kernel, 1, 1024, 0, q->ids, q->seq, q->ctr, q->capacity - 1, n, d_ids,
              first_id, d_ok, q->timeout_ns, c->d_flags);
  return APPO_OK;
}

int slotq_pop_launch(Ctx* c, appo_slotq* q, int32_t* d_out, int n, int* d_ok) {
  APPO_LAUNCH(c, slotq_pop_kernel, 1, 1024, 0, q->ids, q->seq, q->ctr, q->capacity - 1,
              q->capacity, n, q->n_slots, d_out, d_ok, q->timeout_ns, c->d_flags);
  return APPO_OK;
}

}  // namespace appo_b200

extern "C" {

int appo_slotq_create(int device, int32_t n_slots, int32_t capacity, double timeout_s,
                      appo_slotq** out) {
  APPO_REQUIRE(out != nullptr, APPO_ERR_CONTRACT, "slotq_create: null out");
  *out = nullptr;
  APPO_REQUIRE(n_slots >= 1, APPO_ERR_CONTRACT, "slotq_create: n_slots must be >= 1");
  APPO_REQUIRE(timeout_s > 0.0 && timeout_s <= 3600.0, APPO_ERR_CONTRACT,
               "slotq_create: timeout must be in (0, 3600] s");
  uint32_t cap = 1;
  const int64_t want = capacity > n_slots ? capacity : n_slots;
  APPO_REQUIRE(want <= (1 << 30), APPO_ERR_CONTRACT, "slotq_create: capacity too large");
  while ((int64_t)cap < want) cap <<= 1;
  APPO_CUDA_TRY(cudaSetDevice(device));
  {
    const int pst = preload_library_kernels();
    if (pst != APPO_OK) return pst;
  }
  auto* q = new appo_slotq;
  q->device = device;
  q->capacity = cap;
  q->n_slots = n_slots;
  q->timeout_ns = (int64_t)(timeout_s * 1e9);
  if (cudaMalloc(&q->ids, sizeof(int32_t) * cap) != cudaSuccess ||
      cudaMalloc(&q->seq, sizeof(unsigned long long) * cap) != cudaSuccess ||
      cudaMalloc(&q->ctr, sizeof(unsigned long long) * 4) != cudaSuccess) {
    cudaFree(q->ids);
    cudaFree(q->seq);
    cudaFree(q->ctr);
    delete q;
    set_error("slotq_create: out of device memory");
    return APPO_ERR_RESOURCE;
  }
  cudaMemset(q->ctr, 0, sizeof(unsigned long long) * 4);
  cudaMemset(q->ids, 0, sizeof(int32_t) * cap);
  slotq_init_kernel<<<(cap + 255) / 256 < 1184 ? (cap + 255) / 256 : 1184, 256>>>(q->seq, cap);
  APPO_CUDA_TRY(cudaDeviceSynchronize());
  *out = q;
  return APPO_OK;
}

int appo_slotq_destroy(appo_slotq* q) {
  if (!q) return APPO_OK;
  cudaSetDevice(q->device);
  cudaDeviceSynchronize();
  cudaFree(q->ids);
  cudaFree(q->seq);
  cudaFree(q->ctr);
  delete q;
  return APPO_OK;
}

int appo_slotq_push(appo_ctx* ctx, appo_slotq* q, const int32_t* d_ids, int n) {
  SQ_CTX_OR_RETURN(ctx);
  APPO_REQUIRE(q && n >= 0 && (n == 0 || d_ids), APPO_ERR_CONTRACT, "slotq_push: bad arguments");
  APPO_REQUIRE((uint32_t)n <= q->capacity, APPO_ERR_CONTRACT, "slotq_push: more ids than capacity");
  return slotq_push_launch(ctx, q, d_ids, 0, n, nullptr);
}

int appo_slotq_push_range(appo_ctx* ctx, appo_slotq* q, int32_t first_id, int n) {
  SQ_CTX_OR_RETURN(ctx);
  APPO_REQUIRE(q && n >= 0 && first_id >= 0, APPO_ERR_CONTRACT, "slotq_push_range: bad arguments");
  APPO_REQUIRE((uint32_t)n <= q->capacity, APPO_ERR_CONTRACT,
               "slotq_push_range: more ids than capacity");
  APPO_REQUIRE((int64_t)first_id + n <= q->n_slots, APPO_ERR_CONTRACT,
               "slotq_push_range: ids outside [0, n_slots)");
  return slotq_push_launch(ctx, q, nullptr, first_id, n, nullptr);
}

int appo_slotq_pop(appo_ctx* ctx, appo_slotq* q, int32_t* d_out, int n) {
  SQ_CTX_OR_RETURN(ctx);
  APPO_REQUIRE(q && d_out && n >= 1, APPO_ERR_CONTRACT, "slotq_pop: bad arguments");
  APPO_REQUIRE((uint32_t)n <= q->capacity, APPO_ERR_CONTRACT, "slotq_pop: more ids than capacity");
  // the ok word lives in the ctx's counter block (index 9 is reserved for it)
  return slotq_pop_launch(ctx, q, d_out, n, reinterpret_cast<int*>(ctx->d_counter + 9));
}

int appo_slotq_stats(appo_slotq* q, int64_t* pushed, int64_t* popped, int64_t* timeouts) {
  APPO_REQUIRE(q != nullptr, APPO_ERR_CONTRACT, "slotq_stats: null queue");
  unsigned long long c[4];
  APPO_CUDA_TRY(cudaSetDevice(q->device));
  APPO_CUDA_TRY(cudaMemcpy(c, q->ctr, sizeof(c), cudaMemcpyDeviceToHost));
  if (pushed) *pushed = (int64_t)c[0];
  if (popped) *popped = (int64_t)c[1];
  if (timeouts) *timeouts = (int64_t)c[2];
  return APPO_OK;
}

}  // extern "C"
