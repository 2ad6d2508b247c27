// Device-side slot queue (ready queue / free list) shared by the sampler and
// the learner step; see slotq.cu.
#pragma once
#include "appo_common.cuh"

struct appo_slotq {
  int device = 0;
  uint32_t capacity = 0;  // power of two
  int32_t n_slots = 0;    // ids must lie in [0, n_slots)
  int64_t timeout_ns = 0;
  int32_t* ids = nullptr;                // [capacity]
  unsigned long long* seq = nullptr;     // [capacity] per-entry sequence (Vyukov ring)
  unsigned long long* ctr = nullptr;     // [0] tail reservation, [1] head, [2] timeouts
};

namespace appo_b200 {
// enqueue n ids (d_ids, or first_id + i when d_ids is null) on c's stream;
// skipped entirely when d_ok != null and *d_ok == 0 (a rejected pop)
int slotq_push_launch(Ctx* c, appo_slotq* q, const int32_t* d_ids, int32_t first_id, int n,
                      const int* d_ok);
// dequeue n ids into d_out on c's stream, waiting on the device until n are
// published (bounded by q->timeout_ns); *d_ok = 1 on success, else 0, the
// queue untouched, d_out zero-filled and ctx flag kFlagQueue raised
int slotq_pop_launch(Ctx* c, appo_slotq* q, int32_t* d_out, int n, int* d_ok);
}  // namespace appo_b200
