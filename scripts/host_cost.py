"""Host-side enqueue cost of one learner step / one sampler step vs their GPU
time (is the step launch-bound?).  usage: python scripts/host_cost.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_11751_b200 as appo  # noqa: E402


def main():
    desc = appo.ModelDesc.doom()
    ctx = appo.Context(0, seed=1, model=desc)
    n = 16384
    store = appo.TrajectoryStore(desc, n)
    smp = appo.Sampler(ctx, n, 256, seed=3)
    for t in range(desc.T):
        smp.step(store, 0, t)
    ids = np.arange(64, dtype=np.int32)
    hp = appo.HParams.defaults()
    for _ in range(3):
        ctx.learner_step(store.region, store.slot_bytes, ids, hp)
    torch.cuda.synchronize()
    # block the stream so the host runs ahead, then time pure enqueue
    for what in ("learner", "sampler"):
        torch.cuda._sleep(400_000_000)  # ~0.2 s of GPU time ahead of the enqueues
        t0 = time.perf_counter()
        for k in range(6):  # fewer than the 8-deep pinned stats ring
            if what == "learner":
                ctx.learner_submit(store.region, store.slot_bytes, ids + 64 * (k % 4), hp)
            else:
                smp.step(store, 0, k % desc.T)
        t1 = time.perf_counter()
        if what == "learner":
            ctx.learner_collect()
        torch.cuda.synchronize()
        print(f"{what}: host enqueue {1e6 * (t1 - t0) / 6:.1f} us per step", flush=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    t0 = time.perf_counter()
    for k in range(50):
        ctx.learner_submit(store.region, store.slot_bytes, ids + 64 * (k % 4), hp)
    t1 = time.perf_counter()
    e1.record()
    ctx.learner_collect()
    torch.cuda.synchronize()
    print(f"learner x50 back-to-back: gpu {e0.elapsed_time(e1) / 50 * 1000:.1f} us/step, "
          f"host {1e6 * (t1 - t0) / 50:.1f} us/step", flush=True)


if __name__ == "__main__":
    main()
