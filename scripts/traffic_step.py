"""One inference step (16384 envs) + 8 learner steps (2048 samples each) at the
bench shapes -- the bench's 32 : 256 launch mix -- inside a cudaProfilerStart/Stop
range, for `ncu --profile-from-start off` captures (DRAM traffic per kernel class
-> profiles/traffic.json via traffic_summary.py)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_11751_b200 as appo  # noqa: E402


def main():
    envs = int(os.environ.get("ENVS", "16384"))
    desc = appo.ModelDesc.doom()
    ctx = appo.Context(0, seed=1, model=desc)
    store = appo.TrajectoryStore(desc, max(envs, 64))
    smp = appo.Sampler(ctx, envs, 256, seed=3)
    for t in range(desc.T):
        smp.step(store, 0, t)
    ids = np.arange(64, dtype=np.int32)
    for _ in range(2):
        ctx.learner_step(store.region, store.slot_bytes, ids)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    smp.step(store, 0, 5)
    for _ in range(8):
        ctx.learner_step(store.region, store.slot_bytes, ids)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("traffic step done")


if __name__ == "__main__":
    main()
