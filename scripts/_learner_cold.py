"""Learner step wall time with hot (same 64 slots every step) vs cold (a new set
of 64 slots every step, as the bench's minibatches) slot data."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
import paper_2006_11751_b200 as appo
desc = appo.ModelDesc.doom()
ctx = appo.Context(0, seed=1, model=desc)
n = 4096
store = appo.TrajectoryStore(desc, n)
smp = appo.Sampler(ctx, n, 256, seed=3)
for t in range(desc.T):
    smp.step(store, 0, t)
torch.cuda.synchronize()
ids = np.arange(n, dtype=np.int32).reshape(-1, 64)
for _ in range(3):
    ctx.learner_step(store.region, store.slot_bytes, ids[0])
for name, sel in (("hot", [0] * 32), ("cold", list(range(32))), ("hot", [0] * 32), ("cold", list(range(32, 64)))):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in sel:
        ctx.learner_submit(store.region, store.slot_bytes, ids[k])
    ctx.learner_collect()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / len(sel):.3f} ms per learner step")
