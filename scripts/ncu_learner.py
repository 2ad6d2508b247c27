"""One learner step (2,048 samples, Doom shape) inside cudaProfilerStart/Stop,
after warm-up steps, for `ncu --profile-from-start off` captures of every
learner kernel (scripts/gpu_ncu_learner.sh)."""
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
for k in range(4):
    ctx.learner_step(store.region, store.slot_bytes, ids[k])
torch.cuda.synchronize()
torch.cuda.profiler.start()
ctx.learner_step(store.region, store.slot_bytes, ids[5])
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
