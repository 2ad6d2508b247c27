"""Debug: sampler inference + learner step at the bench layout (T=32), small env count."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_11751_b200 as appo

envs = int(os.environ.get("ENVS", "64"))
desc = appo.ModelDesc.doom()
ctx = appo.Context(0, seed=1, model=desc)
store = appo.TrajectoryStore(desc, max(envs, 64))
smp = appo.Sampler(ctx, envs, 256, seed=3)
for t in range(desc.T):
    smp.step(store, 0, t)
    torch.cuda.synchronize()
print("sampler ok", flush=True)
ids = np.arange(min(64, envs), dtype=np.int32)
out = ctx.learner_step(store.region, store.slot_bytes, ids)
torch.cuda.synchronize()
print("learner ok", out, flush=True)
