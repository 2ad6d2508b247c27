import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2006_11751_b200 as appo
desc = appo.ModelDesc.doom()
ctx = appo.Context(0, seed=1, model=desc)
store = appo.TrajectoryStore(desc, 64)
smp = appo.Sampler(ctx, 64, 256, seed=3)
for t in range(desc.T):
    smp.step(store, 0, t)
ids = np.arange(64, dtype=np.int32)
for _ in range(3):
    ctx.learner_step(store.region, store.slot_bytes, ids)
torch.cuda.synchronize()
os.environ["APPO_GRU_PROF"] = "1"
ctx.learner_step(store.region, store.slot_bytes, ids)
torch.cuda.synchronize()
