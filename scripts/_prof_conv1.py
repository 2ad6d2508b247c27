"""One inference step at 16,384 envs with the conv1 per-tile timeline (APPO_C1_PROF=1)."""
import os, sys
import torch
sys.path.insert(0, os.getcwd())
import paper_2006_11751_b200 as appo
desc = appo.ModelDesc.doom()
ctx = appo.Context(0, seed=1, model=desc)
n = 16384
store = appo.TrajectoryStore(desc, n)
smp = appo.Sampler(ctx, n, 256, seed=3)
smp.step(store, 0, 0)
smp.step(store, 0, 1)
torch.cuda.synchronize()
smp.step(store, 0, 2)
torch.cuda.synchronize()
