"""One bench iteration's parts on one stream: 32 sampler steps (16,384 envs),
256 learner steps (2,048 samples), and both interleaved as in bench.py."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
import paper_2006_11751_b200 as appo
desc = appo.ModelDesc.doom()
ctx = appo.Context(0, seed=1, model=desc)
n = 16384
store = appo.TrajectoryStore(desc, 2 * n)
smp = appo.Sampler(ctx, n, 256, seed=3)
ids = np.arange(n, dtype=np.int32).reshape(-1, 64)
for t in range(desc.T):
    smp.step(store, n, t)
torch.cuda.synchronize()


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def sampler():
    for t in range(desc.T):
        smp.step(store, 0, t)


def learner():
    for mb in ids:
        ctx.learner_submit(store.region, store.slot_bytes, mb + n)
    ctx.learner_collect()


def both():
    for t in range(desc.T):
        smp.step(store, 0, t)
        for mb in ids[t * 8:(t + 1) * 8]:
            ctx.learner_submit(store.region, store.slot_bytes, mb + n)
    ctx.learner_collect()


for _ in range(2):
    print(f"sampler 32 steps {timed(sampler):.1f} ms | learner 256 steps {timed(learner):.1f} ms | "
          f"interleaved one stream {timed(both):.1f} ms")
