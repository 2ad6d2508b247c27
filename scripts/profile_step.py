"""Per-kernel (and per-GEMM-shape) CUDA-event timing of one inference step and
one learner step at the benchmark shapes.  usage: python scripts/profile_step.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_11751_b200 as appo  # noqa: E402


def show(title, rep):
    tot = sum(r["ms"] for r in rep)
    print(f"\n== {title}: {tot:.3f} ms over {sum(r['launches'] for r in rep)} launches")
    for r in sorted(rep, key=lambda r: -r["ms"])[:40]:
        extra = ""
        if r["flops"] > 0:
            extra = f" {r['flops'] / (r['ms'] * 1e-3) / 1e12:7.1f} TF/s"
        elif r["bytes"] > 0:
            extra = f" {r['bytes'] / (r['ms'] * 1e-3) / 1e9:7.1f} GB/s"
        print(f"{r['name'][:58]:58s} n={r['launches']:4d} ms={r['ms']:8.3f} "
              f"avg_us={1000 * r['ms'] / r['launches']:8.1f} share={r['ms'] / tot:.3f}{extra}")


def main():
    envs = int(os.environ.get("ENVS", "16384"))
    desc = appo.ModelDesc.doom()
    ctx = appo.Context(0, seed=1, model=desc)
    store = appo.TrajectoryStore(desc, max(envs, 64))
    smp = appo.Sampler(ctx, envs, 256, seed=3)
    for t in range(desc.T):
        smp.step(store, 0, t)
    ids = np.arange(64, dtype=np.int32)
    for _ in range(3):
        ctx.learner_step(store.region, store.slot_bytes, ids)
    torch.cuda.synchronize()
    for filt in (None, "gemm_shapes"):
        ctx.set_timing(True, filt)
        smp.step(store, 0, 5)
        show(f"inference step ({envs} envs) [{filt}]", ctx.timing_report())
        ctx.set_timing(True, filt)
        ctx.learner_step(store.region, store.slot_bytes, ids)
        show(f"learner step (2048 samples) [{filt}]", ctx.timing_report())
    ctx.set_timing(False)
    # wall-clock per learner step without timing
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ctx.learner_step(store.region, store.slot_bytes, ids)
    e1.record()
    torch.cuda.synchronize()
    print(f"\nlearner step wall (events): {e0.elapsed_time(e1) / 10:.3f} ms")
    e0.record()
    for t in range(desc.T):
        smp.step(store, 0, t)
    e1.record()
    torch.cuda.synchronize()
    print(f"inference step wall (events): {e0.elapsed_time(e1) / desc.T:.3f} ms ({envs} envs)")


if __name__ == "__main__":
    main()
