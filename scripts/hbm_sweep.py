"""HBM sweep of the memory-bound kernels (V-trace / GAE at C1
256x32 up to 65,536x32, the fused PPO loss, Adam): per-launch duration from
the library's CUDA-event timing on the ctx stream (appo_ctx_set_timing), the
algorithmic bytes the launcher records, and GB/s against MEASURED_PEAKS.json.
Inputs rotate over enough buffer sets that every launch reads from HBM, not
from the 126 MB L2.  One JSON line per (kernel, size).

    python scripts/hbm_sweep.py            # event timing
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none python scripts/hbm_sweep.py --quick   # DRAM traffic
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2006_11751_b200 as appo  # noqa: E402

L2 = 126 << 20
RET = "returns32v_kernel<MODE>|returns32_kernel<MODE>"  # T = 32 paths (offpolicy.cu)
QUICK = "--quick" in sys.argv
REPS = 3 if QUICK else 20


def peak():
    try:
        with open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) as f:
            return json.load(f)["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


def n_sets(bytes_per_set):
    return max(2, int(np.ceil(3 * L2 / max(bytes_per_set, 1))))


def timed(ctx, name_filter, calls):
    """calls: list of thunks (one per launch, rotating buffer sets)."""
    for f in calls[:3]:
        f()
    ctx.sync()
    ctx.set_timing(True, name_filter)
    for i in range(REPS):
        calls[i % len(calls)]()
    ctx.sync()
    rep = ctx.timing_report()
    ctx.set_timing(False)
    return rep


def emit(kind, size, rep, hbm):
    for r in rep:
        avg_us = r["ms"] / r["launches"] * 1e3
        b = r["bytes"] / r["launches"]
        gbs = b / (avg_us * 1e-6) / 1e9
        print(json.dumps({"kernel": r["name"], "case": kind, "size": size, "launches": r["launches"],
                          "avg_us": round(avg_us, 2), "algorithmic_bytes": b,
                          "gbs": round(gbs, 1), "frac_hbm": round(gbs / hbm[0], 4),
                          "peak_source": hbm[1]}), flush=True)


def main():
    hbm = peak()
    ctx = appo.Context(0, seed=1, model=appo.ModelDesc.doom())
    rs = np.random.default_rng(0)
    dev = lambda x, dt=torch.float32: torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dt)
    T = 32
    sizes = [256, 4096, 65536] if not QUICK else [256, 65536]
    for n in sizes:
        per_set = n * T * (4 * 4 + 1 + 4 * 4) + n * 4
        sets = []
        for _ in range(n_sets(per_set)):
            sets.append(dict(r=dev(rs.uniform(-1, 1, (n, T))), v=dev(rs.uniform(-1, 1, (n, T))),
                             b=dev(rs.uniform(-1, 1, n)), tl=dev(rs.uniform(-2.5, -0.1, (n, T))),
                             bl=dev(rs.uniform(-2.5, -0.1, (n, T))),
                             d=dev(rs.uniform(size=(n, T)) < 0.15, torch.uint8)))
        vt = [lambda s=s: ctx.vtrace(s["r"], s["v"], s["b"], s["tl"], s["bl"], s["d"], sync=False)
              for s in sets]
        emit("vtrace", f"{n}x{T}", timed(ctx, RET, vt), hbm)
        gae = [lambda s=s: ctx.gae(s["r"], s["v"], s["b"], s["d"], 0.99, 0.95, sync=False)
               for s in sets]
        emit("gae", f"{n}x{T}", timed(ctx, RET, gae), hbm)
        del sets
        torch.cuda.empty_cache()
    # fused PPO loss (ratio, clipped surrogate, value, entropy, dlogits, dV)
    for B in ([2048, 65536] if not QUICK else [65536]):
        A = 6
        per_set = B * (A * 4 + 4 + 4 + 4 + 4 + 4 + (A + 1) * 4)
        sets = []
        for _ in range(n_sets(per_set)):
            lg = dev(rs.normal(size=(B, A)))
            sets.append(dict(lg=lg, v=dev(rs.normal(size=B)),
                             a=dev(rs.integers(0, A, B), torch.int32),
                             bl=dev(rs.uniform(-2.5, -0.5, B)), adv=dev(rs.normal(size=B)),
                             vt=dev(rs.normal(size=B))))
        calls = [lambda s=s: ctx.ppo_loss_injected(s["lg"], s["v"], s["a"], s["bl"], s["adv"],
                                                   s["vt"]) for s in sets]
        emit("ppo_loss", B, timed(ctx, "ppo_loss_kernel", calls), hbm)
        del sets
        torch.cuda.empty_cache()
    # Adam + global-norm clip at the model's size and at a large vector
    for n in ([2872551, 33554432] if not QUICK else [2872551]):
        sets = []
        for _ in range(n_sets(16 * n)):
            sets.append([dev(np.abs(rs.normal(size=n)) * 0.01) for _ in range(4)])
        calls = [lambda s=s: ctx.optimizer_step(s[0], s[1], s[2], s[3], 1) for s in sets]
        emit("adam", n, timed(ctx, "adam_kernel", calls), hbm)
        emit("adam-norm", n, timed(ctx, "sumsq_kernel", calls), hbm)
        del sets
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
