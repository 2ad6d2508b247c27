#!/usr/bin/env python
"""APPO hot-path benchmark (BASELINE.json metric: env frames/sec of policy
inference + V-trace/PPO learning per B200, and at 2/4/8 GPUs).

Workload (BASELINE.json configs[3], single GPU shard of it): 16,384 synthetic
envs per GPU with the on-GPU observation generator (u8 3x72x128, frameskip 4),
convnet_simple + GRU-512 + 6-way categorical head, T = 32.  One bench step =
one full APPO iteration: a T-step rollout of every env through batched policy
inference (obs written straight into HBM trajectory slots), then every sealed
trajectory trained once by the learner (V-trace + PPO clipped surrogate +
value + entropy loss, BPTT over the 32-step window, encoder backward,
global-norm clip + Adam) in minibatches of 2048 samples (64 trajectories).
frames per step = n_envs * T * frameskip.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Under torchrun (N > 1) every rank drives its own GPU; the learner is
data-parallel with an NCCL gradient all-reduce (appo_dp_init) unless --mode pbt
(independent policy per GPU, configs[4]).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "env frames/sec (inference + V-trace/PPO learn) per GPU and at 2/4/8 B200"


# prime: no aliasing with the 26-launch learner step / 9-launch sampler step
TIMING_STRIDE = int(os.environ.get("APPO_BENCH_TIMING_STRIDE", "13"))


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--envs", type=int, default=16384)
    p.add_argument("--T", type=int, default=32)
    p.add_argument("--traj-per-batch", type=int, default=64)
    p.add_argument("--frameskip", type=int, default=4)
    p.add_argument("--episode-len", type=int, default=256)
    p.add_argument("--mode", default="dp", choices=["dp", "pbt"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-overlap", action="store_true", help="sampler and learner on one stream")
    p.add_argument("--sampler-sms", type=int, default=64,
                   help="SM budget of the sampler context (persistent grids sized to it; 0 = all): "
                        "leaves SMs to the learner's kernels while both streams run")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-traj", type=int, default=0, help="trajectories per CPU-baseline sample")
    return p.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        self.f.seek(0)
        rows = [l.strip().split(",") for l in self.f.read().splitlines() if l.strip()]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for k, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(k)
            except Exception:
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# --------------------------------------------------------------------- CPU baseline
def host_cpu():
    """lscpu model name and the usable core count of this host."""
    model = None
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if line.startswith("Model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:  # noqa: BLE001
        pass
    return model, len(os.sched_getaffinity(0))


_NATIVE_ORACLE = {}


def native_oracle():
    """The oracle port compiled for THIS host (-O3 -march=native, SURVEY §8(d)
    CPU plan) into a temporary directory; the prebuilt portable -O3 build
    (oracle/liboracle.so) if the compiler is unavailable."""
    from oracle.oracle import Oracle
    if "o" not in _NATIVE_ORACLE:
        d = tempfile.mkdtemp(prefix="appo_oracle_")
        so = os.path.join(d, "liboracle_native.so")
        r = subprocess.run(["gcc", "-O3", "-march=native", "-std=c99", "-fPIC", "-shared", "-o", so,
                            os.path.join(ROOT, "oracle", "appo_oracle.c"), "-lm"],
                           capture_output=True)
        _NATIVE_ORACLE["o"] = (Oracle(so), "gcc -O3 -march=native") if r.returncode == 0 else \
            (Oracle(), "prebuilt -O3 (native build failed)")
    return _NATIVE_ORACLE["o"]


def reference_mlp_timing():
    """The reference's own learner math (its MLP stand-in 27,648 -> 512 -> 512
    -> 6 at the Doom input, oracle/_ref) on one thread: the CPU cost the
    reference would pay per sample with its own model."""
    try:
        from oracle.oracle import Reference
        if not Reference.available():
            return None
        st, r = Reference().mlp_stand_in_time(B=8, reps=2)
        if st != 0:
            return {"error": f"status {st}"}
        per = r["forward_s_per_sample"] + r["gradient_s_per_sample"]
        return dict(r, threads=1, frames_per_s_per_thread=4.0 / per,
                    note="forward_batch (inference) + compute_gradients (learner) per sample, "
                         "optimizer_step per call excluded; fp64, 1 thread, best of 2, B=8")
    except Exception as ex:  # noqa: BLE001
        return {"error": repr(ex)}


def cpu_baseline_sample(args, n_traj=None, seed=0):
    """Oracle port (oracle/appo_oracle.c, fp64) on the host cores: every thread
    runs one trajectory through T+1 inference steps and one learner step over
    it -- the same per-sample work as the GPU step (the learner's cost is
    linear in the trajectories of a minibatch), bounded in size."""
    orc, build = native_oracle()
    model, cores = host_cpu()
    n = n_traj or 8 * cores  # ~8-10 s of CPU work on the GPU box's host
    shape = (3, 72, 128, 6)
    T = args.T
    theta = orc.init_params(*shape, 1)
    rs = np.random.default_rng(seed)
    obs_all = rs.integers(0, 256, (n, T + 1, 3 * 72 * 128), dtype=np.uint8)

    def work(i):
        h = np.zeros((1, 512))
        acts, lps = [], []
        for t in range(T + 1):
            u = np.array([orc.L.orc_uniform(i, t)])
            out = orc.policy_forward(shape, theta, obs_all[i, t][None], h, u=u)
            h = out["h_out"]
            acts.append(out["actions"][0]); lps.append(out["logp"][0])
        th = theta.copy()
        m = np.zeros_like(th); v = np.zeros_like(th)
        rew = rs.uniform(-0.5, 0.5, T)
        dn = np.zeros(T, np.uint8)
        orc.learner_step(shape, th, m, v, 0, obs_all[i][None], np.zeros((1, 512)),
                         np.array(acts[:T], np.int32), np.array(lps[:T]), rew, dn)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(n)]
    t0 = time.perf_counter()
    for th_ in threads:
        th_.start()
    for th_ in threads:
        th_.join()
    dt = time.perf_counter() - t0
    frames = n * T * args.frameskip
    return {"value": frames / dt, "unit": "frames/s", "cores": min(cores, n), "kind": "port",
            "cpu_model": model, "nproc": cores, "build": build,
            "sample": f"{n} trajectories x T={T} (inference of T+1 steps + one learner step each), "
                      f"fp64 C oracle, {min(cores, n)} threads, {dt:.1f} s"}


def run_reference(args, ws, rank):
    if rank != 0:
        return
    K, W = args.steps, args.warmup
    for _ in range(min(W, 1)):
        cpu_baseline_sample(args, n_traj=max(1, host_cpu()[1] // 4))
    vals = []
    t0 = time.perf_counter()
    res = None
    for k in range(K):
        res = cpu_baseline_sample(args, n_traj=args.cpu_traj or None, seed=k)
        vals.append(res["value"])
    wall = time.perf_counter() - t0
    v = float(np.mean(vals))
    line = {"metric": METRIC, "value": v, "unit": "frames/s", "n_gpus": args.gpus, "steps": K,
            "warmup": W, "ms_per_step": 1000.0 * wall / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "C4 per-sample work (inference + learner), Doom shape",
                       "obs": "u8 3x72x128", "T": args.T, "frameskip": args.frameskip},
            "cpu_baseline": dict(res, value=v, reference_mlp_stand_in=reference_mlp_timing()),
            "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- GPU arm
def merge_reports(*reps):
    out = {}
    for rep in reps:
        for r in rep:
            a = out.setdefault(r["name"], dict(name=r["name"], launches=0, ms=0.0, flops=0.0,
                                               bytes=0.0))
            for k in ("launches", "ms", "flops", "bytes"):
                a[k] += r[k]
    return list(out.values())


def run_ours(args, ws, rank, local):
    import torch
    import paper_2006_11751_b200 as appo

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    desc = appo.ModelDesc.doom(T=args.T)
    seed = 1 if args.mode == "dp" else 1 + rank
    # learner on a high-priority stream (its GRU phases are latency-bound and
    # use few SMs); the sampler fills the rest of the GPU at low priority
    hi = torch.cuda.Stream(local, priority=int(os.environ.get("APPO_BENCH_LEARNER_PRIO", "-1")))
    torch.cuda.set_stream(hi)
    lctx = appo.Context(local, seed=seed, model=desc, stream=hi)    # learner
    if args.no_overlap:
        sctx = lctx
    else:
        sctx = lctx.shared(torch.cuda.Stream(local, priority=0))    # sampler / policy worker
        if args.sampler_sms:
            sctx.set_sm_budget(args.sampler_sms)
    if ws > 1 and args.mode == "dp":
        appo.dp_init(lctx, dist, rank, ws)
    n = args.envs
    tpb = args.traj_per_batch
    assert n % tpb == 0
    # two rollout sets: the sampler fills set k%2 while the learner trains on
    # set (k-1)%2 (APPO's sampler/learner decoupling, §3)
    store = appo.TrajectoryStore(desc, 2 * n, device=local)
    sampler = appo.Sampler(sctx, n, args.episode_len, seed=1000 + rank)
    hp = appo.HParams.defaults()
    ids = np.arange(n, dtype=np.int32).reshape(-1, tpb)
    lstream, sstream = lctx.stream, sctx.stream
    state = {"k": 0}

    def host_step(h, base, t):
        """CPU actors (appo_rollout_act / _feedback, orchestrator.hpp:435-552):
        every env step's observations, rewards and dones -- and at T-1 the
        bootstrap observations -- come from pinned host memory, and the actions
        reach the host before the step's feedback (an actor needs them to step
        its envs).  Two env groups, as the reference's double-buffered rollout
        workers (orchestrator.hpp:434, exchange slot id*2+g): a group's next
        act is issued right after its feedback, so its observation transfer
        overlaps the other group's wait and inference."""
        T = args.T
        for g, smp in enumerate(h["samplers"]):
            if t == 0:
                smp.act(store, base + g * h["gn"], 0, h["obs"][g][0], h["act"][g])
        for g, smp in enumerate(h["samplers"]):
            smp.wait()
            smp.feedback(store, base + g * h["gn"], t, h["rew"][g][t], h["dn"][g][t],
                         h["obs"][g][(t + 1) % 2] if t == T - 1 else None)
            if t + 1 < T:
                smp.act(store, base + g * h["gn"], t + 1, h["obs"][g][(t + 1) % 2], h["act"][g])

    def iteration(h=None):
        k = state["k"]
        base = (k % 2) * n
        # interleave submission (one sampler step per len(ids)/T learner steps)
        # so each inference picks up the newest completed parameters
        per = (len(ids) + args.T - 1) // args.T
        prev = ((k - 1) % 2) * n
        for t in range(args.T):
            if h is None:
                sampler.step(store, base, t)
            else:
                host_step(h, base, t)
            if k > 0:
                for mb in ids[t * per:(t + 1) * per]:  # asynchronous learner steps
                    lctx.learner_submit(store.region, store.slot_bytes, mb + prev, hp)
        last = lctx.learner_collect() if k > 0 else None
        done = torch.cuda.Event()
        done.record(sstream)
        lstream.wait_event(done)  # iteration boundary: both streams joined on the learner stream
        state["k"] = k + 1
        return last

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def timing(on, filt=None):
        lctx.set_timing(on, filt)
        if sctx is not lctx:
            sctx.set_timing(on, filt)

    def report():
        r = lctx.timing_report()
        return merge_reports(r, sctx.timing_report()) if sctx is not lctx else r

    def launches():
        return lctx.launches + (sctx.launches if sctx is not lctx else 0)

    # warm-up (the first iteration only samples); the last warm-up iteration
    # also finds the dominant kernel family
    for w in range(max(args.warmup, 2)):
        if w == max(args.warmup, 2) - 1:
            timing(True)
        iteration()
    barrier()
    rep = report()
    timing(False)
    total_ms = sum(r["ms"] for r in rep)
    # the top kernel classes of the warm-up are timed live (the dominant one is
    # `roofline`, the others `roofline_kernels`); conv1 forward is always among them
    top = sorted(rep, key=lambda r: -r["ms"])[:4]
    if not any(r["name"].startswith("conv1_s2d") for r in top):
        top += [r for r in rep if r["name"].startswith("conv1_s2d")][:1]
    live_names = "|".join(r["name"] for r in top)

    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    l0 = launches()
    # per-kernel events on a sample of the launches only (every TIMING_STRIDE-th
    # launch of the timed classes): an event between two kernels ends their
    # programmatic-dependent-launch overlap, and timing every launch of these
    # classes measured 10 % off the step rate
    timing(True, f"@{TIMING_STRIDE}:" + live_names)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(lstream)
    last = None
    for k in range(args.steps):
        last = iteration()
    e1.record(lstream)
    barrier()
    ms = e0.elapsed_time(e1)
    n_launch = launches() - l0
    live = report()
    timing(False)
    clk = clocks.stop()
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    frames_step = n * args.T * args.frameskip
    value = frames_step * args.steps * ws / (ms / 1000.0)

    # e2e: every env step's observations, rewards and dones (and the bootstrap
    # observations) from pinned host memory (CPU actors), actions back to the
    # host each step, learner stats back to the host
    e2e = None
    if not args.no_e2e:
        gn = n // 2
        rs = np.random.default_rng(rank)
        T = args.T
        h = {"gn": gn, "samplers": [appo.Sampler(sctx, gn, args.episode_len, seed=2000 + rank + g)
                                    for g in range(2)],
             "obs": [[torch.from_numpy(rs.integers(0, 256, (gn, desc.obs_dim), dtype=np.uint8))
                      .pin_memory() for _ in range(2)] for _ in range(2)],
             "act": [torch.empty(gn, dtype=torch.int32).pin_memory() for _ in range(2)],
             # SyntheticLatencyEnv's reward schedule / episode ends (envs.hpp:127-128)
             "rew": [[torch.from_numpy((0.1 * ((np.arange(gn) + t + 1 + g) % 11) - 0.5)
                                       .astype(np.float32)).pin_memory() for t in range(T)]
                     for g in range(2)],
             "dn": [[torch.from_numpy(((np.arange(gn) * 7 + t + g) % args.episode_len == 0)
                                      .astype(np.uint8)).pin_memory() for t in range(T)]
                    for g in range(2)]}
        iteration(h)
        barrier()
        e0.record(lstream)
        for k in range(args.steps):
            iteration(h)
        e1.record(lstream)
        barrier()
        ems = e0.elapsed_time(e1)
        if dist is not None:
            t_ = torch.tensor([ems], device="cuda")
            dist.all_reduce(t_, op=dist.ReduceOp.MAX)
            ems = t_.item()
        n_mb = ids.shape[0]
        e2e = {"value": frames_step * args.steps * ws / (ems / 1000.0), "unit": "frames/s",
               "h2d_bytes_per_step": n * desc.obs_dim * (T + 1) + n * 5 * T + n_mb * tpb * 4,
               "d2h_bytes_per_step": n * 4 * T + n_mb * (8 * 10 + 16),
               "path": "appo_rollout_act(h_obs) + wait + appo_rollout_feedback(h_rewards, "
                       "h_dones, h_next_obs at T-1), 2 env groups; appo_learner_submit/collect"}
        # the host link is the e2e bound: H2D rate achieved over the timed region
        e2e["h2d_gbps"] = e2e["h2d_bytes_per_step"] * args.steps / (ems / 1000.0) / 1e9
        for smp in h["samplers"]:
            smp.close()

    peaks, peak_src = load_peaks()
    ridge = peaks["bf16_tflops_sustained"] * 1e12 / (peaks["hbm_gbs"] * 1e9)

    def roofline(d):
        avg_ms = d["ms"] / d["launches"]
        # bound by arithmetic intensity against the machine balance (measured
        # peaks): FLOP-heavy kernels against the tensor peak, the rest against HBM
        intensity = d["flops"] / d["bytes"] if d["bytes"] > 0 else float("inf")
        if d["flops"] > 0 and intensity >= ridge:
            achieved = d["flops"] / d["launches"] / (avg_ms * 1e-3) / 1e12
            peak = peaks["bf16_tflops_sustained"]
            r = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                 "frac": achieved / peak}
        else:
            achieved = d["bytes"] / d["launches"] / (avg_ms * 1e-3) / 1e9
            peak = peaks["hbm_gbs"]
            r = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                 "frac": achieved / peak}
        r.update({"kernel": d["name"], "launches": d["launches"], "avg_us": avg_ms * 1e3,
                  "algorithmic_bytes_per_launch": d["bytes"] / d["launches"],
                  "algorithmic_flops_per_launch": d["flops"] / d["launches"],
                  "intensity_flop_per_byte": intensity, "ridge_flop_per_byte": ridge,
                  "share_of_step": d["ms"] * TIMING_STRIDE / ms, "peak_source": peak_src,
                  "timing_sample": f"CUDA events around every {TIMING_STRIDE}th launch of the "
                                   "timed classes during the timed region",
                  "traffic": load_traffic(d["name"])})
        return r

    roof = None
    others = []
    if live:
        live_sorted = sorted(live, key=lambda r: -r["ms"])
        roof = roofline(live_sorted[0])
        roof["note"] = ("sampler and learner overlap on two streams; shares are per-stream "
                        "busy time over the wall step")
        roof["kernel_shares_warmup"] = {r["name"]: round(r["ms"] / total_ms, 4) for r in
                                        sorted(rep, key=lambda r: -r["ms"])[:8]}
        others = [roofline(d) for d in live_sorted[1:]]

    if rank != 0:
        return
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_sample(args, n_traj=args.cpu_traj or None)
            cpu["reference_mlp_stand_in"] = reference_mlp_timing()
        except Exception as ex:  # noqa: BLE001
            cpu = {"error": repr(ex)}
    line = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (on-GPU SyntheticLatencyEnv hash generator), random-init weights",
            "config": {"workload": "C4: sampler+learner loop, convnet_simple+GRU-512, Doom shape",
                       "envs_per_gpu": n, "T": args.T, "batch": tpb * args.T,
                       "frameskip": args.frameskip, "obs": "u8 3x72x128",
                       "parallelism": (f"dp{ws}" if args.mode == "dp" else f"pbt{ws}"),
                       "learner_steps_per_step": int(ids.shape[0]),
                       "overlap": ("sampler stream || learner stream, sampler grids on "
                                   f"{args.sampler_sms or 'all'} SMs") if sctx is not lctx else "off",
                       "l2": "inputs larger than L2 (2 x 16 GB slot sets, 453 MB obs per env step)"},
            "samples_per_s": value / args.frameskip,
            "gpu_launches": n_launch,
            "roofline": roof,
            "roofline_kernels": others,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk,
            "last_step": last}
    print(json.dumps(line), flush=True)


def load_traffic(name):
    """DRAM bytes per launch of kernel class `name` from the committed ncu capture
    (profiles/traffic.json, scripts/traffic_summary.py); None if absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)["traffic_bytes_per_launch"].get(name.split("@")[0])
    except Exception:
        return None


def main():
    args = parse()
    ws, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
