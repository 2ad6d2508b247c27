"""Parity at the shapes the bench runs (BASELINE.json configs[1..3]).

* learner: 64 trajectories x T=32 (config 3, B = 2048), plus 17 and 33
  trajectories so every cell slot of the persistent GRU kernels (forward: 4
  cells per thread, slots c >= 1 start at 17 trajectories; BPTT: 2 cells per
  thread, c = 1 starts at 33) is executed under test.  The oracle runs one
  trajectory per call in a thread pool: with advantage normalisation off the
  batch loss is the mean of the per-trajectory losses (policy.hpp:318 1/B), so
  the full-batch gradient is the mean of the per-trajectory gradients.
* inference: appo_policy_forward at 4,096 (config 2) and 16,384 envs (config 4)
  and the sampler's slot-strided path at 16,384 envs, 128 random rows each
  against the oracle.
* the loss kernels at the north_star's 1e-5: ppo_loss_kernel with injected
  logits / values against the reference's own compute_gradients
  (tests/golden/ppo_grad.npz), and the learner's production loss block
  (traj_loss_kernel) on injected core rows against the oracle's V-trace / GAE
  and the compiled reference's compute_gradients.

Tolerances (bf16 operands, fp32 accumulate): as
tests/test_model_gpu.py.  Observed errors are appended to $APPO_PARITY_LOG
(JSON lines) when set, so DESIGN.md can quote them.
"""
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from conftest import golden
from test_model_gpu import GNORM_TOL, GRAD_TOL, H_TOL, LOGPI_TOL, LOSS_ATOL, LOSS_RTOL

pytestmark = pytest.mark.gpu

import paper_2006_11751_b200 as appo  # noqa: E402

SHAPE = (3, 72, 128, 6)


def log_softmax(x):
    x = x - x.max(-1, keepdims=True)
    return x - np.log(np.exp(x).sum(-1, keepdims=True))


def record(name, **kw):
    path = os.environ.get("APPO_PARITY_LOG")
    kw = {k: (float(v) if isinstance(v, (np.floating, float)) else v) for k, v in kw.items()}
    print(name, kw)
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(dict(test=name, **kw)) + "\n")


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def block_offsets(n_actions=6, F=2304):
    sizes = [("c1w", 32 * 3 * 64), ("c1b", 32), ("c2w", 64 * 512), ("c2b", 64),
             ("c3w", 128 * 576), ("c3b", 128), ("fcw", 512 * F), ("fcb", 512),
             ("wih", 1536 * 512), ("whh", 1536 * 512), ("bih", 1536), ("bhh", 1536),
             ("wpi", n_actions * 512), ("bpi", n_actions), ("wv", 512), ("bv", 1)]
    out, o = {}, 0
    for k, n in sizes:
        out[k] = (o, o + n)
        o += n
    return out


def oracle_learner_mean(oracle, th, d, hp, workers=None):
    """Per-trajectory oracle learner steps in threads (ctypes drops the GIL);
    returns (mean gradient, mean stats[0..4])."""
    n = d["obs"].shape[0]

    def one(i):
        r = oracle.learner_step(SHAPE, th, np.zeros(th.size), np.zeros(th.size), 0,
                                d["obs"][i:i + 1], d["h0"][i:i + 1].astype(np.float64),
                                d["actions"][i], d["blogp"][i].astype(np.float64),
                                d["rewards"][i].astype(np.float64), d["dones"][i], hp=hp,
                                do_adam=False)
        assert r["status"] == 0
        return r["grad"], r["stats"][:5]

    workers = workers or max(1, min(n, os.cpu_count() or 1))
    g = np.zeros(th.size)
    st = np.zeros(5)
    with ThreadPoolExecutor(workers) as ex:
        for gi, si in ex.map(one, range(n)):
            g += gi
            st += si
    return g / n, st / n


def fill(store, n_traj, rs):
    T = store.T
    d = dict(obs=[], h0=[], actions=[], blogp=[], rewards=[], dones=[])
    for i in range(n_traj):
        obs = rs.integers(0, 256, (T + 1, store.obs_dim), dtype=np.uint8)
        h0 = rs.normal(scale=0.3, size=512).astype(np.float32)
        act = rs.integers(0, 6, T).astype(np.int32)
        blogp = rs.uniform(-2.2, -1.5, T).astype(np.float32)
        rew = rs.uniform(-1, 1, T).astype(np.float32)
        dn = (rs.uniform(size=T) < 0.1).astype(np.uint8)
        store.write_slot(i, obs[:T], h0, act, rew, blogp, dn, boot_obs=obs[T])
        for k, v in zip(d, (obs, h0, act, blogp, rew, dn)):
            d[k].append(v)
    return {k: np.stack(v) for k, v in d.items()}


# 65 trajectories exceed the persistent GRU kernels (<= 64): the per-step
# GEMM + cell fallback path
@pytest.mark.parametrize("n_traj,adv_source", [(64, 0), (33, 2), (17, 1), (65, 0)])
def test_learner_production_shape_matches_oracle(oracle, n_traj, adv_source):
    desc = appo.ModelDesc.doom(T=32)
    ctx = appo.Context(0, seed=40 + n_traj, model=desc)
    store = appo.TrajectoryStore(desc, n_traj + 3)
    rs = np.random.default_rng(n_traj)
    d = fill(store, n_traj, rs)
    # FIFO order is a permutation of the slots (slot-id indirection at full size)
    order = rs.permutation(n_traj)
    sel = {k: v[order] for k, v in d.items()}
    th0, _ = ctx.get_params()
    hp = appo.HParams.defaults(adv_source=adv_source, normalize_adv=0, gamma=0.99,
                               gae_lambda=0.95)
    out = ctx.learner_step(store.region, store.slot_bytes, order.tolist(), hp)
    g = ctx.grad().astype(np.float64)
    gr, st = oracle_learner_mean(oracle, th0.astype(np.float64), sel,
                                 dict(adv_source=adv_source, normalize=0, gamma=0.99,
                                      gae_lambda=0.95))
    errs = {}
    for name, got, exp in (("policy", out["policy_loss"], st[0]),
                           ("value", out["value_loss"], st[1]),
                           ("entropy", out["entropy"], st[2]),
                           ("total", out["total_loss"], st[3]),
                           ("ratio", out["mean_ratio"], st[4])):
        errs["loss_" + name] = abs(got - exp) / max(abs(exp), 1e-4)
        assert abs(got - exp) <= LOSS_RTOL * abs(exp) + LOSS_ATOL, (name, got, exp)
    gn = np.linalg.norm(gr)
    errs["grad_norm"] = abs(out["grad_norm"] - gn) / gn
    assert errs["grad_norm"] <= GNORM_TOL
    for name, (a, b) in block_offsets().items():
        e = rel_l2(g[a:b], gr[a:b])
        errs["grad_" + name] = e
        assert e <= GRAD_TOL, (name, e)
    record(f"learner_{n_traj}x32_adv{adv_source}", **errs)


@pytest.mark.parametrize("B", [4096, 16384])
def test_policy_forward_production_batch(oracle, B):
    ctx = appo.Context(0, seed=9, model=appo.ModelDesc.doom(T=32))
    rs = np.random.default_rng(B)
    obs = torch.randint(0, 256, (B, 27648), dtype=torch.uint8, device="cuda")
    h = torch.from_numpy(rs.normal(scale=0.5, size=(B, 512)).astype(np.float32)).cuda()
    out = ctx.policy_forward(obs, h, rng_counter0=7, want_logits=True)
    torch.cuda.synchronize()
    rows = np.sort(rs.choice(B, 128, replace=False))
    rows[0], rows[-1] = 0, B - 1  # first and last M tile
    th, _ = ctx.get_params()
    ref = oracle.policy_forward(SHAPE, th.astype(np.float64), obs[rows].cpu().numpy(),
                                h[rows].cpu().numpy().astype(np.float64))
    lg = out["logits"][rows].cpu().numpy().astype(np.float64)
    e_lp = np.abs(log_softmax(lg) - log_softmax(ref["logits"])).max()
    vals = out["values"][rows].cpu().numpy()
    e_v = np.abs(vals - ref["values"]).max()
    e_h = np.abs(out["h_out"][rows].cpu().numpy() - ref["h_out"]).max()
    record(f"policy_forward_B{B}", max_dlogpi=e_lp, max_dvalue=e_v, max_dh=e_h)
    assert e_lp <= LOGPI_TOL
    assert np.all(np.abs(vals - ref["values"]) <= 2e-4 + 2e-3 * np.abs(ref["values"]))
    assert e_h <= H_TOL
    key = oracle.L.orc_derive_seed(9, 0x9900)
    acts = out["actions"][rows].cpu().numpy()
    n_cmp = 0
    for i, b in enumerate(rows):
        u = oracle.L.orc_uniform(key, 7 + int(b))
        p = np.exp(log_softmax(ref["logits"][i]))
        if np.min(np.abs(np.cumsum(p) - u)) < 1e-3:
            continue
        a, _ = oracle.sample(lg[i], u)
        assert acts[i] == a
        n_cmp += 1
    assert n_cmp >= 100


def test_policy_forward_batch_invariance_all_rows():
    # rows are independent: every row of a 300-batch equals the same rows run
    # in other batch positions (split 300 = 128 + 172 across M tiles)
    ctx = appo.Context(0, seed=5, model=appo.ModelDesc.doom(T=32))
    rs = np.random.default_rng(1)
    obs = torch.from_numpy(rs.integers(0, 256, (300, 27648), dtype=np.uint8)).cuda()
    h = torch.from_numpy(rs.normal(size=(300, 512)).astype(np.float32)).cuda()
    a = ctx.policy_forward(obs, h, want_logits=True)
    b1 = ctx.policy_forward(obs[:128].contiguous(), h[:128].contiguous(), want_logits=True)
    b2 = ctx.policy_forward(obs[128:].contiguous(), h[128:].contiguous(), rng_counter0=128,
                            want_logits=True)
    torch.cuda.synchronize()
    for k in ("logits", "values", "h_out", "actions", "logp"):
        assert torch.equal(a[k], torch.cat([b1[k], b2[k]])), k


def test_sampler_production_envs_match_oracle(oracle):
    # config 4's sampler path: 16,384 envs, obs read from the slots (stride =
    # slot size); the stored behaviour logp / action / next hidden of 128 random
    # envs equal the oracle's inference on the stored obs + input hidden
    desc = appo.ModelDesc.doom(T=32)
    ctx = appo.Context(0, seed=17, model=desc)
    n = 16384
    store = appo.TrajectoryStore(desc, n)
    smp = appo.Sampler(ctx, n, episode_len=1000, seed=5)
    for t in range(2):
        smp.step(store, 0, t)
    torch.cuda.synchronize()
    rs = np.random.default_rng(3)
    envs = np.sort(rs.choice(n, 128, replace=False))
    envs[-1] = n - 1
    th, _ = ctx.get_params()
    t = 1
    obs = np.stack([store.obs(e)[t].cpu().numpy() for e in envs])
    hin = np.stack([store.hidden(e)[t].cpu().numpy() for e in envs]).astype(np.float64)
    assert np.any(hin != 0)  # the t=1 input hidden is the t=0 output
    ref = oracle.policy_forward(SHAPE, th.astype(np.float64), obs, hin)
    key = oracle.L.orc_derive_seed(17, 0x9900)
    lps = np.array([store.logp(e)[t].item() for e in envs])
    acts = np.array([store.actions(e)[t].item() for e in envs])
    ref_lp = log_softmax(ref["logits"])
    e_lp = np.abs(lps - ref_lp[np.arange(128), acts]).max()
    record("sampler_16384", max_dlogp_stored=e_lp)
    assert e_lp <= LOGPI_TOL
    n_cmp = 0
    for i, e in enumerate(envs):
        u = oracle.L.orc_uniform(key, n * t + int(e))  # counter = steps_done * n_envs + env
        p = np.exp(ref_lp[i])
        if np.min(np.abs(np.cumsum(p) - u)) < 1e-3:
            continue
        a, _ = oracle.sample(ref["logits"][i], u)
        assert acts[i] == a, (e, acts[i], a)
        n_cmp += 1
    assert n_cmp >= 100


def test_ppo_loss_kernel_matches_reference_compute_gradients():
    # north_star: losses within 1e-5 (fp32 vs the reference's fp64); the fused
    # kernel's dlogits / dV against compute_gradients with injected inputs
    g = golden("ppo_grad")
    ctx = appo.Context(0, seed=1)
    dev = "cuda"
    f = lambda k, dt=torch.float32: torch.from_numpy(np.ascontiguousarray(g[k])).to(dev, dt)
    dlog, stats = ctx.ppo_loss_injected(f("logits"), f("values"), f("actions", torch.int32),
                                        f("blogp"), f("adv"), f("vt"))
    dlog = dlog.cpu().numpy().astype(np.float64)
    A = g["logits"].shape[1]
    tol = lambda ref: 1e-5 * np.maximum(np.abs(ref), 1.0)
    e_dl = np.abs(dlog[:, :A] - g["dlogits"])
    e_dv = np.abs(dlog[:, A] - g["dv"])
    # per-sample gradients are O(1/B) (O(e^20/B) past the log-ratio clamp):
    # relative to each row's largest entry
    row = np.abs(g["dlogits"]).max(1, keepdims=True)
    rel_dl = (e_dl / row).max()
    rel_dv = (e_dv / np.maximum(np.abs(g["dv"]), 1e-30)).max()
    record("ppo_loss_injected", max_rel_dlogits=rel_dl, max_rel_dv=rel_dv,
           max_rel_loss=(np.abs(stats[:4] - g["loss"]) / np.maximum(np.abs(g["loss"]), 1)).max(),
           ratio_err=abs(stats[4] - float(g["mean_ratio"])))
    assert rel_dl <= 1e-5 and rel_dv <= 1e-5
    assert np.all(np.abs(stats[:4] - g["loss"]) <= tol(g["loss"])), (stats[:4], g["loss"])
    assert abs(stats[4] - float(g["mean_ratio"])) <= 1e-5 * max(1.0, float(g["mean_ratio"]))


@pytest.mark.parametrize("adv_source", [0, 2])
def test_traj_loss_kernel_matches_reference(oracle, reference, adv_source):
    """The learner's production loss block (traj_loss_kernel: heads, target logp,
    V-trace / GAE, loss gradient, heads backward in one CTA per trajectory) on
    injected core rows at the bench shape (64 x 32, 6 actions).  The heads are
    checked against an fp64 product of the same fp32 inputs; everything after
    them against the reference chain run in fp64 on the kernel's own logits /
    values -- the oracle's V-trace / GAE and the reference's compute_gradients
    (ref_ppo_grads_injected) -- at the north_star's 1e-5."""
    rs = np.random.default_rng(41 + adv_source)
    n, T, A, H = 64, 32, 6, 512
    B = n * T
    f32 = np.float32
    core = rs.normal(scale=0.5, size=(B + n, H)).astype(f32)
    wpi = rs.normal(scale=0.05, size=(A, H)).astype(f32)
    bpi = rs.normal(scale=0.1, size=A).astype(f32)
    wv = rs.normal(scale=0.05, size=H).astype(f32)
    bv = np.array([0.1], f32)
    act = rs.integers(0, A, B).astype(np.int32)
    rew = rs.uniform(-1, 1, B).astype(f32)
    blogp = rs.uniform(-2.5, -0.5, B).astype(f32)
    done = (rs.uniform(size=B) < 0.1).astype(np.uint8)
    dev = lambda x, dt=torch.float32: torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dt)
    ctx = appo.Context(0, seed=1)
    out = ctx.traj_loss_injected(T, dev(core), dev(wpi), dev(bpi), dev(wv), dev(bv),
                                 dev(act, torch.int32), dev(rew), dev(blogp),
                                 dev(done, torch.uint8), gamma=0.99, adv_source=adv_source,
                                 gae_lambda=0.95)
    g = {k: (v.cpu().numpy().astype(np.float64) if isinstance(v, torch.Tensor) else v)
         for k, v in out.items()}
    c64 = core.astype(np.float64)
    # heads: fp32 dot products of 512 terms vs fp64
    lg_ref = c64 @ wpi.T.astype(np.float64) + bpi
    v_ref = c64 @ wv.astype(np.float64) + float(bv[0])
    e_lg = np.abs(g["logits"] - lg_ref).max() / np.abs(lg_ref).max()
    e_v = np.abs(g["values"] - v_ref).max() / np.abs(v_ref).max()
    assert e_lg <= 1e-5 and e_v <= 1e-5, (e_lg, e_v)
    # the reference chain on the kernel's own logits / values
    lg, val = g["logits"], g["values"]
    lsm = lg - lg.max(1, keepdims=True)
    lsm = lsm - np.log(np.exp(lsm).sum(1, keepdims=True))
    tlogp = lsm[np.arange(B), act]
    st, (vs, pg, _, _) = oracle.vtrace_batch(rew.reshape(n, T), val[:B].reshape(n, T), val[B:],
                                             tlogp.reshape(n, T), blogp.reshape(n, T),
                                             done.reshape(n, T), 1.0, 1.0, 0.99)
    assert st == 0
    tol = lambda ref: 1e-5 * np.maximum(np.abs(ref), 1.0)
    assert np.all(np.abs(g["vt"] - vs.reshape(-1)) <= tol(vs.reshape(-1)))
    assert np.all(np.abs(g["pg"] - pg.reshape(-1)) <= tol(pg.reshape(-1)))
    if adv_source == 0:
        adv = pg.reshape(-1)
    else:
        adv = np.concatenate([oracle.gae(rew[i * T:(i + 1) * T], val[i * T:(i + 1) * T],
                                         val[B + i], done[i * T:(i + 1) * T], 0.99, 0.95)[0]
                              for i in range(n)])
        assert np.all(np.abs(g["adv"] - adv) <= tol(adv))
    st, ref = reference.ppo_grads_injected(lg[:B], val[:B], act, blogp, adv, vs.reshape(-1))
    assert st == 0
    # samples whose ratio sits within 1e-4 of a clip bound may take the other
    # branch in fp32: left out of the per-sample comparison (none expected)
    ratio = np.exp(np.clip(tlogp - blogp, -20, 20))
    keep = (np.abs(ratio - 1.1) > 1e-4) & (np.abs(ratio - 1 / 1.1) > 1e-4)
    dl, dv = ref["dlogits"], ref["dv"]
    dcore = dl @ wpi.astype(np.float64) + dv[:, None] * wv.astype(np.float64)
    rel = lambda a, b: np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)
    e_dcore = np.abs(g["dcore"] - dcore)[keep].max() / np.abs(dcore).max()
    gh = g["ghead"]
    gwpi, gbpi = gh[:A * H].reshape(A, H), gh[A * H:A * H + A]
    gwv, gbv = gh[A * H + A:A * H + A + H], gh[-1]
    e_heads = max(rel(gwpi, dl.T @ c64[:B]), rel(gbpi, dl.sum(0)), rel(gwv, dv @ c64[:B]),
                  abs(gbv - dv.sum()) / max(abs(dv.sum()), 1e-30))
    e_loss = (np.abs(g["stats"][:4] - ref["loss"]) / np.maximum(np.abs(ref["loss"]), 1)).max()
    record(f"traj_loss_injected_adv{adv_source}", max_rel_logits=e_lg, max_rel_values=e_v,
           max_rel_dcore=e_dcore, max_rel_head_grads=e_heads, max_rel_loss=e_loss,
           clip_edge_samples=int((~keep).sum()))
    assert e_dcore <= 1e-5 and e_heads <= 1e-5, (e_dcore, e_heads)
    assert np.all(np.abs(g["stats"][:4] - ref["loss"]) <= tol(ref["loss"])), (g["stats"], ref["loss"])
    assert abs(g["stats"][4] - ref["mean_ratio"]) <= 1e-5 * max(1.0, ref["mean_ratio"])
