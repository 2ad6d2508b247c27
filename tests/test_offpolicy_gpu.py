"""CUDA V-trace / n-step / GAE / PPO loss / heads / Adam vs the oracle and
the reference's golden vectors.  Tolerance (north_star):
|got - ref| <= 1e-5 * max(|ref|, 1) for fp32 device math vs fp64 reference."""
import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu

import paper_2006_11751_b200 as appo  # noqa: E402

TOL = 1e-5


def close(got, ref, tol=TOL):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)
    return err.max() if err.size else 0.0


@pytest.fixture(scope="module")
def ctx():
    return appo.Context(0)


def dev(x, dt=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(x)).to(dtype=dt, device="cuda")


def test_vtrace_config1_matches_reference(ctx):
    g = golden("vtrace_c1")
    v, pg, rho, c = ctx.vtrace(dev(g["rewards"]), dev(g["values"]), dev(g["bootstrap"]),
                               dev(g["tlogp"]), dev(g["blogp"]), dev(g["dones"], torch.uint8),
                               gamma=0.99, with_weights=True)
    assert close(v.cpu(), g["v"]) <= TOL
    assert close(pg.cpu(), g["pg_adv"]) <= TOL
    ret = ctx.nstep_returns(dev(g["rewards"]), dev(g["bootstrap"]), dev(g["dones"], torch.uint8),
                            0.99)
    assert close(ret.cpu(), g["nstep"]) <= TOL


def test_vtrace_acceptance_instances(ctx):
    # acceptance criterion 1 instances (T = 1..16, rho_bar in {1, 1.25, 1.5})
    g = golden("vtrace_accept1")
    for rb in (1.0, 1.25, 1.5):
        for T in range(1, 17):
            idx = [i for i in range(500) if g["T"][i] == T and abs(g["rho_bar"][i] - rb) < 1e-9]
            if not idx:
                continue
            sl = lambda k: dev(g[k][idx][:, :T])
            v, pg = ctx.vtrace(sl("rewards"), sl("values"), dev(g["bootstrap"][idx]), sl("tlogp"),
                               sl("blogp"), dev(g["dones"][idx][:, :T], torch.uint8), gamma=0.99,
                               rho_bar=rb, c_bar=1.0)
            assert close(v.cpu(), g["v"][idx][:, :T]) <= TOL
            assert close(pg.cpu(), g["pg_adv"][idx][:, :T]) <= TOL


def test_vtrace_known_answer_and_long_T(ctx, oracle):
    g = golden("vtrace_kat")
    v, pg = ctx.vtrace(dev([g["rewards"]]), dev([g["values"]]), dev([float(g["bootstrap"])]),
                       dev([g["tlogp"]]), dev([g["blogp"]]), dev([g["dones"]], torch.uint8),
                       gamma=1.0)
    assert np.allclose(v.cpu().numpy(), [[2.0, 1.0]]) and np.allclose(pg.cpu().numpy(), [[2, 1]])
    # T > 32 exercises the multi-step-per-lane path
    rs = np.random.default_rng(9)
    for T in (33, 100, 257):
        n = 5
        r = rs.uniform(-1, 1, (n, T)); vv = rs.uniform(-1, 1, (n, T)); b = rs.uniform(-1, 1, n)
        tl = rs.uniform(-2.5, -0.1, (n, T)); bl = rs.uniform(-2.5, -0.1, (n, T))
        d = (rs.uniform(size=(n, T)) < 0.05).astype(np.uint8)
        st, (ov, opg, _, _) = oracle.vtrace_batch(r, vv, b, tl, bl, d, 1.2, 1.0, 0.99)
        v, pg = ctx.vtrace(dev(r), dev(vv), dev(b), dev(tl), dev(bl), dev(d, torch.uint8),
                           gamma=0.99, rho_bar=1.2, c_bar=1.0)
        assert close(v.cpu(), ov) <= TOL and close(pg.cpu(), opg) <= TOL


def test_vtrace_errors(ctx):
    x = dev(np.zeros((1, 1)))
    d = dev(np.zeros((1, 1)), torch.uint8)
    with pytest.raises(appo.ConfigError):
        ctx.vtrace(x, x, dev([0.0]), x, x, d, rho_bar=0.5, c_bar=1.0)
    with pytest.raises(appo.ConfigError):
        ctx.vtrace(x, x, dev([0.0]), x, x, d, gamma=0.0)
    with pytest.raises(appo.NumericError):
        ctx.vtrace(dev([[np.nan]]), x, dev([0.0]), x, x, d)
    ctx.vtrace(x, x, dev([0.0]), x, x, d)  # flag cleared, next call fine


def test_vtrace_done_cuts_influence(ctx):
    rs = np.random.default_rng(31)
    r = rs.uniform(-1, 1, (1, 10)); v = rs.uniform(-1, 1, (1, 10))
    tl = rs.uniform(-2.5, -0.1, (1, 10)); bl = rs.uniform(-2.5, -0.1, (1, 10))
    d = np.zeros((1, 10), np.uint8); d[0, 4] = 1
    a = ctx.vtrace(dev(r), dev(v), dev([0.3]), dev(tl), dev(bl), dev(d, torch.uint8))
    r2, v2 = r.copy(), v.copy(); r2[0, 5:] += 13.37; v2[0, 5:] -= 7.7
    b = ctx.vtrace(dev(r2), dev(v2), dev([99.0]), dev(tl), dev(bl), dev(d, torch.uint8))
    assert torch.equal(a[0][0, :5], b[0][0, :5]) and torch.equal(a[1][0, :5], b[1][0, :5])


def test_gae(ctx, oracle):
    g = golden("vtrace_c1")
    for lam in (1.0, 0.95, 0.0):
        adv, ret = ctx.gae(dev(g["rewards"]), dev(g["values"]), dev(g["bootstrap"]),
                           dev(g["dones"], torch.uint8), 0.99, lam)
        exp = np.stack([oracle.gae(g["rewards"][i], g["values"][i], g["bootstrap"][i],
                                   g["dones"][i], 0.99, lam)[0] for i in range(256)])
        assert close(adv.cpu(), exp) <= TOL
        assert close(ret.cpu(), exp + g["values"]) <= TOL
        if lam == 1.0:  # reference NStep advantage (orchestrator.hpp:831-833)
            assert close(adv.cpu(), g["nstep"] - g["values"]) <= TOL


def test_total_loss(ctx):
    g = golden("ppo")
    out = ctx.total_loss(dev(g["l_ratios"]), dev(g["l_adv"]), dev(g["l_values"]), dev(g["l_vt"]),
                         dev(g["l_ent"]))
    got = [out["policy"], out["value"], out["entropy"], out["total"]]
    assert close(got, g["loss"]) <= TOL
    with pytest.raises(appo.ConfigError):
        ctx.total_loss(dev([1.0]), dev([1.0]), dev([1.0]), dev([1.0]), dev([1.0]), clip_low=1.2)


def test_heads(ctx, oracle):
    g = golden("heads")
    lg = g["logits"][1:]  # skip the 1e9 row (fp32 logits)
    lp, en = ctx.log_prob_and_entropy(dev(lg), dev(g["actions"][1:], torch.int32))
    assert close(lp.cpu(), g["logp"][1:]) <= TOL and close(en.cpu(), g["entropy"][1:]) <= TOL
    with pytest.raises(appo.ContractError):
        ctx.log_prob_and_entropy(dev(lg[:2]), dev([0, 6], torch.int32))
    # sampler: same counter-based uniforms as the oracle -> same actions
    key = 1234
    a, lpa = ctx.sample_actions(dev(lg), key, 0)
    for i in range(len(lg)):
        u = oracle.L.orc_uniform(key, i)
        ea, elp = oracle.sample(lg[i].astype(np.float32).astype(np.float64), u)
        assert a[i].item() == ea
        assert abs(lpa[i].item() - elp) <= 1e-5 * max(abs(elp), 1)


def test_sampling_frequencies(ctx):
    # test_policy.cpp:205-224, 10^6 draws within 3 sigma
    g = golden("heads")
    logits = np.tile(g["freq_logits"], (1000000, 1))
    a, _ = ctx.sample_actions(dev(logits), 77, 0)
    counts = np.bincount(a.cpu().numpy(), minlength=4)
    p = np.exp(g["freq_logits"]) / np.exp(g["freq_logits"]).sum()
    N = 1000000
    assert np.all(np.abs(counts - N * p) < 3 * np.sqrt(N * p * (1 - p)))


def test_adam_sequence(ctx):
    g = golden("adam")
    th = dev(g["theta0"]); m = torch.zeros_like(th); v = torch.zeros_like(th)
    for k in range(len(g["grads"])):
        norm = ctx.optimizer_step(th, m, v, dev(g["grads"][k]), k + 1)
        assert abs(norm - np.linalg.norm(g["grads"][k])) <= 1e-5 * norm
        assert close(th.cpu(), g["thetas"][k]) <= TOL
        assert close(m.cpu(), g["ms"][k]) <= TOL


def test_adam_nonfinite_leaves_params(ctx):
    th = dev(np.ones(1000)); m = torch.zeros_like(th); v = torch.zeros_like(th)
    gr = dev(np.ones(1000)); gr[17] = float("nan")
    with pytest.raises(appo.NumericError):
        ctx.optimizer_step(th, m, v, gr, 1)
    assert torch.equal(th, torch.ones_like(th))


def test_large_sweep_vs_oracle(ctx, oracle):
    # 65,536 x 32 config-1 sweep shape (random subset checked against the oracle)
    rs = np.random.default_rng(3)
    n, T = 65536, 32
    r = rs.uniform(-1, 1, (n, T)).astype(np.float32); vv = rs.uniform(-1, 1, (n, T)).astype(np.float32)
    tl = rs.uniform(-2.5, -0.1, (n, T)).astype(np.float32); bl = rs.uniform(-2.5, -0.1, (n, T)).astype(np.float32)
    d = (rs.uniform(size=(n, T)) < 0.15).astype(np.uint8); b = rs.uniform(-1, 1, n).astype(np.float32)
    v, pg = ctx.vtrace(dev(r), dev(vv), dev(b), dev(tl), dev(bl), dev(d, torch.uint8))
    idx = rs.choice(n, 64, replace=False)
    st, (ov, opg, _, _) = oracle.vtrace_batch(r[idx].astype(np.float64), vv[idx].astype(np.float64),
                                              b[idx].astype(np.float64), tl[idx].astype(np.float64),
                                              bl[idx].astype(np.float64), d[idx], 1.0, 1.0, 0.99)
    assert close(v.cpu().numpy()[idx], ov) <= TOL and close(pg.cpu().numpy()[idx], opg) <= TOL


@pytest.mark.parametrize("name", ["doom", "h34", "h22"])
def test_factored_heads_logp_entropy(ctx, name):
    """log_prob_and_entropy over factored heads vs the reference
    (heads_factored.npz: {3,3,2,2,2,8,21}, {3,4}, and the 2 ln 2 KAT)."""
    g = golden("heads_factored")
    sizes = [int(x) for x in g[f"{name}_sizes"]]
    lp, en = ctx.log_prob_and_entropy_heads(sizes, dev(g[f"{name}_logits"]),
                                            dev(g[f"{name}_actions"], torch.int32))
    assert close(lp.cpu(), g[f"{name}_logp"]) <= TOL
    assert close(en.cpu(), g[f"{name}_entropy"]) <= TOL
    bad = g[f"{name}_actions"][:2].copy()
    bad[1, -1] = sizes[-1]  # out of range for the last head: ContractError
    with pytest.raises(appo.ContractError):
        ctx.log_prob_and_entropy_heads(sizes, dev(g[f"{name}_logits"][:2]), dev(bad, torch.int32))


def test_factored_heads_sampling(ctx, oracle):
    """sample_action over factored heads: per head the oracle's inverse CDF on
    the same counter-based uniform, joint logp = sum; and per-head marginal
    frequencies within 3 sigma over 2e5 rows."""
    g = golden("heads_factored")
    sizes = [int(x) for x in g["doom_sizes"]]
    lg = g["doom_logits"]
    key = 4321
    a, lpa = ctx.sample_actions_heads(sizes, dev(lg), key, 5)
    a = a.cpu().numpy()
    off = np.concatenate([[0], np.cumsum(sizes)])
    n = len(sizes)
    for b in range(len(lg)):
        tot = 0.0
        for j in range(n):
            u = oracle.L.orc_uniform(key, 5 + b * n + j)
            ea, elp = oracle.sample(lg[b, off[j]:off[j + 1]].astype(np.float32).astype(np.float64), u)
            assert a[b, j] == ea
            tot += elp
        assert abs(lpa[b].item() - tot) <= 1e-5 * max(abs(tot), 1)
    N = 200000
    a, _ = ctx.sample_actions_heads(sizes, dev(np.tile(lg[0], (N, 1))), 9, 0)
    a = a.cpu().numpy()
    for j in range(n):
        x = lg[0, off[j]:off[j + 1]]
        p = np.exp(x - x.max()); p /= p.sum()
        c = np.bincount(a[:, j], minlength=sizes[j])
        assert np.all(np.abs(c - N * p) < 3.5 * np.sqrt(N * p * (1 - p)) + 1)
