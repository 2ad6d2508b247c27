"""Device sampler (synthetic envs + rollout writer) vs the oracle's restatement
of SyntheticLatencyEnv and the rollout contracts of orchestrator.hpp."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2006_11751_b200 as appo  # noqa: E402


@pytest.fixture(scope="module")
def setup():
    desc = appo.ModelDesc(3, 72, 128, 6, 32)
    ctx = appo.Context(0, seed=2, model=desc)
    n = 40
    store = appo.TrajectoryStore(desc, 2 * n)
    smp = appo.Sampler(ctx, n, episode_len=5, seed=77)
    for t in range(desc.T):
        smp.step(store, n, t)  # second half of the region
    torch.cuda.synchronize()
    return desc, ctx, store, smp, n


def env_start(e, episode_len):
    return (e * 2654435761) % episode_len


def test_observations_bit_exact(setup, oracle):
    desc, ctx, store, smp, n = setup
    for e in (0, 7, 39):
        step = env_start(e, 5)
        episode = 0
        for t in range(desc.T):
            es = oracle.L.orc_derive_seed(77, (e << 24) ^ episode)
            exp = oracle.gen_obs(es, step, desc.obs_dim)
            got = store.obs(n + e)[t].cpu().numpy()
            assert np.array_equal(got, exp), (e, t)
            step += 1
            if step >= 5:
                step, episode = 0, episode + 1
        es = oracle.L.orc_derive_seed(77, (e << 24) ^ episode)
        assert np.array_equal(store.boot_obs(n + e).cpu().numpy(),
                              oracle.gen_obs(es, step, desc.obs_dim))


def test_rewards_dones_versions_header(setup, oracle):
    desc, ctx, store, smp, n = setup
    for e in (3, 11):
        step, episode = env_start(e, 5), 0
        for t in range(desc.T):
            es = oracle.L.orc_derive_seed(77, (e << 24) ^ episode)
            r = oracle.L.orc_gen_reward(es, step + 1)
            assert abs(store.rewards(n + e)[t].item() - r) < 1e-6
            done = step + 1 >= 5
            assert store.dones(n + e)[t].item() == int(done)
            step += 1
            if done:
                step, episode = 0, episode + 1
        assert store.versions(n + e).cpu().tolist() == [0] * desc.T
        hdr = store.header(n + e)[:40].cpu().numpy().view(np.uint32)
        assert list(hdr[:6]) == [desc.T, desc.obs_dim, 512, 1, desc.T, e] and hdr[9] == 1
    # logp <= 0, actions in range (write_step contracts, trajstore.hpp:166-189)
    lp = torch.stack([store.logp(n + e) for e in range(n)])
    a = torch.stack([store.actions(n + e) for e in range(n)])
    assert (lp <= 1e-6).all() and (a >= 0).all() and (a < 6).all()


def test_hidden_recorded_is_input_and_reset_after_done(setup, oracle):
    desc, ctx, store, smp, n = setup
    for e in range(n):
        hid = store.hidden(n + e).cpu().numpy()
        dn = store.dones(n + e).cpu().numpy()
        assert np.all(hid[0] == 0)  # fresh sampler: zero initial hidden
        for t in range(1, desc.T):
            if dn[t - 1]:
                assert np.all(hid[t] == 0), (e, t)
            else:
                assert np.any(hid[t] != 0)


def test_logp_replays_under_recorded_version(setup, oracle):
    # test_orchestrator.cpp:112-145 analogue: re-running the policy on the stored
    # obs + stored input hidden reproduces the stored behaviour log-prob
    desc, ctx, store, smp, n = setup
    t = 3
    obs = torch.stack([store.obs(n + e)[t] for e in range(n)]).contiguous()
    hid = torch.stack([store.hidden(n + e)[t] for e in range(n)]).contiguous()
    acts = torch.stack([store.actions(n + e)[t] for e in range(n)])
    out = ctx.policy_forward(obs, hid, want_logits=True)
    lp, _ = ctx.log_prob_and_entropy(out["logits"], acts)
    stored = torch.stack([store.logp(n + e)[t] for e in range(n)])
    assert (lp - stored).abs().max().item() < 1e-4


def test_learner_consumes_sampler_slots(setup):
    desc, ctx, store, smp, n = setup
    out = ctx.learner_step(store.region, store.slot_bytes, list(range(n, 2 * n)))
    assert np.isfinite(out["total_loss"]) and out["version"] == 1
    assert out["lag_mean"] == 0.0  # every step stamped with version 0


def test_overlapped_sampler_and_learner_streams():
    # APPO decoupling: the sampler runs on a context sharing the model on its own
    # stream while the learner trains on the other rollout set.  Inference must
    # only ever see complete published versions: stamped versions are
    # non-decreasing within a trajectory (trajstore.hpp:174-176) and never ahead
    # of the learner.
    desc = appo.ModelDesc(3, 72, 128, 6, 32)
    learner = appo.Context(0, seed=4, model=desc)
    actor = learner.shared()
    n = 128
    store = appo.TrajectoryStore(desc, 2 * n)
    smp = appo.Sampler(actor, n, episode_len=9, seed=5)
    ids = np.arange(n, dtype=np.int32).reshape(-1, 32)
    for k in range(4):
        base = (k % 2) * n
        for t in range(desc.T):
            smp.step(store, base, t)
        if k > 0:
            prev = ((k - 1) % 2) * n
            for mb in ids:
                learner.learner_submit(store.region, store.slot_bytes, mb + prev)
            out = learner.learner_collect()
            assert np.isfinite(out["total_loss"])
        torch.cuda.synchronize()
    final = learner.version
    assert final == 3 * len(ids)
    for s in range(2 * n):
        v = store.versions(s).cpu().numpy()
        assert np.all(np.diff(v) >= 0) and v.min() >= 0 and v.max() <= final


def test_host_observations_staged_into_slots():
    # CPU-actor path: pinned host obs per step, copied on the sampler's copy
    # stream through two staging buffers and scattered into the slots
    desc = appo.ModelDesc(3, 72, 128, 6, 32)
    ctx = appo.Context(0, seed=4, model=desc)
    n = 24
    store = appo.TrajectoryStore(desc, 2 * n)
    smp = appo.Sampler(ctx, n, episode_len=9, seed=5)
    rs = np.random.default_rng(7)
    host = [torch.from_numpy(rs.integers(0, 256, (n, desc.obs_dim), dtype=np.uint8)).pin_memory()
            for _ in range(desc.T)]
    acts = torch.empty(n, dtype=torch.int32).pin_memory()
    for rep in range(2):  # second rollout reuses the staging buffers
        for t in range(desc.T):
            smp.step(store, n * rep, t, h_obs=host[(t + rep) % desc.T], h_actions=acts)
        torch.cuda.synchronize()
        for e in (0, 11, n - 1):
            got = store.obs(n * rep + e).cpu()
            for t in range(desc.T):
                assert torch.equal(got[t], host[(t + rep) % desc.T][e]), (rep, e, t)
