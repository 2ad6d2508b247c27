"""CPU-actor rollout path: appo_rollout_act / _feedback restate
RolloutWorker::submit_group + step_group (orchestrator.hpp:435-552) with every
input from host memory -- observations, rewards, dones and the bootstrap
observation.  Every slot field must equal the host inputs (or, for the
policy's outputs, the actions returned to the host and the oracle's
inference), and a sampler-written slot dumps byte-identically to the
reference's dump_trajectory of the same records."""
import struct

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2006_11751_b200 as appo  # noqa: E402


H_TOL = 1.5e-2     # max |d h'| (bf16 operands), as tests/test_model_gpu.py
LOGP_TOL = 2e-3    # stored behaviour logp vs the oracle's log-softmax


def host(x):
    return torch.from_numpy(np.ascontiguousarray(x)).pin_memory()


@pytest.fixture(scope="module")
def rollout():
    desc = appo.ModelDesc(3, 72, 128, 6, 32)
    T = desc.T
    ctx = appo.Context(0, seed=21, model=desc)
    n = 24
    store = appo.TrajectoryStore(desc, 2 * n)
    smp = appo.Sampler(ctx, n, episode_len=1000, seed=3)
    q = appo.SlotQueue(0, 2 * n)
    smp.set_ready_queue(q)
    rs = np.random.default_rng(12)
    rec = []
    for rep in range(2):  # the second rollout continues the first one's hidden state
        obs = rs.integers(0, 256, (T, n, desc.obs_dim), dtype=np.uint8)
        rew = rs.uniform(-1, 1, (T, n)).astype(np.float32)
        dn = (rs.uniform(size=(T, n)) < 0.1).astype(np.uint8)
        nxt = rs.integers(0, 256, (n, desc.obs_dim), dtype=np.uint8)
        acts = np.zeros((T, n), np.int32)
        h_obs = [host(obs[t]) for t in range(T)]
        h_act = torch.empty(n, dtype=torch.int32).pin_memory()
        for t in range(T):
            smp.act(store, rep * n, t, h_obs[t], h_act)
            smp.wait()  # the actor needs the actions before stepping its envs
            acts[t] = h_act.numpy()
            smp.feedback(store, rep * n, t, host(rew[t]), host(dn[t]),
                         host(nxt) if t == T - 1 else None)
        smp.wait()
        rec.append(dict(obs=obs, rew=rew, dn=dn, nxt=nxt, acts=acts))
    torch.cuda.synchronize()
    popped = q.pop(ctx, 2 * n)
    ctx.sync()
    return dict(desc=desc, ctx=ctx, n=n, store=store, rec=rec, popped=popped.cpu().numpy())


def test_slot_fields_equal_host_inputs(rollout):
    desc, store, n = rollout["desc"], rollout["store"], rollout["n"]
    T = desc.T
    for rep, r in enumerate(rollout["rec"]):
        for e in range(n):
            s = rep * n + e
            assert np.array_equal(store.obs(s).cpu().numpy(), r["obs"][:, e]), (rep, e)
            assert np.array_equal(store.rewards(s).cpu().numpy(), r["rew"][:, e])
            assert np.array_equal(store.dones(s).cpu().numpy(), r["dn"][:, e])
            assert np.array_equal(store.actions(s).cpu().numpy(), r["acts"][:, e])
            assert np.array_equal(store.boot_obs(s).cpu().numpy(), r["nxt"][e])
            assert np.all(store.versions(s).cpu().numpy() == 0)
            hdr = struct.unpack("<10I", bytes(store.header(s)[:40].cpu().numpy()))
            assert hdr == (T, desc.obs_dim, 512, 1, T, e, 0, 0, 0, 1)
    # sealed slots entered the ready queue in env order, rollout after rollout
    assert rollout["popped"].tolist() == list(range(2 * n))


def test_hidden_chain_and_logp_match_oracle(rollout, oracle):
    """Stored hidden rows: h_0 = 0, h_{t+1} = GRU(x_t, h_t) * (1 - done_t)
    (orchestrator.hpp:402,518-524); bootstrap hidden = h'_{T-1}; behaviour logp =
    log pi(a_t) under the oracle's forward on the same inputs."""
    desc, ctx, store, n = rollout["desc"], rollout["ctx"], rollout["store"], rollout["n"]
    T = desc.T
    th, _ = ctx.get_params()
    th = th.astype(np.float64)
    shape = (3, 72, 128, 6)
    envs = [0, 5, n - 1]
    r = rollout["rec"][0]
    h = np.zeros((len(envs), 512))
    for t in range(T):
        got_h = np.stack([store.hidden(e)[t].cpu().numpy() for e in envs])
        assert np.abs(got_h - h).max() <= H_TOL, t
        if t > 0:  # a reset row is exactly zero
            for i, e in enumerate(envs):
                if r["dn"][t - 1, e]:
                    assert not got_h[i].any()
        out = oracle.policy_forward(shape, th, r["obs"][t, envs], got_h.astype(np.float64))
        lg = out["logits"]
        ls = lg - lg.max(1, keepdims=True)
        ls = ls - np.log(np.exp(ls).sum(1, keepdims=True))
        for i, e in enumerate(envs):
            a = r["acts"][t, e]
            assert abs(store.logp(e)[t].item() - ls[i, a]) <= LOGP_TOL, (t, e)
        hn = out["h_out"]
        if t == T - 1:
            boot = np.stack([store.boot_hidden(e).cpu().numpy() for e in envs])
            assert np.abs(boot - hn).max() <= H_TOL
        h = hn * (1 - r["dn"][t, envs])[:, None]
    # the second rollout starts from the first one's final (reset-masked) hidden
    h1 = np.stack([store.hidden(n + e)[0].cpu().numpy() for e in envs])
    assert np.abs(h1 - h).max() <= H_TOL


def test_sampler_written_slot_dumps_like_reference(rollout, tmp_path):
    """dump_trajectory (trajstore.hpp:335-359) by the reference of a slot it
    fills through write_step / set_bootstrap with the host records plus the
    policy outputs, vs to_reference_dump of the device-written slot."""
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    ref = Reference()
    store, n = rollout["store"], rollout["n"]
    r = rollout["rec"][1]
    for e in (2, n - 1):
        s = n + e
        path = str(tmp_path / f"d{e}.bin")
        st = ref.dump_trajectory(path, r["obs"][:, e].astype(np.float64),
                                 store.hidden(s).cpu().numpy().astype(np.float64),
                                 r["acts"][:, e], r["rew"][:, e].astype(np.float64),
                                 store.logp(s).cpu().numpy().astype(np.float64),
                                 r["dn"][:, e], store.versions(s).cpu().numpy(),
                                 r["nxt"][e].astype(np.float64),
                                 store.boot_hidden(s).cpu().numpy().astype(np.float64))
        assert st == 0
        assert store.to_reference_dump(s) == open(path, "rb").read()


def test_rollout_order_contract():
    """write_step's ordering (trajstore.hpp:172-174) and seal's completeness
    (:269) apply to the host-fed writer."""
    desc = appo.ModelDesc(3, 72, 128, 6, 2)
    ctx = appo.Context(0, seed=2, model=desc)
    n = 4
    store = appo.TrajectoryStore(desc, n)
    smp = appo.Sampler(ctx, n, seed=1)
    obs = host(np.zeros((n, desc.obs_dim), np.uint8))
    rew, dn = host(np.zeros(n, np.float32)), host(np.zeros(n, np.uint8))
    with pytest.raises(appo.ContractError):
        smp.feedback(store, 0, 0, rew, dn)          # feedback before act
    with pytest.raises(appo.ContractError):
        smp.act(store, 0, 1, obs)                   # step 1 before step 0
    smp.act(store, 0, 0, obs)
    with pytest.raises(appo.ContractError):
        smp.act(store, 0, 0, obs)                   # act twice
    smp.feedback(store, 0, 0, rew, dn)
    smp.act(store, 0, 1, obs)
    with pytest.raises(appo.ContractError):
        smp.feedback(store, 0, 1, rew, dn)          # last step without a bootstrap obs
    smp.feedback(store, 0, 1, rew, dn, obs)
    smp.wait()
    ctx.sync()
