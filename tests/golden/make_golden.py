"""Generates the golden vectors in tests/golden/ from the REFERENCE itself.

Run in the build container (needs /root/reference, via oracle/_ref/libappo_ref.so
built by ``make -C oracle``):

    python tests/golden/make_golden.py

Every array stored here is an output of the unmodified reference headers
(oracle/ref_shim.cpp forwards to offpolicy.hpp / policy.hpp / trajstore.hpp),
on inputs drawn exactly as the reference's own tests draw them where the
test names a seed (acceptance.cpp:42-56, test_offpolicy.cpp:20-34), otherwise
from numpy with the seed recorded here.  The GPU box has no /root/reference,
so tests read these fixtures instead.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle.oracle import Reference  # noqa: E402


def pack_instances(insts):
    T = max(len(x["rewards"]) for x in insts)
    n = len(insts)
    out = {k: np.zeros((n, T)) for k in ["rewards", "values", "tlogp", "blogp"]}
    out["dones"] = np.zeros((n, T), dtype=np.uint8)
    out["bootstrap"] = np.zeros(n)
    out["T"] = np.array([len(x["rewards"]) for x in insts], dtype=np.int32)
    for i, x in enumerate(insts):
        t = len(x["rewards"])
        for k in ["rewards", "values", "tlogp", "blogp", "dones"]:
            out[k][i, :t] = x[k]
        out["bootstrap"][i] = x["bootstrap"]
    return out


def main():
    ref = Reference()

    # 1. V-trace known answer, test_offpolicy.cpp:71-86
    st, (v, pg, rho, c) = ref.vtrace([1.0, 1.0], [0.0, 0.0], 0.0, [-0.5, -0.7], [-0.5, -0.7],
                                     [0, 0], 1.0, 1.0, 1.0)
    assert st == 0
    np.savez(os.path.join(HERE, "vtrace_kat.npz"), rewards=[1.0, 1.0], values=[0.0, 0.0],
             bootstrap=0.0, tlogp=[-0.5, -0.7], blogp=[-0.5, -0.7], dones=np.array([0, 0], np.uint8),
             gamma=1.0, v=v, pg_adv=pg, rho=rho, c=c)

    # 2. acceptance criterion 1 (acceptance.cpp:83-115): 500 instances, seed 101,
    #    T = 1 + rep % 16, rho_bar = 1 + (rep % 3) * 0.25, c_bar = 1, gamma 0.99;
    #    then 100 on-policy instances (gamma 0.95) from the same engine.
    Ts = [1 + rep % 16 for rep in range(500)] + [1 + rep % 16 for rep in range(100)]
    insts = ref.random_instances(101, Ts)
    main_i, onp = insts[:500], insts[500:]
    pk = pack_instances(main_i)
    n, Tm = pk["rewards"].shape
    V = np.zeros((n, Tm)); PG = np.zeros((n, Tm)); RHO = np.zeros((n, Tm)); CC = np.zeros((n, Tm))
    rho_bar = np.array([1.0 + (rep % 3) * 0.25 for rep in range(500)])
    for i, x in enumerate(main_i):
        st, (v, pg, r_, c_) = ref.vtrace(x["rewards"], x["values"], x["bootstrap"], x["tlogp"],
                                         x["blogp"], x["dones"], rho_bar[i], 1.0, 0.99)
        assert st == 0
        t = len(v)
        V[i, :t], PG[i, :t], RHO[i, :t], CC[i, :t] = v, pg, r_, c_
    pk2 = pack_instances(onp)
    n2, T2 = pk2["rewards"].shape
    V2 = np.zeros((n2, T2)); RET2 = np.zeros((n2, T2))
    for i, x in enumerate(onp):
        st, (v, pg, r_, c_) = ref.vtrace(x["rewards"], x["values"], x["bootstrap"], x["tlogp"],
                                         x["tlogp"], x["dones"], 1.0, 1.0, 0.95)
        assert st == 0
        t = len(v)
        V2[i, :t] = v
        RET2[i, :t] = ref.nstep_returns(x["rewards"], x["bootstrap"], x["dones"], 0.95)
    np.savez(os.path.join(HERE, "vtrace_accept1.npz"), **pk, rho_bar=rho_bar, v=V, pg_adv=PG,
             rho=RHO, c=CC, **{"onp_" + k: val for k, val in pk2.items()}, onp_v=V2,
             onp_ret=RET2)

    # 3. config 1: 256 trajectories x T=32 (BASELINE.json configs[0]) drawn with
    #    the acceptance generator from seed 101, gamma 0.99, rho_bar = c_bar = 1.
    insts = ref.random_instances(101, [32] * 256)
    pk = pack_instances(insts)
    V = np.zeros((256, 32)); PG = np.zeros((256, 32)); RET = np.zeros((256, 32))
    for i, x in enumerate(insts):
        st, (v, pg, _, _) = ref.vtrace(x["rewards"], x["values"], x["bootstrap"], x["tlogp"],
                                       x["blogp"], x["dones"], 1.0, 1.0, 0.99)
        assert st == 0
        V[i], PG[i] = v, pg
        RET[i] = ref.nstep_returns(x["rewards"], x["bootstrap"], x["dones"], 0.99)
    np.savez(os.path.join(HERE, "vtrace_c1.npz"), **pk, v=V, pg_adv=PG, nstep=RET)

    # 4. PPO clip + total loss (offpolicy.hpp:117-168), numpy inputs seed 41
    rs = np.random.default_rng(41)
    ratio = rs.uniform(0.01, 5.0, 10000)
    A = rs.uniform(-3.0, 3.0, 10000)
    ratio[:4] = [1.1, 1 / 1.1, 1.0, 1.1]  # ties with the clip bounds
    obj = np.array([ref.L.ref_ppo_objective(r, a, 1 / 1.1, 1.1) for r, a in zip(ratio, A)])
    dr = np.array([ref.L.ref_ppo_dratio(r, a, 1 / 1.1, 1.1) for r, a in zip(ratio, A)])
    n = 8192
    lr = rs.uniform(-0.4, 0.4, n)
    ratios = np.exp(lr)
    adv = rs.normal(size=n)
    values = rs.normal(size=n)
    vt = rs.normal(size=n)
    ent = rs.uniform(0, np.log(6), n)
    st, loss = ref.total_loss(ratios, adv, values, vt, ent)
    assert st == 0
    np.savez(os.path.join(HERE, "ppo.npz"), ratio=ratio, adv=A, objective=obj, dratio=dr,
             l_ratios=ratios, l_adv=adv, l_values=values, l_vt=vt, l_ent=ent, loss=loss)

    # 5. heads: softmax / logp / entropy on 6-action logits (policy.hpp:214-281)
    lg = rs.normal(scale=2.0, size=(512, 6))
    lg[0] = [1e9, 0, 0, 0, 0, 0]  # degenerate, test_policy.cpp:195-203
    acts = rs.integers(0, 6, 512).astype(np.int32)
    P = np.stack([ref.softmax(x) for x in lg])
    LP = np.zeros(512); EN = np.zeros(512)
    for i in range(512):
        st, LP[i], EN[i] = ref.logp_entropy(lg[i], acts[i])
        assert st == 0
    # sampling frequencies: 10^6 draws from mt19937_64(14) (test_policy.cpp:205-224)
    freq_logits = np.array([0.3, -0.8, 1.1, 0.0])
    fa, _ = ref.sample_actions(freq_logits, 14, 1000000)
    counts = np.bincount(fa, minlength=4)
    np.savez(os.path.join(HERE, "heads.npz"), logits=lg, actions=acts, probs=P, logp=LP,
             entropy=EN, freq_logits=freq_logits, freq_counts=counts)

    # 6. Adam + global-norm clip (policy.hpp:431-455): 5 steps on a 4096 vector,
    #    gradient norms straddling the clip; plus the "norm 8 halved" case.
    n = 4096
    th = rs.normal(size=n); m = np.zeros(n); v = np.zeros(n); t = 0
    th0 = th.copy()
    grads = [rs.normal(size=n) * s for s in (0.01, 0.5, 0.05, 2.0, 0.001)]
    thetas, ms, vs = [], [], []
    for g in grads:
        st, t = ref.optimizer_step(th, m, v, g, t)
        assert st == 0
        thetas.append(th.copy()); ms.append(m.copy()); vs.append(v.copy())
    np.savez(os.path.join(HERE, "adam.npz"), theta0=th0, grads=np.stack(grads),
             thetas=np.stack(thetas), ms=np.stack(ms), vs=np.stack(vs))

    # 7. trajectory slot layout (trajstore.hpp:62-87), reference f64 element types
    shapes = [(32, 27648, 512, 1), (16, 6, 2, 3), (8, 6, 2, 3), (32, 60, 0, 4), (32, 32, 64, 1)]
    offs = np.array([ref.slot_offsets(*s) for s in shapes], dtype=np.uint64)
    np.savez(os.path.join(HERE, "layout.npz"), shapes=np.array(shapes, dtype=np.uint32),
             offsets=offs)
    # 8. PPO loss + its logit / value gradient from the reference's own
    #    compute_gradients with injected logits and values (policy.hpp:302-428,
    #    ref_shim.cpp ref_ppo_grads_injected): fp32-representable inputs, 6
    #    actions, a few samples beyond the +-20 log-ratio clamp
    #    (offpolicy.hpp:48-54).
    rs = np.random.default_rng(77)
    n, A = 1024, 6
    lg = rs.normal(scale=1.5, size=(n, A)).astype(np.float32).astype(np.float64)
    vals = rs.normal(size=n).astype(np.float32).astype(np.float64)
    acts = rs.integers(0, A, n).astype(np.int32)
    shift = rs.uniform(-0.3, 0.3, n)
    shift[:8] = [25.0, -25.0, 21.0, -21.0, 19.5, -19.5, 30.0, -30.0]  # clamp
    lp = np.zeros(n)
    for i in range(n):
        _, lp[i], _ = ref.logp_entropy(lg[i], acts[i])
    blogp = (lp - shift).astype(np.float32).astype(np.float64)
    advs = rs.normal(size=n).astype(np.float32).astype(np.float64)
    vt = rs.normal(size=n).astype(np.float32).astype(np.float64)
    st, g = ref.ppo_grads_injected(lg, vals, acts, blogp, advs, vt)
    assert st == 0
    np.savez(os.path.join(HERE, "ppo_grad.npz"), logits=lg, values=vals, actions=acts,
             blogp=blogp, adv=advs, vt=vt, dlogits=g["dlogits"], dv=g["dv"], loss=g["loss"],
             mean_ratio=g["mean_ratio"])
    # 9. factored action heads (ActionHeadsSpec, policy.hpp:25-35,262-281): the
    #    full Doom factored space {3,3,2,2,2,8,21} (test_policy.cpp:188-193),
    #    {3,4} (:254-290) and the two-binary-head uniform KAT (:241-252).
    rs = np.random.default_rng(91)
    fact = {}
    for name, sizes in (("doom", [3, 3, 2, 2, 2, 8, 21]), ("h34", [3, 4]), ("h22", [2, 2])):
        B = 256
        lg = rs.uniform(-2, 2, (B, sum(sizes))).astype(np.float32).astype(np.float64)
        if name == "h22":
            lg[0] = 0.0
        acts = np.stack([rs.integers(0, n, B) for n in sizes], 1).astype(np.int32)
        if name == "h22":
            acts[0] = [0, 1]
        st, lp, en = ref.logp_entropy_heads(sizes, lg, acts)
        assert st == 0
        fact.update({f"{name}_sizes": np.array(sizes, np.int32), f"{name}_logits": lg,
                     f"{name}_actions": acts, f"{name}_logp": lp, f"{name}_entropy": en})
    np.savez(os.path.join(HERE, "heads_factored.npz"), **fact)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
