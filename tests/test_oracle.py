"""Pins the oracle restatement (oracle/appo_oracle.c) before anything trusts it:
against the golden vectors generated from the reference (tests/golden/) and,
where oracle/_ref is built, against the live reference.  CPU only."""
import numpy as np
import pytest

from conftest import golden


def test_vtrace_known_answer(oracle):
    # test_offpolicy.cpp:71-86
    g = golden("vtrace_kat")
    st, (v, pg, rho, c) = oracle.vtrace(g["rewards"], g["values"], float(g["bootstrap"]),
                                        g["tlogp"], g["blogp"], g["dones"], 1.0, 1.0, 1.0)
    assert st == 0
    np.testing.assert_allclose(v, [2.0, 1.0], atol=1e-12)
    np.testing.assert_allclose(pg, [2.0, 1.0], atol=1e-12)
    np.testing.assert_array_equal(v, g["v"])


def test_vtrace_acceptance_criterion1(oracle):
    # acceptance.cpp:83-115: 500 instances, tol 1e-12 (oracle matches ref bit-for-bit
    # in practice since the recursion is restated in the same order)
    g = golden("vtrace_accept1")
    worst = 0.0
    for i in range(len(g["T"])):
        T = int(g["T"][i])
        st, (v, pg, rho, c) = oracle.vtrace(g["rewards"][i, :T], g["values"][i, :T],
                                            g["bootstrap"][i], g["tlogp"][i, :T],
                                            g["blogp"][i, :T], g["dones"][i, :T],
                                            g["rho_bar"][i], 1.0, 0.99)
        assert st == 0
        worst = max(worst, np.abs(v - g["v"][i, :T]).max(), np.abs(pg - g["pg_adv"][i, :T]).max(),
                    np.abs(rho - g["rho"][i, :T]).max(), np.abs(c - g["c"][i, :T]).max())
    assert worst < 1e-12
    # on-policy reduction to n-step returns
    for i in range(len(g["onp_T"])):
        T = int(g["onp_T"][i])
        ret = oracle.nstep_returns(g["onp_rewards"][i, :T], g["onp_bootstrap"][i],
                                   g["onp_dones"][i, :T], 0.95)
        np.testing.assert_allclose(ret, g["onp_ret"][i, :T], atol=1e-12)
        np.testing.assert_allclose(g["onp_v"][i, :T], ret, atol=1e-12)


def test_vtrace_config1(oracle):
    g = golden("vtrace_c1")
    st, (v, pg, _, _) = oracle.vtrace_batch(g["rewards"], g["values"], g["bootstrap"],
                                            g["tlogp"], g["blogp"], g["dones"], 1.0, 1.0, 0.99)
    assert st == 0
    np.testing.assert_allclose(v, g["v"], atol=1e-12, rtol=0)
    np.testing.assert_allclose(pg, g["pg_adv"], atol=1e-12, rtol=0)
    for i in range(4):
        ret = oracle.nstep_returns(g["rewards"][i], g["bootstrap"][i], g["dones"][i], 0.99)
        np.testing.assert_allclose(ret, g["nstep"][i], atol=1e-12)


def test_vtrace_validation(oracle):
    # test_offpolicy.cpp:186-196: NaN -> NumericError (3), rho < c -> ConfigError (2)
    st, _ = oracle.vtrace([np.nan], [0.0], 0.0, [-1.0], [-1.0], [0])
    assert st == 3
    st, _ = oracle.vtrace([0.0], [0.0], 0.0, [-1.0], [-1.0], [0], 0.5, 1.0, 0.99)
    assert st == 2
    st, _ = oracle.vtrace([0.0], [0.0], 0.0, [-1.0], [-1.0], [0], 1.0, 1.0, 0.0)
    assert st == 2


def test_gae_lambda1_equals_nstep_minus_value(oracle):
    g = golden("vtrace_c1")
    for i in range(16):
        adv, ret = oracle.gae(g["rewards"][i], g["values"][i], g["bootstrap"][i], g["dones"][i],
                              0.99, 1.0)
        np.testing.assert_allclose(adv, g["nstep"][i] - g["values"][i], atol=1e-12)


def test_ppo_and_loss(oracle):
    g = golden("ppo")
    lo, hi = 1 / 1.1, 1.1
    obj = np.array([oracle.L.orc_ppo_objective(r, a, lo, hi) for r, a in zip(g["ratio"], g["adv"])])
    dr = np.array([oracle.L.orc_ppo_dratio(r, a, lo, hi) for r, a in zip(g["ratio"], g["adv"])])
    np.testing.assert_array_equal(obj, g["objective"])
    np.testing.assert_array_equal(dr, g["dratio"])
    st, loss = oracle.total_loss(g["l_ratios"], g["l_adv"], g["l_values"], g["l_vt"], g["l_ent"])
    assert st == 0
    np.testing.assert_allclose(loss, g["loss"], rtol=1e-13, atol=1e-15)


def test_heads(oracle):
    g = golden("heads")
    for i in range(len(g["actions"])):
        np.testing.assert_allclose(oracle.softmax(g["logits"][i]), g["probs"][i], atol=1e-15)
        st, lp, e = oracle.logp_entropy(g["logits"][i], g["actions"][i])
        assert st == 0
        assert abs(lp - g["logp"][i]) < 1e-12 and abs(e - g["entropy"][i]) < 1e-12
    assert oracle.logp_entropy(g["logits"][1], 6)[0] == 1  # ContractError
    # degenerate logits select action 0 with logp ~ 0 (test_policy.cpp:195-203)
    a, lp = oracle.sample(g["logits"][0], 0.999)
    assert a == 0 and abs(lp) < 1e-9


def test_sampler_frequencies_match_reference(oracle):
    # The reference's 10^6-draw frequencies (mt19937_64(14)) and the oracle's
    # counter-based sampler both sit within 3 sigma of the softmax
    # (test_policy.cpp:205-224); the draws differ, the distribution must not.
    g = golden("heads")
    p = oracle.softmax(g["freq_logits"])
    N = 200000
    us = np.array([oracle.L.orc_uniform(1234, i) for i in range(N)])
    acts = np.array([oracle.sample(g["freq_logits"], u)[0] for u in us])
    for counts, n in ((g["freq_counts"], 1000000), (np.bincount(acts, minlength=4), N)):
        sigma = np.sqrt(n * p * (1 - p))
        assert np.all(np.abs(counts - n * p) < 3 * sigma)


def test_adam_matches_reference_sequence(oracle):
    g = golden("adam")
    th = g["theta0"].copy(); m = np.zeros_like(th); v = np.zeros_like(th); t = 0
    for k in range(len(g["grads"])):
        st, t = oracle.adam_step(th, m, v, g["grads"][k].copy(), t)
        assert st == 0
        np.testing.assert_allclose(th, g["thetas"][k], rtol=0, atol=1e-15)
        np.testing.assert_allclose(m, g["ms"][k], rtol=0, atol=1e-15)
        np.testing.assert_allclose(v, g["vs"][k], rtol=0, atol=1e-15)
    # NaN gradient -> NumericError
    st, _ = oracle.adam_step(th, m, v, np.full_like(th, np.nan), t)
    assert st == 3


def test_adam_clip_halving(oracle):
    # test_policy.cpp:399-419: |g| = 8 under clip 4 equals g/2 without clip
    n = 64
    a = np.linspace(-1, 1, n); b = a.copy()
    g = np.zeros(n); g[0] = 8.0
    h = np.zeros(n); h[0] = 4.0
    oracle.adam_step(a, np.zeros(n), np.zeros(n), g, 0, clip=4.0)
    oracle.adam_step(b, np.zeros(n), np.zeros(n), h, 0, clip=0.0)
    np.testing.assert_array_equal(a, b)


def test_layout_matches_reference(oracle):
    g = golden("layout")
    for s, off in zip(g["shapes"], g["offsets"]):
        got = oracle.slot_offsets(int(s[0]), int(s[1]), int(s[2]), int(s[3]), elems=(8, 8, 8, 8))
        assert got == [int(x) for x in off]


def test_device_layout_v2_at_doom_shape(oracle):
    # u8 obs + f32 hidden/reward/logp slot = 980,704 B
    offs = oracle.slot_offsets(32, 3 * 72 * 128, 512, 1)
    assert offs == [64, 884800, 950336, 950464, 950592, 950720, 950752, 951008, 978656, 980704]


def test_live_reference_agrees(oracle, reference):
    rs = np.random.default_rng(5)
    for T in (1, 7, 32):
        x = dict(rewards=rs.uniform(-1, 1, T), values=rs.uniform(-1, 1, T),
                 tlogp=rs.uniform(-2.5, -0.1, T), blogp=rs.uniform(-2.5, -0.1, T),
                 dones=(rs.uniform(size=T) < 0.2).astype(np.uint8))
        a = oracle.vtrace(x["rewards"], x["values"], 0.3, x["tlogp"], x["blogp"], x["dones"],
                          1.5, 1.2, 0.97)
        b = reference.vtrace(x["rewards"], x["values"], 0.3, x["tlogp"], x["blogp"], x["dones"],
                             1.5, 1.2, 0.97)
        assert a[0] == b[0] == 0
        for u, w in zip(a[1], b[1]):
            np.testing.assert_array_equal(u, w)
    assert reference.vtrace([np.nan], [0.0], 0.0, [-1.0], [-1.0], [0])[0] == 3
    assert oracle.slot_offsets(32, 27648, 512, 1, (8, 8, 8, 8)) == \
        reference.slot_offsets(32, 27648, 512, 1)
    assert oracle.L.orc_derive_seed(7, 99) == reference.L.ref_derive_seed(7, 99)
