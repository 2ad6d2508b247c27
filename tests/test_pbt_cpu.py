"""PBT controller (population.hpp:131-186, runner.hpp:169-252) against the
reference compiled here (oracle/_ref: its own pbt_step over the same schedule)
and against the decision-log hash the reference freezes in its acceptance
suite (acceptance.cpp:573-662, kExpectedLogHash)."""
import pytest

import paper_2006_11751_b200 as appo

FROZEN_LOG_HASH = 0x6725D10D928ABD62  # acceptance.cpp:655


def synthetic_scores(P, period):
    # acceptance.cpp:589-594: every third period compresses the spread below 0.35
    out = []
    for i in range(P):
        base = ((i * 13 + period * 7) % 23) / 23.0
        out.append(0.5 + 0.2 * base if period % 3 == 2 else base)
    return out


def run_ours(P, seed, periods, threshold, copy=None):
    cfg = appo.PbtConfig.defaults(exchange_threshold=threshold)
    init = [appo.AgentMeta.make(reward_weights=(1.0, 0.2, -0.5)) for _ in range(P)]
    pbt = appo.PbtController(cfg, P, seed, init=init, copy_weights=copy)
    events = []
    for period in range(periods):
        events += pbt.step(synthetic_scores(P, period), period * 5_000_000)
    return pbt, events


def ref_log(reference, P, seed, periods, threshold):
    import ctypes as C
    L = reference.L
    L.ref_pbt_log.restype = C.c_long
    L.ref_pbt_log.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_double, C.c_char_p, C.c_size_t]
    buf = C.create_string_buffer(1 << 20)
    n = L.ref_pbt_log(P, seed, periods, -1.0 if threshold is None else threshold, buf, 1 << 20)
    assert n > 0
    return buf.value.decode()


def test_decision_log_matches_frozen_reference_hash(reference):
    lineage = list(range(8))

    def copy(dst, src):
        lineage[dst] = lineage[src]

    pbt, events = run_ours(8, 808, 100, 0.35, copy)
    text = appo.PbtController.format_events(events)
    assert appo.fnv1a64(text.encode()) == FROZEN_LOG_HASH
    assert text == ref_log(reference, 8, 808, 100, 0.35)
    kinds = {e.as_tuple()[2] for e in events}
    assert kinds == {"mutate", "exchange", "skip-threshold"}
    assert len(set(lineage)) < 8  # exchanges happened through the callback
    for i in range(8):
        assert pbt.agent(i).adam_beta1 < 1.0


@pytest.mark.parametrize("P,seed,periods,threshold", [(5, 3, 40, None), (16, 99, 25, 0.1),
                                                      (3, 7, 30, None)])
def test_decision_log_matches_reference(reference, P, seed, periods, threshold):
    _, events = run_ours(P, seed, periods, threshold)
    assert appo.PbtController.format_events(events) == ref_log(reference, P, seed, periods,
                                                               threshold)


def test_exchange_calls_copy_weights_with_event_pairs():
    calls = []
    _, events = run_ours(8, 808, 30, 0.35, lambda d, s: calls.append((d, s)))
    ex = [(e.agent, int(e.old_value)) for e in events if e.as_tuple()[2] == "exchange"]
    assert calls == ex and len(calls) > 0


def test_copy_failure_propagates():
    def boom(d, s):
        raise RuntimeError("peer copy failed")

    with pytest.raises(appo.ContractError):
        run_ours(8, 808, 10, None, boom)


def test_tick_windows_and_period_boundaries():
    cfg = appo.PbtConfig.defaults(pbt_period=1000, window=3)
    pbt = appo.PbtController(cfg, 4, appo.LIB.appo_pbt_controller_seed(1))
    assert pbt.score(0) is None
    for v in (1.0, 2.0, 3.0, 4.0):
        pbt.record(0, v)  # window of 3: mean(2, 3, 4)
    assert pbt.score(0) == 3.0
    pbt.record(7, 1.0)  # foreign policy id: ignored
    assert pbt.tick(999) is None
    ev = pbt.tick(1000)
    assert ev is not None  # boundary reached: a step on the window scores ran
    # only policy 0 has a score; the others are exempt, so nobody is mutated
    # (floor(0.7 * 1) == 0) and nobody replaced
    assert ev == []
    assert pbt.tick(1500) is None and pbt.tick(2000) is not None
    one = appo.PbtController(cfg, 1, 5)
    one.record(0, 1.0)
    assert one.tick(10**9) is None  # a population of one never steps


def test_hparams_and_config_validation():
    cfg = appo.PbtConfig.defaults()
    pbt = appo.PbtController(cfg, 2, 1, init=[appo.AgentMeta.make(learning_rate=3e-4,
                                                                  entropy_coef=0.01,
                                                                  adam_beta1=0.8)] * 2)
    hp = pbt.hparams(1)
    assert abs(hp.lr - 3e-4) < 1e-9 and abs(hp.entropy_coef - 0.01) < 1e-9
    assert abs(hp.beta1 - 0.8) < 1e-7 and pbt.agent(1).policy_id == 1
    with pytest.raises(appo.ConfigError):
        appo.PbtController(appo.PbtConfig.defaults(mutation_factor=1.0), 2, 1)
    with pytest.raises(appo.ConfigError):
        appo.PbtController(appo.PbtConfig.defaults(replace_fraction=1.5), 2, 1)


def test_overlapping_cohorts_self_exchange_is_logged_not_copied():
    # replace_fraction > 0.5: the top cohort overlaps the replaced one, so a
    # policy can draw itself as the source; the reference's copy_weights is
    # then a harmless self-copy and the exchange is still logged
    calls = []

    def copy(d, s):
        assert d != s, "self-copy must not reach copy_weights"
        calls.append((d, s))

    cfg = appo.PbtConfig.defaults(replace_fraction=0.8)
    pbt = appo.PbtController(cfg, 4, 11, copy_weights=copy)
    events = []
    for period in range(60):
        events += pbt.step(synthetic_scores(4, period), period)
    ex = [(e.agent, int(e.old_value)) for e in events if e.as_tuple()[2] == "exchange"]
    assert any(d == s for d, s in ex)
    assert calls == [(d, s) for d, s in ex if d != s] and calls
