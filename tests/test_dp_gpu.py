"""The data-parallel learner path on the device at nranks = 1 (gpurun has one
GPU): appo_dp_init over a one-rank NCCL communicator engages the whole
bucketed path -- three ncclAllReduce(avg) buckets on the side stream in
reverse layer order (appo_dp_bucket_plan), the grouped max-reduction of the
rejection flags, the learner stream joining before clip + Adam.  Averaging
over one rank is the identity, so the result must be bit-identical to the
plain learner, and a step the rank rejects must stay rejected after the flag
consensus."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2006_11751_b200 as appo  # noqa: E402

from test_model_gpu import fill_store  # noqa: E402


def test_bucket_plan_covers_parameters_in_reverse_layer_order():
    desc = appo.ModelDesc.doom(T=32)
    plan = appo.dp_bucket_plan(desc)
    P = appo.param_count(desc)
    assert sorted((o, o + n) for o, n in plan)[0][0] == 0
    covered = np.zeros(P, np.int32)
    for o, n in plan:
        covered[o:o + n] += 1
    assert np.all(covered == 1)
    assert [o for o, _ in plan] == sorted([o for o, _ in plan], reverse=True)


def test_dp_one_rank_is_bitwise_the_plain_learner():
    desc = appo.ModelDesc.doom(T=32)
    store = appo.TrajectoryStore(desc, 6)
    fill_store(store, 6, np.random.default_rng(3), 6)
    hp = appo.HParams.defaults(lr=3e-4)
    ref = appo.Context(0, seed=23, model=desc)
    dp = appo.Context(0, seed=23, model=desc)
    appo.dp_init(dp, None, 0, 1)
    for ids in ([0, 1, 2], [3, 4, 5], [5, 0, 2, 1]):
        a = ref.learner_step(store.region, store.slot_bytes, ids, hp)
        b = dp.learner_step(store.region, store.slot_bytes, ids, hp)
        assert a["total_loss"] == b["total_loss"] and a["grad_norm"] == b["grad_norm"]
        assert a["version"] == b["version"]
    assert np.array_equal(ref.get_params()[0], dp.get_params()[0])
    assert np.array_equal(ref.grad(), dp.grad())


def test_dp_rejected_step_stays_rejected_after_flag_consensus():
    desc = appo.ModelDesc.doom(T=32)
    store = appo.TrajectoryStore(desc, 3)
    fill_store(store, 3, np.random.default_rng(4), 6)
    dp = appo.Context(0, seed=29, model=desc)
    appo.dp_init(dp, None, 0, 1)
    dp.learner_step(store.region, store.slot_bytes, [0, 1])
    th0, v0 = dp.get_params()
    store.actions(2)[5] = 17  # out of range: ContractError on this rank
    with pytest.raises(appo.ContractError):
        dp.learner_step(store.region, store.slot_bytes, [2, 0])
    th1, v1 = dp.get_params()
    assert v1 == v0 and np.array_equal(th0, th1)
    store.actions(2)[5] = 1  # the next step is accepted again
    out = dp.learner_step(store.region, store.slot_bytes, [2, 0])
    assert out["version"] == v0 + 1


def test_dp_learner_overlaps_a_running_sampler():
    # the bench configuration: sampler on a shared context, DP learner on the
    # base context, both streams busy; the learner's averaged steps still
    # match a plain learner bit for bit on the same slots
    desc = appo.ModelDesc.doom(T=32)
    n = 64
    store = appo.TrajectoryStore(desc, 2 * n)
    base = appo.Context(0, seed=31, model=desc)
    smp_ctx = base.shared(stream=torch.cuda.Stream())
    smp = appo.Sampler(smp_ctx, n, episode_len=40, seed=3)
    for t in range(desc.T):
        smp.step(store, 0, t)
    smp_ctx.sync()
    plain = appo.Context(0, seed=31, model=desc)
    appo.dp_init(base, None, 0, 1)
    for t in range(desc.T):  # keep the sampler busy on the second half of the region
        smp.step(store, n, t)
    a = base.learner_step(store.region, store.slot_bytes, list(range(16)))
    b = plain.learner_step(store.region, store.slot_bytes, list(range(16)))
    smp_ctx.sync()
    assert a["total_loss"] == b["total_loss"]
    assert np.array_equal(base.get_params()[0], plain.get_params()[0])
