"""Device slot queues (ready queue + free list) and the queue-fed learner step:
assemble_minibatch semantics (trajstore.hpp:293-331) -- strict FIFO arrival
order, a pop blocks until the producer (another stream) publishes, shutdown /
timeout consumes nothing -- and slot release after the step
(orchestrator.hpp:870)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2006_11751_b200 as appo  # noqa: E402

from test_model_gpu import fill_store  # noqa: E402


def ids(*v):
    return torch.tensor(v, dtype=torch.int32, device="cuda:0")


def test_fifo_order_and_stats():
    ctx = appo.Context(0)
    q = appo.SlotQueue(0, n_slots=16, capacity=8)
    q.push_range(ctx, 0, 5)
    q.push(ctx, ids(9, 7, 8))
    a = q.pop(ctx, 4)
    b = q.pop(ctx, 4)
    ctx.sync()
    assert a.tolist() == [0, 1, 2, 3] and b.tolist() == [4, 9, 7, 8]
    # wrap around the 16-entry ring several times
    seen = []
    for r in range(10):
        q.push(ctx, ids(*[(3 * r + i) % 16 for i in range(6)]))
        seen += q.pop(ctx, 6).tolist() if r % 2 else []
        if r % 2 == 0:
            seen += q.pop(ctx, 3).tolist() + q.pop(ctx, 3).tolist()
    ctx.sync()
    assert seen == [(3 * r + i) % 16 for r in range(10) for i in range(6)]
    st = q.stats()
    assert st["pushed"] == st["popped"] == 68 and st["timeouts"] == 0 and st["size"] == 0


def test_pop_waits_for_producer_on_another_stream():
    s_cons, s_prod = torch.cuda.Stream(0), torch.cuda.Stream(0)
    cons = appo.Context(0, stream=s_cons)
    prod = appo.Context(0, stream=s_prod)
    q = appo.SlotQueue(0, n_slots=64, timeout_s=10.0)
    # a producer's kernels must be loaded before a consumer spins on them (CUDA
    # lazy loading); the library preloads its own, torch's sleep kernel we warm
    torch.cuda._sleep(10)
    ids(0)
    torch.cuda.synchronize()
    out = q.pop(cons, 40)          # enqueued first: spins on the device
    with torch.cuda.stream(s_prod):
        torch.cuda._sleep(2_000_000)  # ~1 ms before the producer publishes
    q.push_range(prod, 10, 25)
    q.push(prod, ids(*range(63, 48, -1)))
    cons.sync()
    prod.sync()
    assert out.tolist() == list(range(10, 35)) + list(range(63, 48, -1))
    assert q.stats()["timeouts"] == 0


def test_timeout_consumes_nothing():
    ctx = appo.Context(0)
    q = appo.SlotQueue(0, n_slots=8, timeout_s=0.02)
    q.push_range(ctx, 0, 2)
    q.pop(ctx, 3)
    with pytest.raises(appo.ResourceError):
        ctx.sync()
    st = q.stats()
    assert st["timeouts"] == 1 and st["popped"] == 0 and st["size"] == 2
    q.push_range(ctx, 5, 1)
    got = q.pop(ctx, 3)
    ctx.sync()
    assert got.tolist() == [0, 1, 5]


def test_foreign_id_is_contract_error():
    ctx = appo.Context(0)
    q = appo.SlotQueue(0, n_slots=4)
    q.push(ctx, ids(1, 9))
    got = q.pop(ctx, 2)
    with pytest.raises(appo.ContractError):
        ctx.sync()
    assert got.tolist() == [1, 0]  # clamped: never addresses outside the region
    with pytest.raises(appo.ContractError):
        q.push_range(ctx, 3, 2)  # host-checked range


def test_queued_learner_step_matches_host_ids():
    desc = appo.ModelDesc(3, 72, 128, 6, 32)
    store = appo.TrajectoryStore(desc, 6)
    fill_store(store, 6, np.random.default_rng(5), 6)
    hp = appo.HParams.defaults(lr=3e-4)
    a = appo.Context(0, seed=17, model=desc)
    b = appo.Context(0, seed=17, model=desc)
    rq = appo.SlotQueue(0, n_slots=6, capacity=16)  # slots 0, 2, 5 are queued twice
    fq = appo.SlotQueue(0, n_slots=6, capacity=16)
    order = [[2, 0, 5], [1, 4, 3], [0, 2, 5]]
    rq.push(b, ids(*order[0], *order[1]))
    rq.push(b, ids(*order[2]))
    for o in order:
        oa = a.learner_step(store.region, store.slot_bytes, o, hp)
        b.learner_submit_queued(store.region, store.slot_bytes, rq, fq, 3, hp)
        ob = b.learner_collect()
        for k in ("total_loss", "policy_loss", "value_loss", "lag_mean", "lag_max", "version"):
            assert oa[k] == ob[k], k
    assert np.array_equal(a.get_params()[0], b.get_params()[0])
    freed = fq.pop(b, 9)
    b.sync()
    assert freed.tolist() == sum(order, [])


def test_queued_learner_step_timeout_is_rejected():
    desc = appo.ModelDesc(3, 72, 128, 6, 32)
    store = appo.TrajectoryStore(desc, 4)
    fill_store(store, 4, np.random.default_rng(6), 6)
    ctx = appo.Context(0, seed=3, model=desc)
    th0, v0 = ctx.get_params()
    rq = appo.SlotQueue(0, n_slots=4, timeout_s=0.02)
    fq = appo.SlotQueue(0, n_slots=4)
    rq.push_range(ctx, 0, 1)
    ctx.learner_submit_queued(store.region, store.slot_bytes, rq, fq, 2)
    with pytest.raises(appo.ResourceError):
        ctx.learner_collect()
    th1, v1 = ctx.get_params()
    assert v1 == v0 and np.array_equal(th0, th1)
    st = rq.stats()
    assert st["size"] == 1 and st["timeouts"] == 1 and fq.stats()["pushed"] == 0
    # the producer catches up: the next step runs on slots [0, 1] in order
    rq.push_range(ctx, 1, 1)
    ctx.learner_submit_queued(store.region, store.slot_bytes, rq, fq, 2)
    assert ctx.learner_collect()["version"] == v0 + 1
    got = fq.pop(ctx, 2)
    ctx.sync()
    assert got.tolist() == [0, 1]


def test_sampler_feeds_ready_queue():
    desc = appo.ModelDesc(3, 72, 128, 6, 32)
    lctx = appo.Context(0, seed=5, model=desc, stream=torch.cuda.Stream(0))
    sctx = lctx.shared(torch.cuda.Stream(0))
    n = 16
    store = appo.TrajectoryStore(desc, 2 * n)
    rq = appo.SlotQueue(0, n_slots=2 * n, timeout_s=10.0)
    fq = appo.SlotQueue(0, n_slots=2 * n)
    smp = appo.Sampler(sctx, n, episode_len=7, seed=3)
    smp.set_ready_queue(rq)
    # first rollout: slots [0, n) (its first steps allocate scratch, which may
    # synchronise the device, so nothing spins on the device yet)
    for t in range(desc.T):
        smp.step(store, 0, t)
    sctx.sync()
    # four learner steps: two over the first rollout, two that are submitted
    # before the second rollout exists and wait for it on the device
    for _ in range(4):
        lctx.learner_submit_queued(store.region, store.slot_bytes, rq, fq, n // 2)
    for t in range(desc.T):
        smp.step(store, n, t)
    out = lctx.learner_collect()
    sctx.sync()
    assert out["version"] == 4 and np.isfinite(out["total_loss"])
    assert rq.stats()["timeouts"] == 0
    freed = fq.pop(lctx, 2 * n)
    lctx.sync()
    assert freed.tolist() == list(range(2 * n))
