"""Multi-process (gloo, world_size 2, CPU) checks of the data-parallel learner's
host logic, with the fp64 oracle standing in for the device gradient:

  * parity mode: two ranks each take half of the trajectories and average
    their per-shard gradients bucket by bucket in the order the product
    library plans them (appo_dp_bucket_plan, host code of libappo_b200.so --
    what appo_learner_step does with ncclAllReduce(avg) on its side stream
    before clip + Adam), together with the max-reduction of the rejection
    flags, then apply the same Adam step; both replicas must end bit-identical
    and equal to the single-process full-batch step (the reference's 1/B mean,
    policy.hpp:318, makes the average of equal shard means the full mean);
  * a step rejected on one rank is rejected on both (flag consensus);
  * the NCCL unique-id broadcast helper used by paper_2006_11751_b200.dp_init;
  * bench.py's max-over-ranks timing reduction.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

SHAPE = (3, 36, 36, 6)
N_TRAJ, T = 4, 4


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def make_batch():
    from oracle.oracle import Oracle
    orc = Oracle()
    C, H, W, A = SHAPE
    rs = np.random.default_rng(7)
    obs = rs.integers(0, 256, (N_TRAJ, T + 1, C * H * W), dtype=np.uint8)
    h0 = rs.normal(scale=0.3, size=(N_TRAJ, 512))
    act = rs.integers(0, A, N_TRAJ * T).astype(np.int32)
    blogp = rs.uniform(-2.2, -1.5, N_TRAJ * T)
    rew = rs.uniform(-1, 1, N_TRAJ * T)
    dn = (rs.uniform(size=N_TRAJ * T) < 0.2).astype(np.uint8)
    theta = orc.init_params(*SHAPE, 3)
    return orc, theta, obs, h0, act, blogp, rew, dn


def shard_grad(orc, theta, obs, h0, act, blogp, rew, dn, lo, hi):
    sl = slice(lo * T, hi * T)
    r = orc.learner_step(SHAPE, theta.copy(), np.zeros_like(theta), np.zeros_like(theta), 0,
                         obs[lo:hi], h0[lo:hi], act[sl], blogp[sl], rew[sl], dn[sl],
                         do_adam=False)
    assert r["status"] == 0
    return r["grad"]


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc, theta, obs, h0, act, blogp, rew, dn = make_batch()
        per = N_TRAJ // world
        g = shard_grad(orc, theta, obs, h0, act, blogp, rew, dn, rank * per, (rank + 1) * per)
        import paper_2006_11751_b200 as appo
        plan = appo.dp_bucket_plan(appo.ModelDesc(*SHAPE, T))
        gt = torch.from_numpy(g)
        for off, n in plan:  # reverse layer order, as the learner launches them
            b = gt[off:off + n]
            dist.all_reduce(b, op=dist.ReduceOp.SUM)
            b /= world
        # rejection consensus: rank 1 flags a contract error on its shard
        flags = torch.tensor([0, 1 if rank == 1 else 0, 0, 0], dtype=torch.int32)
        dist.all_reduce(flags, op=dist.ReduceOp.MAX)
        assert flags.tolist() == [0, 1, 0, 0]
        th = theta.copy()
        m = np.zeros_like(th)
        v = np.zeros_like(th)
        st, _ = orc.adam_step(th, m, v, gt.numpy().copy(), 0)
        assert st == 0
        # unique-id broadcast as in dp_init (rank 0's 128-byte id reaches all)
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        # max-over-ranks timing as in bench.py
        t = torch.tensor([10.0 + rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, th, gt.numpy(), obj[0], t.item()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_dp_two_ranks_match_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, th0, g0, id0, t0), (_, th1, g1, id1, t1) = res
    assert np.array_equal(th0, th1) and np.array_equal(g0, g1)  # replicas in lockstep
    assert id0 == id1 == bytes(range(128))
    assert t0 == t1 == 11.0
    orc, theta, obs, h0, act, blogp, rew, dn = make_batch()
    g_full = shard_grad(orc, theta, obs, h0, act, blogp, rew, dn, 0, N_TRAJ)
    assert np.abs(g0 - g_full).max() <= 1e-12 * np.abs(g_full).max()
    th = theta.copy()
    orc.adam_step(th, np.zeros_like(th), np.zeros_like(th), g_full, 0)
    assert np.abs(th0 - th).max() <= 1e-12
