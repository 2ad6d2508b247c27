"""Cross-process PBT exchange (configs[4]: one policy learner per process):
copy_weights(dst, src) between two processes through appo_params_export /
appo_params_import (CUDA IPC handles shipped over torch.distributed, then a
device-to-device copy; across GPUs the same call is an NVLink peer copy).
gpurun has one GPU, so both processes share device 0.  Every rank runs the
same PBT controller on the all-gathered scores and reaches the same
(dst, src) decisions, as the reference's single controller does
(runner.hpp:209-227)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, port, q):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist
    import paper_2006_11751_b200 as appo
    from test_model_gpu import fill_store
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        desc = appo.ModelDesc.doom(T=32)
        ctx = appo.Context(0, seed=100 + rank, model=desc)
        store = appo.TrajectoryStore(desc, 2)
        fill_store(store, 2, np.random.default_rng(rank), 6)
        for _ in range(1 + rank):  # different Adam step counts / versions
            ctx.learner_step(store.region, store.slot_bytes, [0, 1],
                             appo.HParams.defaults(lr=1e-3))
        th, ver = ctx.get_params()
        m, v, t = ctx.get_adam()
        states = [None, None]
        dist.all_gather_object(states, (th, m, v, t, ver))
        # the controller on both ranks: policy 0 has the better score, so the
        # exchange copies 0 -> 1 (P = 2, replace 50 %: n_replace = floor(1.0) =
        # 1, n_top = 1, population.hpp:151-152; the default 30 % floors to 0)
        cfg = appo.PbtConfig.defaults(replace_fraction=0.5)
        calls = []
        pbt = appo.PbtController(cfg, 2, 7, copy_weights=lambda d, s: calls.append((d, s)))
        pbt.step([1.0, 0.0], 0)
        assert calls == [(1, 0)]
        appo.pbt_exchange(ctx, dist, rank, *calls[0])
        th2, ver2 = ctx.get_params()
        m2, v2, t2 = ctx.get_adam()
        # the copied weights are what inference uses right away
        obs = torch.from_numpy(np.random.default_rng(5).integers(
            0, 256, (8, desc.obs_dim), dtype=np.uint8)).cuda()
        h = torch.zeros(8, 512, device="cuda")
        lg = ctx.policy_forward(obs, h, want_logits=True)["logits"].cpu().numpy()
        outs = [None, None]
        dist.all_gather_object(outs, (obs.cpu().numpy(), lg))
        q.put((rank, states, th2, m2, v2, t2, ver2, outs))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_pbt_exchange_between_processes():
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    r0, r1 = res
    states = r0[1]
    th_src, m_src, v_src, t_src, ver_src = states[0]
    _, _, _, _, ver_dst = states[1]
    # rank 1 (dst) now holds rank 0's theta / m / v / t, published as its next version
    _, _, th, m, v, t, ver, outs = r1
    assert np.array_equal(th, th_src) and np.array_equal(m, m_src) and np.array_equal(v, v_src)
    assert t == t_src == 1 and ver == ver_dst + 1
    # the source is untouched
    assert np.array_equal(r0[2], th_src) and r0[6] == ver_src
    # both processes' inference now computes the same logits on the same obs
    (o0, l0), (o1, l1) = outs
    assert np.array_equal(o0, o1) and np.array_equal(l0, l1)
