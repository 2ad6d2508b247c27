"""The dedicated convolution kernels (csrc/conv1.cu, conv2.cu) at model shapes
other than the Doom 3x72x128 the bench runs: observation width 64 (s2d width
16: padding columns in every tile), 1, 2 and 4 channels (conv1 templated on C;
C = 4 takes the engine path for the conv1 weight gradient), heights whose last
tile is partial, and T in {8, 16} (bootstrap observations not 16-byte aligned
at T = 8 -> the engine fallbacks).  Policy forward and the full learner
gradient against the fp64 oracle with the tolerances of test_model_gpu.py."""
import numpy as np
import pytest
import torch

import paper_2006_11751_b200 as appo
from test_model_gpu import (GNORM_TOL, GRAD_TOL, H_TOL, LOGPI_TOL, LOSS_ATOL, LOSS_RTOL,
                            block_offsets, fill_store, log_softmax, rel_l2)

pytestmark = pytest.mark.gpu

# the last shape has 12 actions: above the fused GRU step's 7, so inference
# takes the unfused gate GEMMs + gru_infer_kernel
SHAPES = [(1, 40, 64, 4, 8), (2, 48, 64, 3, 16), (4, 72, 128, 5, 16), (3, 56, 128, 6, 8),
          (3, 72, 128, 12, 8)]


@pytest.mark.parametrize("shape", SHAPES)
def test_policy_forward_other_shapes(oracle, shape):
    C_, H, W, A, T = shape
    ctx = appo.Context(0, seed=3, model=appo.ModelDesc(C_, H, W, A, T))
    rs = np.random.default_rng(C_ * 100 + H)
    B = 40
    obs = rs.integers(0, 256, (B, C_ * H * W), dtype=np.uint8)
    h = rs.normal(scale=0.5, size=(B, 512)).astype(np.float32)
    th, _ = ctx.get_params()
    ctx.set_timing(True)
    out = ctx.policy_forward(torch.from_numpy(obs).cuda(), torch.from_numpy(h).cuda(),
                             rng_counter0=5, want_logits=True)
    torch.cuda.synchronize()
    launched = {r["name"] for r in ctx.timing_report()}
    ctx.set_timing(False)
    # the dedicated kernels ran (not an engine fallback)
    gru = "gru_infer_fused_tcgen05" if A <= 7 else "gru_infer_kernel"
    assert {"conv1_s2d_tcgen05", "conv2_s2d_tcgen05", gru} <= launched, launched
    ref = oracle.policy_forward((C_, H, W, A), th.astype(np.float64), obs, h.astype(np.float64))
    lg = out["logits"].cpu().numpy().astype(np.float64)
    assert np.abs(log_softmax(lg) - log_softmax(ref["logits"])).max() <= LOGPI_TOL
    vals = out["values"].cpu().numpy()
    assert np.all(np.abs(vals - ref["values"]) <= 2e-4 + 2e-3 * np.abs(ref["values"]))
    assert np.abs(out["h_out"].cpu().numpy() - ref["h_out"]).max() <= H_TOL


@pytest.mark.parametrize("shape", SHAPES)
def test_learner_step_other_shapes(oracle, shape):
    C_, H, W, A, T = shape
    desc = appo.ModelDesc(C_, H, W, A, T)
    ctx = appo.Context(0, seed=7, model=desc)
    store = appo.TrajectoryStore(desc, 4)
    rs = np.random.default_rng(W + T)
    d = fill_store(store, 3, rs, A)
    th0, _ = ctx.get_params()
    hp = appo.HParams.defaults(gamma=0.99, gae_lambda=0.95)
    out = ctx.learner_step(store.region, store.slot_bytes, [1, 0, 2], hp)
    g = ctx.grad()
    order = [1, 0, 2]
    sel = {k: v[order] for k, v in d.items()}
    ref = oracle.learner_step((C_, H, W, A), th0.astype(np.float64), np.zeros(th0.size),
                              np.zeros(th0.size), 0, sel["obs"], sel["h0"].astype(np.float64),
                              sel["actions"].reshape(-1),
                              sel["blogp"].reshape(-1).astype(np.float64),
                              sel["rewards"].reshape(-1).astype(np.float64),
                              sel["dones"].reshape(-1), hp=dict(gamma=0.99, gae_lambda=0.95),
                              do_adam=False)
    assert ref["status"] == 0
    st = ref["stats"]
    for got, exp in ((out["policy_loss"], st[0]), (out["value_loss"], st[1]),
                     (out["entropy"], st[2]), (out["total_loss"], st[3])):
        assert abs(got - exp) <= LOSS_RTOL * abs(exp) + LOSS_ATOL, (got, exp)
    gr = ref["grad"]
    assert abs(out["grad_norm"] - np.linalg.norm(gr)) <= GNORM_TOL * np.linalg.norm(gr)
    for name, (a, b) in block_offsets(ctx).items():
        e = rel_l2(g[a:b].astype(np.float64), gr[a:b])
        assert e <= GRAD_TOL, (name, e)


def test_doom_learner_runs_the_dedicated_kernels():
    """At the bench shape every convolution of the learner step except conv3's
    runs in the space-to-depth kernels (no silent engine fallback), and the
    loss block runs fused per trajectory (traj_loss.cu)."""
    desc = appo.ModelDesc.doom(T=32)
    ctx = appo.Context(0, seed=2, model=desc)
    store = appo.TrajectoryStore(desc, 4)
    fill_store(store, 4, np.random.default_rng(5), 6)
    ctx.set_timing(True)
    ctx.learner_step(store.region, store.slot_bytes, [0, 1, 2, 3], appo.HParams.defaults())
    torch.cuda.synchronize()
    # weight-gradient kernels on the learner side stream time as "<class>@side"
    launched = {r["name"].split("@")[0] for r in ctx.timing_report()}
    ctx.set_timing(False)
    assert {"conv1_s2d_tcgen05", "conv1_s2d_wgrad_tcgen05", "conv2_s2d_tcgen05",
            "conv2_dgrad_s2d_tcgen05", "conv2_wgrad_s2d_tcgen05", "gru_seq_fwd_kernel",
            "gru_seq_bwd_kernel", "traj_loss_kernel"} <= launched, launched
    # the fused loss block replaces the four unfused launches
    assert not {"heads_fwd_kernel", "ppo_loss_kernel", "heads_bwd_fused_kernel"} & launched
