"""Second, independent oracle for the parts the reference does not pin
(convnet_simple, GRU-512, BPTT, GAE, u8/255 input): torch fp64 autograd on
CPU (test-only).  Checks the C restatement's forward and its full learner
gradient (policy + value + entropy loss through heads, GRU over the T-step
window with done resets, and the encoder)."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

SHAPE = (3, 36, 36, 6)  # small obs so the fp64 loops run in a second


def unpack(theta, shape):
    C, H, W, A = shape
    H1, W1 = (H - 8) // 4 + 1, (W - 8) // 4 + 1
    H2, W2 = (H1 - 4) // 2 + 1, (W1 - 4) // 2 + 1
    H3, W3 = (H2 - 3) // 2 + 1, (W2 - 3) // 2 + 1
    sizes = [("c1w", (32, C, 8, 8)), ("c1b", (32,)), ("c2w", (64, 4, 4, 32)), ("c2b", (64,)),
             ("c3w", (128, 3, 3, 64)), ("c3b", (128,)), ("fcw", (512, H3 * W3 * 128)),
             ("fcb", (512,)), ("wih", (1536, 512)), ("whh", (1536, 512)), ("bih", (1536,)),
             ("bhh", (1536,)), ("wpi", (A, 512)), ("bpi", (A,)), ("wv", (512,)), ("bv", (1,))]
    out, o = {}, 0
    for k, s in sizes:
        n = int(np.prod(s))
        out[k] = theta[o:o + n].view(*s)
        o += n
    assert o == theta.numel()
    return out, (H3, W3)


def encoder(p, obs, hw3):
    x = obs.double() / 255.0
    x = F.elu(F.conv2d(x, p["c1w"], p["c1b"], stride=4))
    x = F.elu(F.conv2d(x, p["c2w"].permute(0, 3, 1, 2), p["c2b"], stride=2))
    x = F.elu(F.conv2d(x, p["c3w"].permute(0, 3, 1, 2), p["c3b"], stride=2))
    x = x.permute(0, 2, 3, 1).reshape(x.shape[0], -1)  # (h, w, c) flatten
    return F.elu(x @ p["fcw"].T + p["fcb"])


def gru(p, x, h):
    gi = x @ p["wih"].T + p["bih"]
    gh = h @ p["whh"].T + p["bhh"]
    r = torch.sigmoid(gi[:, :512] + gh[:, :512])
    z = torch.sigmoid(gi[:, 512:1024] + gh[:, 512:1024])
    n = torch.tanh(gi[:, 1024:] + r * gh[:, 1024:])
    return (1 - z) * n + z * h


def heads(p, h):
    return h @ p["wpi"].T + p["bpi"], h @ p["wv"] + p["bv"]


@pytest.fixture(scope="module")
def setup(oracle):
    th = oracle.init_params(*SHAPE, 77)
    return th


def test_param_count_doom_shape(oracle):
    # 2,872,551 params at 3x72x128 with 6 actions
    assert oracle.param_count(3, 72, 128, 6) == 2872551


def test_forward_matches_torch(oracle, setup):
    th = setup
    rs = np.random.default_rng(1)
    B = 3
    obs = rs.integers(0, 256, (B, 3, 36, 36), dtype=np.uint8)
    h = rs.normal(scale=0.5, size=(B, 512))
    out = oracle.policy_forward(SHAPE, th, obs, h)
    p, hw3 = unpack(torch.from_numpy(th), SHAPE)
    with torch.no_grad():
        hn = gru(p, encoder(p, torch.from_numpy(obs), hw3), torch.from_numpy(h))
        lg, v = heads(p, hn)
    np.testing.assert_allclose(out["h_out"], hn.numpy(), atol=1e-12)
    np.testing.assert_allclose(out["logits"], lg.numpy(), atol=1e-12)
    np.testing.assert_allclose(out["values"], v.numpy(), atol=1e-12)


def vtrace_np(r, v, boot, tl, bl, d, gamma, rho_bar=1.0, c_bar=1.0):
    T = len(r)
    vs, pg = np.zeros(T), np.zeros(T)
    vn, valn = boot, boot
    for i in range(T - 1, -1, -1):
        ratio = np.exp(np.clip(tl[i] - bl[i], -20, 20))
        rho, c = min(rho_bar, ratio), min(c_bar, ratio)
        disc = 0.0 if d[i] else gamma
        delta = rho * (r[i] + disc * valn - v[i])
        vs[i] = v[i] + delta + disc * c * (vn - valn)
        pg[i] = rho * (r[i] + disc * vn - v[i])
        vn, valn = vs[i], v[i]
    return vs, pg


@pytest.mark.parametrize("adv_source,normalize", [(0, 0), (2, 1)])
def test_learner_gradient_matches_torch_autograd(oracle, setup, adv_source, normalize):
    th0 = setup.copy()
    rs = np.random.default_rng(2)
    n_traj, T = 2, 4
    C, H, W, A = SHAPE
    obs = rs.integers(0, 256, (n_traj, T + 1, C, H, W), dtype=np.uint8)
    h0 = rs.normal(scale=0.3, size=(n_traj, 512))
    actions = rs.integers(0, A, n_traj * T).astype(np.int32)
    blogp = rs.uniform(-2.2, -1.5, n_traj * T)
    rewards = rs.uniform(-1, 1, n_traj * T)
    dones = np.zeros(n_traj * T, dtype=np.uint8)
    dones[1] = 1  # reset inside trajectory 0
    hp = dict(adv_source=adv_source, normalize=normalize, gamma=0.99, gae_lambda=0.95)
    m = np.zeros_like(th0); v = np.zeros_like(th0)
    res = oracle.learner_step(SHAPE, th0.copy(), m, v, 0, obs.reshape(n_traj, T + 1, -1), h0,
                              actions, blogp, rewards, dones, hp=hp, do_adam=False)
    assert res["status"] == 0

    theta = torch.from_numpy(th0.copy()).requires_grad_(True)
    p, hw3 = unpack(theta, SHAPE)
    x = encoder(p, torch.from_numpy(obs.reshape(-1, C, H, W)), hw3).view(n_traj, T + 1, 512)
    h = torch.from_numpy(h0)
    lgs, vals = [], []
    for t in range(T + 1):
        hn = gru(p, x[:, t], h)
        lg, vv = heads(p, hn)
        lgs.append(lg); vals.append(vv)
        if t < T:
            keep = torch.from_numpy(1.0 - dones.reshape(n_traj, T)[:, t].astype(np.float64))
            h = hn * keep[:, None]
    logits = torch.stack(lgs[:T], 1).reshape(-1, A)
    values = torch.stack(vals[:T], 1).reshape(-1)
    boot = vals[T].detach().numpy()
    logp_all = torch.log_softmax(logits, -1)
    act = torch.from_numpy(actions).long()
    tlogp = logp_all.gather(1, act[:, None]).squeeze(1)
    ent = -(logp_all.exp() * logp_all).sum(-1)
    # targets (constants)
    vv = values.detach().numpy().reshape(n_traj, T)
    tl = tlogp.detach().numpy().reshape(n_traj, T)
    vt = np.zeros((n_traj, T)); adv = np.zeros((n_traj, T))
    for i in range(n_traj):
        vt[i], pg = vtrace_np(rewards.reshape(n_traj, T)[i], vv[i], boot[i], tl[i],
                              blogp.reshape(n_traj, T)[i], dones.reshape(n_traj, T)[i], 0.99)
        if adv_source == 0:
            adv[i] = pg
        else:
            a, _ = oracle.gae(rewards.reshape(n_traj, T)[i], vv[i], boot[i],
                              dones.reshape(n_traj, T)[i], 0.99, 0.95)
            adv[i] = a
    adv = adv.reshape(-1)
    if normalize:
        adv = (adv - adv.mean()) / (adv.std() + 1e-8)
    adv_t = torch.from_numpy(adv)
    ratio = torch.exp(torch.clamp(tlogp - torch.from_numpy(blogp), -20, 20))
    surr = torch.minimum(ratio * adv_t, torch.clamp(ratio, 1 / 1.1, 1.1) * adv_t)
    loss = -surr.mean() + 0.5 * ((values - torch.from_numpy(vt.reshape(-1))) ** 2).mean() \
        - 0.003 * ent.mean()
    loss.backward()
    g = theta.grad.numpy()
    np.testing.assert_allclose(res["stats"][3], loss.item(), rtol=1e-10)
    np.testing.assert_allclose(res["v_targets"], vt.reshape(-1), atol=1e-12)
    np.testing.assert_allclose(res["adv"], adv, atol=1e-12)
    scale = np.abs(g).max()
    assert np.abs(res["grad"] - g).max() <= 1e-10 * scale
