"""PBT weight exchange on the device: appo_params_copy (PbtController's
copy_weights, runner.hpp:211-219: theta + Adam state copied, published as the
destination's next version) and the controller driving it over learner
contexts."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2006_11751_b200 as appo  # noqa: E402

from test_model_gpu import fill_store  # noqa: E402

DESC = appo.ModelDesc(3, 72, 128, 6, 32)


@pytest.fixture(scope="module")
def store():
    s = appo.TrajectoryStore(DESC, 4)
    fill_store(s, 4, np.random.default_rng(8), 6)
    return s


def test_params_copy_state_inference_and_training(store):
    hp = appo.HParams.defaults(lr=3e-4)
    a = appo.Context(0, seed=1, model=DESC)
    b = appo.Context(0, seed=2, model=DESC)
    for _ in range(2):
        a.learner_step(store.region, store.slot_bytes, [0, 1, 2, 3], hp)
    vb = b.version
    appo.params_copy(b, a)
    assert b.version == vb + 1
    assert np.array_equal(b.get_params()[0], a.get_params()[0])
    ma, va, ta = a.get_adam()
    mb, vb_, tb = b.get_adam()
    assert ta == tb and np.array_equal(ma, mb) and np.array_equal(va, vb_)
    # inference on b now uses the copied weights (its newest publish)
    rs = np.random.default_rng(1)
    obs = torch.from_numpy(rs.integers(0, 256, (8, DESC.obs_dim), dtype=np.uint8)).cuda()
    h = torch.from_numpy(rs.normal(size=(8, 512)).astype(np.float32)).cuda()
    oa = a.policy_forward(obs, h, want_logits=True)
    ob = b.policy_forward(obs, h, want_logits=True)
    torch.cuda.synchronize()
    assert torch.equal(oa["logits"], ob["logits"]) and ob["version"] == b.version
    # and training continues identically from the copied state
    for _ in range(2):
        la = a.learner_step(store.region, store.slot_bytes, [3, 1], hp)["total_loss"]
        lb = b.learner_step(store.region, store.slot_bytes, [3, 1], hp)["total_loss"]
        assert la == lb
    assert np.array_equal(a.get_params()[0], b.get_params()[0])


def test_params_copy_contract_checks(store):
    a = appo.Context(0, seed=1, model=DESC)
    b = appo.Context(0, seed=2, model=DESC)
    c = appo.Context(0, seed=3, model=appo.ModelDesc(3, 72, 128, 5, 8))
    with pytest.raises(appo.ConfigError):
        appo.params_copy(c, a)
    b.learner_submit(store.region, store.slot_bytes, [0, 1])
    with pytest.raises(appo.ContractError):
        appo.params_copy(b, a)  # destination has an uncollected step
    b.learner_collect()
    appo.params_copy(b, a)


def test_controller_exchanges_weights_between_learners():
    P = 4
    learners = [appo.Context(0, seed=10 + i, model=DESC) for i in range(P)]
    before = [l.get_params()[0] for l in learners]
    cfg = appo.PbtConfig.defaults(replace_fraction=0.5, mutate_fraction=0.5)
    pbt = appo.PbtController(cfg, P, 42, copy_weights=learners)
    ev = pbt.step([0.9, 0.1, 0.5, 0.0], frame=5_000_000)
    ex = [(e.agent, int(e.old_value)) for e in ev if e.as_tuple()[2] == "exchange"]
    # worst floor(0.5 * 4) = 2 (policies 1 and 3) take weights from the top 2 (0 and 2)
    assert sorted(d for d, _ in ex) == [1, 3] and all(s in (0, 2) for _, s in ex)
    for d, s in ex:
        assert np.array_equal(learners[d].get_params()[0], before[s])
        assert pbt.agent(d).learning_rate == pbt.agent(s).learning_rate
    for i in (0, 2):
        assert np.array_equal(learners[i].get_params()[0], before[i])
