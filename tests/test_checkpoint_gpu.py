"""Checkpoint / resume through the C ABI (save_checkpoint / load_checkpoint,
policy.hpp:545-605): exact round trip of parameters, Adam moments, step counter and
version; training resumed from a checkpoint is bit-identical to uninterrupted training."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2006_11751_b200 as appo  # noqa: E402

from test_model_gpu import fill_store  # noqa: E402


def test_checkpoint_roundtrip_and_resume(tmp_path):
    desc = appo.ModelDesc(3, 72, 128, 6, 32)
    a = appo.Context(0, seed=21, model=desc)
    store = appo.TrajectoryStore(desc, 4)
    fill_store(store, 4, np.random.default_rng(4), 6)
    hp = appo.HParams.defaults(lr=3e-4)
    for _ in range(3):
        a.learner_step(store.region, store.slot_bytes, [0, 1, 2, 3], hp)
    path = str(tmp_path / "a.ckpt")
    a.save_checkpoint(path)
    th, ver = a.get_params()
    m, v, t = a.get_adam()
    ck = appo.checkpoint_read(path)
    assert ck["version"] == ver == 3 and ck["adam_t"] == t == 3 and ck["n"] == th.size
    assert ck["spec_hash"] == appo.model_spec_hash(desc)
    np.testing.assert_array_equal(ck["theta"], th.astype(np.float64))
    np.testing.assert_array_equal(ck["m"], m.astype(np.float64))
    np.testing.assert_array_equal(ck["v"], v.astype(np.float64))
    # resume in a fresh context (different init seed): identical state ...
    b = appo.Context(0, seed=99, model=desc)
    b.load_checkpoint(path)
    th2, ver2 = b.get_params()
    m2, v2, t2 = b.get_adam()
    assert ver2 == ver and t2 == t
    assert np.array_equal(th2, th) and np.array_equal(m2, m) and np.array_equal(v2, v)
    # ... and identical training from there on
    for _ in range(2):
        oa = a.learner_step(store.region, store.slot_bytes, [0, 1, 2, 3], hp)
        ob = b.learner_step(store.region, store.slot_bytes, [0, 1, 2, 3], hp)
        assert oa["total_loss"] == ob["total_loss"] and oa["version"] == ob["version"]
    assert np.array_equal(a.get_params()[0], b.get_params()[0])


def test_checkpoint_shape_mismatch_is_config_error(tmp_path):
    a = appo.Context(0, seed=1, model=appo.ModelDesc(3, 72, 128, 6, 32))
    path = str(tmp_path / "a.ckpt")
    a.save_checkpoint(path)
    b = appo.Context(0, seed=1, model=appo.ModelDesc(3, 72, 128, 5, 8))
    with pytest.raises(appo.ConfigError):
        b.load_checkpoint(path)
