"""Byte-exact trajectory dump (SURVEY §8(c) layout check): a layout-v2 slot
exported by TrajectoryStore.to_reference_dump equals, byte for byte, the file
the reference's own dump_trajectory (trajstore.hpp:335-359) writes for a slot
it filled through TrajectorySlotView::write_step / set_bootstrap
(trajstore.hpp:166-215) with the same records (u8 pixels as f64 values)."""
import numpy as np
import pytest

import paper_2006_11751_b200 as appo


def _records(rs, T, od, boot_hidden):
    return dict(obs=rs.integers(0, 256, (T, od), dtype=np.uint8),
                h0=rs.normal(size=512).astype(np.float32),
                actions=rs.integers(0, 6, T).astype(np.int32),
                rewards=rs.uniform(-1, 1, T).astype(np.float32),
                logp=rs.uniform(-3, 0, T).astype(np.float32),
                dones=(rs.uniform(size=T) < 0.2).astype(np.uint8),
                versions=np.sort(rs.integers(0, 50, T)).astype(np.int64),
                boot_obs=rs.integers(0, 256, od, dtype=np.uint8),
                boot_hidden=boot_hidden)


@pytest.mark.parametrize("shape", [(3, 72, 128, 6, 32), (1, 36, 36, 3, 5), (3, 36, 64, 6, 1)])
def test_dump_matches_reference_dump_trajectory(reference, tmp_path, shape):
    desc = appo.ModelDesc(*shape)
    T, od = desc.T, desc.obs_dim
    store = appo.TrajectoryStore(desc, 3, device="cpu")
    rs = np.random.default_rng(sum(shape))
    slot = 2
    r = _records(rs, T, od, rs.normal(size=512).astype(np.float32))
    store.write_slot(slot, r["obs"], r["h0"], r["actions"], r["rewards"], r["logp"], r["dones"],
                     versions=r["versions"], boot_obs=r["boot_obs"],
                     boot_hidden=r["boot_hidden"], env_id=7, worker_id=2, policy_id=1)
    mine = store.to_reference_dump(slot)
    hid = np.zeros((T, 512), np.float64)
    hid[0] = r["h0"]
    path = str(tmp_path / "ref.bin")
    st = reference.dump_trajectory(path, r["obs"].astype(np.float64), hid, r["actions"],
                                   r["rewards"].astype(np.float64), r["logp"].astype(np.float64),
                                   r["dones"], r["versions"], r["boot_obs"].astype(np.float64),
                                   r["boot_hidden"].astype(np.float64), env=7, worker=2, policy=1)
    assert st == 0
    theirs = open(path, "rb").read()
    assert len(mine) == len(theirs)
    assert mine == theirs


def test_write_step_contracts_match_reference(reference, tmp_path):
    """The slot writer rejects what the reference's write_step rejects
    (trajstore.hpp:172-183): positive behaviour log-prob, decreasing versions."""
    desc = appo.ModelDesc(1, 36, 36, 3, 4)
    store = appo.TrajectoryStore(desc, 1, device="cpu")
    rs = np.random.default_rng(0)
    r = _records(rs, 4, desc.obs_dim, np.zeros(512, np.float32))
    hid = np.zeros((4, 512))
    for bad in ("logp", "versions"):
        rr = dict(r)
        rr[bad] = r[bad].copy()
        if bad == "logp":
            rr["logp"][2] = 0.5
        else:
            rr["versions"] = np.array([3, 2, 4, 5], np.int64)
        st = reference.dump_trajectory(str(tmp_path / "x.bin"), rr["obs"].astype(np.float64), hid,
                                       rr["actions"], rr["rewards"].astype(np.float64),
                                       rr["logp"].astype(np.float64), rr["dones"], rr["versions"],
                                       rr["boot_obs"].astype(np.float64), hid[0])
        assert st == 1  # ContractError
        with pytest.raises(appo.ContractError):
            store.write_slot(0, rr["obs"], rr["h0"], rr["actions"], rr["rewards"], rr["logp"],
                             rr["dones"], versions=rr["versions"], boot_obs=rr["boot_obs"])
