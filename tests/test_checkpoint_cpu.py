"""APPOCKP1 checkpoint format parity (policy.hpp:545-605, docs/shared_memory_layout.md:95-107),
host side: the library reads the reference's own checkpoint files bit-exactly, its FNV-1a
matches common.hpp:66-74, and corrupted / foreign files are rejected like load_checkpoint."""
import os

import numpy as np
import pytest

import paper_2006_11751_b200 as appo


def test_fnv1a64_matches_reference(reference):
    rs = np.random.default_rng(3)
    for n in (0, 1, 7, 64, 1000):
        b = rs.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert appo.fnv1a64(b) == reference.L.ref_fnv1a64(b, len(b))


def test_reads_reference_checkpoint(reference, tmp_path):
    path = str(tmp_path / "ref.ckpt")
    n = reference.save_checkpoint_mlp(path, obs_dim=24, trunk=16, heads=[3, 2], seed=5,
                                      version=77, t=12)
    assert n > 0
    ck = appo.checkpoint_read(path)
    assert ck["n"] == n and ck["version"] == 77 and ck["adam_t"] == 12
    assert ck["spec_hash"] == reference.spec_hash_mlp(24, 0, 16, [3, 2])
    # the shim sets m = theta / 2 and v = theta^2 before saving
    np.testing.assert_array_equal(ck["m"], 0.5 * ck["theta"])
    np.testing.assert_array_equal(ck["v"], ck["theta"] * ck["theta"])
    assert np.abs(ck["theta"]).max() > 0
    # byte layout: magic "APPOCKP1", then the header, then theta | m | v
    raw = open(path, "rb").read()
    assert int.from_bytes(raw[:8], "little") == 0x4150504F434B5031
    assert len(raw) == 48 + 3 * 8 * n
    assert int.from_bytes(raw[40:48], "little") == appo.fnv1a64(raw[48:48 + 8 * n])


def test_corrupted_and_foreign_files_rejected(reference, tmp_path):
    path = str(tmp_path / "ref.ckpt")
    n = reference.save_checkpoint_mlp(path, 8, 8, [4], 1, 1, 1)
    raw = bytearray(open(path, "rb").read())
    bad = bytearray(raw)
    bad[48 + 8 * (n // 2)] ^= 0x40  # theta byte: checksum mismatch
    open(path, "wb").write(bad)
    with pytest.raises(appo.AppoError):
        appo.checkpoint_read(path)
    bad = bytearray(raw)
    bad[0] ^= 1  # magic
    open(path, "wb").write(bad)
    with pytest.raises(appo.AppoError):
        appo.checkpoint_read(path, arrays=False)
    open(path, "wb").write(raw[: 48 + 8 * n])  # truncated after theta
    with pytest.raises(appo.AppoError):
        appo.checkpoint_read(path)
    with pytest.raises(appo.AppoError):
        appo.checkpoint_read(os.path.join(str(tmp_path), "missing.ckpt"))


def test_model_spec_hash_is_shape_keyed():
    d = appo.ModelDesc.doom()
    h = appo.model_spec_hash(d)
    assert h == appo.model_spec_hash(appo.ModelDesc.doom(T=8))  # T is not part of the shape
    assert h != appo.model_spec_hash(appo.ModelDesc(3, 72, 128, 5, 32))
    assert h != appo.model_spec_hash(appo.ModelDesc(1, 72, 128, 6, 32))
