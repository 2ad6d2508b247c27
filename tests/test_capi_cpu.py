"""CPU-side checks of the product library: it loads without a GPU, exports
every symbol the public headers declare, and its host-only entry points
(layout, parameter contract, validation) behave like the reference."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def header_symbols():
    syms = set()
    for h in ("appo_capi.h", "appo_internal.h"):
        txt = open(os.path.join(ROOT, "include", h)).read()
        syms |= set(re.findall(r"APPO_API\s+[\w\s\*]*?\b(appo_\w+)\s*\(", txt))
    return syms


def test_library_builds_and_exports_header_symbols():
    import paper_2006_11751_b200 as appo
    out = subprocess.run(["nm", "-D", "--defined-only", appo.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    missing = header_symbols() - exported
    assert not missing, missing
    assert len(header_symbols()) >= 30
    assert appo.LIB.appo_capi_version() == 1


def test_sass_contains_tcgen05_and_tma():
    # the GEMM engine really is tcgen05 + TMA (B200_PROFILING.md mnemonics)
    obj = os.path.join(ROOT, "paper_2006_11751_b200", "build", "gemm.cu.o")
    if not os.path.exists(obj):
        pytest.skip("object files not present")
    sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass
    assert "HMMA" not in sass.replace("UTCHMMA", "")


def test_param_count_and_layout_host_only(oracle):
    import paper_2006_11751_b200 as appo
    d = appo.ModelDesc.doom()
    assert appo.param_count(d) == 2872551 == oracle.param_count(3, 72, 128, 6)
    for T, (c, h, w) in ((32, (3, 72, 128)), (8, (3, 36, 36)), (16, (1, 64, 64))):
        desc = appo.ModelDesc(c, h, w, 6, T)
        L = appo.slot_layout(desc)
        ref = oracle.slot_offsets(T, c * h * w, 512, 1)
        assert list(L.values()) == ref
        assert appo.param_count(desc) == oracle.param_count(c, h, w, 6)


def test_layout_v2_follows_reference_offsets_algorithm(reference):
    # same header size / field order / align8 as trajstore.hpp:62-87; only the
    # element sizes differ (u8 obs, f32 hidden/reward/logp)
    import paper_2006_11751_b200 as appo
    ref = reference.slot_offsets(32, 27648, 512, 1)
    L = appo.slot_layout(appo.ModelDesc.doom())
    assert ref[0] == L["obs"] == 64
    # hidden offset = 64 + align8(T*obs_dim*elem)
    assert ref[1] - 64 == 32 * 27648 * 8 and L["hidden"] - 64 == 32 * 27648


def test_bad_desc_is_config_error():
    import paper_2006_11751_b200 as appo
    with pytest.raises(appo.ConfigError):
        appo.slot_layout(appo.ModelDesc(3, 10, 10, 6, 32))
    assert appo.param_count(appo.ModelDesc(3, 72, 128, 99, 32)) == -1


def test_ctx_without_gpu_fails_loudly():
    import torch
    import paper_2006_11751_b200 as appo
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(appo.AppoError):
        appo.Context(0)
    h = C.c_void_p()
    st = appo.LIB.appo_ctx_create(None, 0, 1, C.byref(h))
    assert st in (1, 4)


REF_INC = "/root/reference/proj/include"


@pytest.mark.parametrize("src,ref_inc", [("capi_host_test.cpp", False),
                                         ("cli_exit_test.cpp", True)])
def test_cpp_mirror_compiles(tmp_path, src, ref_inc):
    """include/appo_b200.hpp compiles standalone (own exception types) and,
    with the reference's include path, aliases ::appo::ContractError /
    ConfigError / NumericError (cli_exit_test.cpp static_asserts it)."""
    import paper_2006_11751_b200 as appo
    if ref_inc and not os.path.isdir(os.path.join(REF_INC, "appo")):
        pytest.skip("reference headers absent")
    cmd = ["g++", "-std=c++20", "-O0", "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include"]
    if ref_inc:
        cmd += ["-I", REF_INC]
    cmd += [os.path.join(ROOT, "tests", "cpp", src), "-o", str(tmp_path / "a.out"),
            "-L", os.path.dirname(appo.LIB_PATH), "-lappo_b200", "-L", "/usr/local/cuda/lib64",
            "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
