"""The C++ host mirror (include/appo_b200.hpp) over the C ABI: builds
tests/cpp/capi_host_test.cpp with g++ against libappo_b200.so and runs it."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_cpp_host_api(tmp_path):
    import paper_2006_11751_b200 as appo  # ensures the library is built
    exe = str(tmp_path / "capi_host_test")
    libdir = os.path.dirname(appo.LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    "-I", "/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "cpp", "capi_host_test.cpp"), "-o", exe,
                    "-L", libdir, "-lappo_b200", "-L", "/usr/local/cuda/lib64", "-lcudart",
                    f"-Wl,-rpath,{libdir}"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "capi_host_test ok" in r.stdout
