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


CLI_EXIT = os.path.join(ROOT, "oracle", "_ref", "cli_exit_test")


@pytest.mark.parametrize("scenario,code", [("ok", 0), ("config", 2), ("numeric-vtrace", 3),
                                           ("numeric-adam", 3), ("contract", 4)])
def test_reference_exceptions_map_to_cli_exit_codes(scenario, code):
    """cli_exit_test was compiled against the reference's <appo/common.hpp>
    (oracle/Makefile): the boundary throws ::appo:: exception types and the
    CLI's catch chain (appo_cli.cpp:151-163) maps a device-detected non-finite
    value to exit 3, an invalid config to 2, the rest to 4 (runner.hpp:28-33)."""
    if not os.path.exists(CLI_EXIT):
        pytest.skip("oracle/_ref/cli_exit_test not built (needs /root/reference at build time)")
    r = subprocess.run([CLI_EXIT, scenario], capture_output=True, text=True, timeout=120)
    assert r.returncode == code, r.stderr + r.stdout
    if scenario == "contract":
        assert "caught appo::ContractError" in r.stdout
