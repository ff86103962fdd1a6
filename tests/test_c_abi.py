"""A compiled-C caller of include/dpr.h (tests/c/abi_smoke.c, gcc, no Python in the loop):
the header is self-contained C99 and the library's C ABI works from C."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    from paper_2407_00179_b200 import build
    lib = build.build()
    out = str(tmp_path_factory.mktemp("cabi") / "abi_smoke")
    cuda = "/usr/local/cuda"
    subprocess.check_call(["gcc", "-std=c99", "-O1", "-Wall", "-Werror", "-D_DEFAULT_SOURCE",
                           "-I", os.path.join(ROOT, "include"), "-I", cuda + "/include",
                           os.path.join(ROOT, "tests", "c", "abi_smoke.c"), "-o", out,
                           lib, "-L", cuda + "/lib64", "-lcudart", "-lm",
                           "-Wl,-rpath," + os.path.dirname(lib) + ":" + cuda + "/lib64"])
    return out


def test_c_caller_host_calls(exe):
    r = subprocess.run([exe, "host"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "host ok" in r.stdout


@pytest.mark.gpu
def test_c_caller_renders_closed_form(exe):
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "gpu ok" in r.stdout
