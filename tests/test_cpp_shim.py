"""Builds and runs the C++ parity tests of include/rlu_b200.hpp (tests/cpp/test_shim.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2306_14337_b200", "lib")
EXE = os.path.join(ROOT, "tests", "cpp", "test_shim")


def _build():
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    subprocess.run([cxx, "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"), "-o", EXE, "-L", LIBDIR, "-lb200lu",
                    f"-Wl,-rpath,{LIBDIR}"], check=True)


def test_cpp_mirror_compiles_against_the_c_abi():
    """CPU-side: the header-only mirror and its test build and link against libb200lu.so; without a
    device the binary refuses to compute (exit code 3) instead of falling back."""
    _build()
    from paper_2306_14337_b200 import _capi
    if _capi.lib().b200lu_device_count() == 0:
        r = subprocess.run([EXE], capture_output=True, text=True)
        assert r.returncode == 3 and "no CUDA device" in r.stdout


@pytest.mark.gpu
def test_cpp_mirror_parity_on_device():
    _build()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all ok" in r.stdout and r.stdout.count("\nok ") + r.stdout.startswith("ok ") >= 7
