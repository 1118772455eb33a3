"""The reference-side adapter (integration/rlu/b200_backend.hpp — what a maintainer drops into the reference
tree) compiled against the UNMODIFIED reference headers and core sources and linked with
libb200lu.so. The binary is built by oracle/Makefile where the reference tree exists (target
oracle/_ref/adapter_test; it travels to the GPU box like librlu_ref.so) and runs the per-system loop of
cli::solve_sequence (src/cli.cpp:96-135) twice — reference CPU calls, then their rlu::b200:: twins."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "adapter_test")

needs_exe = pytest.mark.skipif(not os.path.exists(EXE), reason="oracle/_ref/adapter_test not built (needs the reference tree)")


@needs_exe
def test_adapter_builds_and_refuses_without_a_device():
    from paper_2306_14337_b200 import _capi
    if _capi.lib().b200lu_device_count() > 0:
        pytest.skip("a device is present")
    r = subprocess.run([EXE], capture_output=True, text=True)
    assert r.returncode == 3 and "no CUDA device" in r.stdout
    # the host-side part runs without a device: rlu::b200::symbolic_analyze == the reference's symbolic_analyze, field by
    # field, with and without MC64, and the reference's own CPU factorization runs on its product
    assert r.stdout.count("ok symbolic_analyze") == 2


@needs_exe
@pytest.mark.gpu
@pytest.mark.parametrize("shape", [("1400", "600"), ("6300", "2700")], ids=["n2000", "C1"])
def test_adapter_sequence_bitwise_on_device(shape):
    r = subprocess.run([EXE, *shape], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all ok" in r.stdout and r.stdout.count("L/U bitwise") == 10
    assert "ok cgs2" in r.stdout and "ok errors" in r.stdout and r.stdout.count("ok symbolic_analyze") == 2
