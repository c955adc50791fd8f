"""The C++ drop-in (include/lattice/*.hpp over the C ABI) running the reference's own test
expectations on the GPU: tests/cpp/test_dropin.cpp, built by __graft_entry__.build()."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def test_dropin_binary_built():
    assert os.path.exists(BIN), "run __graft_entry__.build()"


@pytest.mark.gpu
def test_dropin_cpp_suite():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
