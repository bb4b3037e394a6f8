"""Runs the C++ drop-in API tests (tests/cpp/test_dropin.cpp) on the GPU: the
reference-shaped C++ interface (include/fusedce) over libfce.so, checked
against the oracle and the reference's known-answer values."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def test_dropin_binary_builds():
    assert os.path.exists(BIN), "run `make` (or __graft_entry__.build()) first"


@pytest.mark.gpu
def test_dropin_cpp_api(cuda):
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout
