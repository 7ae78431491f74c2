"""Runs the drop-in C++ API test program (tests/cpp/test_dropin.cpp, built by
`make`), i.e. reference-style C++ user code against include/spconv/*.hpp."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "tests", "cpp", "_build", "test_dropin")


@pytest.mark.gpu
def test_dropin_cpp_program():
    assert os.path.exists(BIN), "build it with `make` (or __graft_entry__.build())"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
