"""GPU: a short randomised parity run (scripts/fuzz_parity.py, fixed seed):
random geometries, kernels (dense / zero / NaN taps), layouts, batches,
forced paths and band forms, all bit-exact vs the oracle.  The long run
(600 s, 86,012 cases, 0 failures) is in profiles/r01z/fuzz_600s.txt."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_fuzz_parity_short():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "fuzz_parity.py"), "15", "7"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " 0 failures" in r.stdout
