"""Randomised parity sweep (tools/fuzz_parity.py) at a bounded size: ragged
and empty lists, odd dimensions, duplicated rows (exact ties), both metrics,
mixed residency and miss modes, nprobe beyond nc, k beyond the candidate
count, batches that take the tensor-core coarse path. 1750 trials over five
seeds passed on B200 when this was added."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("seed", [11, 12])
def test_fuzz_parity(seed):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_parity.py"),
                        "--trials", "60", "--seed", str(seed)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
