"""The C++ shim of INTEGRATION.md (integration/laiv_gpu_shim.hpp) against the
unmodified reference: integration/_build/shim_demo runs laiv::ivf_search,
laiv::hybrid_search and laiv::coarse_probe from the reference sources next to
their laiv::gpu:: drop-ins on the same index (built by the reference's own
build_index) and requires them to agree (SURVEY §8c rule)."""
import json
import os
import subprocess

import pytest

from common import ROOT

pytestmark = pytest.mark.gpu
DEMO = os.path.join(ROOT, "integration", "_build", "shim_demo")


@pytest.mark.skipif(not os.path.exists(DEMO), reason="shim_demo not built (needs the reference tree)")
@pytest.mark.parametrize("metric", ["ip", "l2"])
def test_cpp_shim_against_reference(metric):
    r = subprocess.run([DEMO, metric], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["agree"] == out["queries"] == out["batch_agree"] == out["probe_identical"]
    # LAIX: reference save_index -> laivg_index_load -> same answers, and
    # laivg_index_save writes the reference's bytes back
    assert out["laix_agree"] == out["queries"] and out["laix_same_bytes"]
