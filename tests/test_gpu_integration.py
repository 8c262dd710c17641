"""The C++ shim of INTEGRATION.md (integration/laiv_gpu_shim.hpp) against the
unmodified reference: integration/_build/shim_demo compiles ONE caller
(integration/caller_body.inc: grouping, cache-aware routing, lookahead plan
and transfer, hybrid retrieval, hotness eviction, incremental prefetch, and
rank/probe/score/search_clusters/ivf/exact/pairwise/coverage) twice, against
namespace laiv and against laiv::gpu with the reference's signatures, and
requires both runs to make the same decisions and return the same results
(SURVEY §8c rule for scores)."""
import json
import os
import subprocess

import pytest

from common import ROOT

pytestmark = pytest.mark.gpu
DEMO = os.path.join(ROOT, "integration", "_build", "shim_demo")


@pytest.mark.skipif(not os.path.exists(DEMO), reason="shim_demo not built (needs the reference tree)")
@pytest.mark.parametrize("metric", ["ip", "l2"])
def test_cpp_shim_against_reference(metric, tmp_path):
    r = subprocess.run([DEMO, metric, str(tmp_path)], capture_output=True, text=True, timeout=600)
    out = json.loads(r.stdout.strip().splitlines()[-1])
    print(out)
    assert r.returncode == 0, r.stdout + r.stderr
    assert out["all"]
    assert out["decisions_identical"] and out["rank_probe_coverage_identical"]
    assert out["pairwise_bit_identical"] and out["score_clusters_agree"]
    assert out["batch_agree"] == out["queries"] == out["hybrid_agree"]
    # LAIX: reference save_index -> laivg_index_load -> same answers, and
    # laivg_index_save writes the reference's bytes back
    assert out["laix_agree"] == out["queries"] and out["laix_same_bytes"]
