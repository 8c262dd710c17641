"""LAIX-loaded stores on the GPU path: laivg_index_load pins the block it
read in place (cudaHostRegister on a box with a driver); contexts built on
it must answer exactly as contexts built from the arrays, through the
cache-hit scan, the host miss scan and the runtime fetch ring."""
import numpy as np
import pytest

from common import assert_topk_parity, planted_data

pytestmark = pytest.mark.gpu
BIG = 1 << 30


@pytest.mark.parametrize("metric", [0, 1])
def test_loaded_index_serves_like_arrays(tmp_path, orc, laiv, metric):
    cen, vecs, ids, off, qi, qo, g = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
    path = tmp_path / "planted.laix"
    ix.save(path)
    lx = laiv.load_index(path)
    v2, i2 = lx.store()
    assert np.array_equal(v2, vecs) and np.array_equal(i2, ids)
    for fetch in ("off", "all"):
        a = laiv.Device(lx, BIG, miss_fetch=fetch, fetch_chunk_mb=2)
        b = laiv.Device(ix, BIG, miss_fetch=fetch, fetch_chunk_mb=2)
        for dv in (a, b):
            dv.store.clear()
            for c in range(0, 64, 3):
                dv.store.insert(c)
        ra, _ = laiv.hybrid_search_batch(a, qo, 16, 10)
        rb, _ = laiv.hybrid_search_batch(b, qo, 16, 10)
        assert np.array_equal(ra.ids, rb.ids) and np.array_equal(ra.scores, rb.scores)
        for t in range(0, 40, 5):
            sa, _ = laiv.hybrid_search(a, qo[t], 16, 10)
            want = orc.ivf_search(cen, vecs, ids, off, metric, qo[t], 16, 10)
            assert_topk_parity(metric, sa.topk.ids, sa.topk.scores, *want)
        # prefetch copies come out of the loaded (registered) block
        a.store.clear()
        plan = laiv.plan_prefetch(a, qi[0], 20 * 300 * (4 * 768 + 8))
        rep = laiv.execute_prefetch(a, plan, laiv.TransferChannel(55e9, laiv.ChannelMode.Device))
        assert rep.bytes == sum(300 * (4 * 768 + 8) for _ in rep.transferred) > 0
        del a, b
