"""The size-unbounded drop-in (VERDICT r01 Missing #1/#2), through the C ABI,
against the UNMODIFIED reference core (oracle/_ref/libref.so) on the same
inputs:

* k > 256 (the register top-k limit): search_clusters / ivf_search /
  hybrid_search / the batched path with resident, host-scanned and
  runtime-fetched lists, k up to 5000 (ivf.cpp:326-343: partial_sort takes any
  k);
* nc > 16384 (the on-chip ranking limit): rank_clusters / coarse_probe /
  ivf_search on a 65,536-list index (ivf.cpp:269-299);
* score_clusters (ivf.cpp:301-324), exact_search (vectorstore.cpp:117-139),
  pairwise_l2 (vectorstore.cpp:141-153) exported through the ABI.

Comparison: bit-for-bit where the test says so, else the SURVEY §8c rule.
"""
import numpy as np
import pytest

from common import IP, L2, assert_topk_parity, planted_data

pytestmark = pytest.mark.gpu
BIG = 1 << 34


def _ref():
    from oracle.oracle import RefLib

    if not RefLib.available():
        pytest.skip("oracle/_ref/libref.so not built")
    return RefLib()


def _set(dev, mask):
    dev.store.clear()
    for c in np.nonzero(mask)[0]:
        dev.store.insert(int(c))


@pytest.mark.parametrize("metric", [IP, L2])
@pytest.mark.parametrize("k", [257, 1000, 5000])
def test_large_k_single(laiv, metric, k):
    ref = _ref()
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    ri = ref.index(cen, vecs, ids, off, metric)
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
    for fetch in ("off", "all"):
        dev = laiv.Device(ix, BIG, miss_fetch=fetch)
        rng = np.random.default_rng(k + metric)
        exact = 0
        for t in range(6):
            _set(dev, rng.random(64) < 0.5)
            L = int(rng.integers(8, 40))
            res, _ = laiv.hybrid_search(dev, qo[t], L, k)
            wi, ws = ri.ivf_search(qo[t], L, k)
            assert_topk_parity(metric, res.topk.ids, res.topk.scores, wi, ws)
            exact += np.array_equal(res.topk.ids, wi) and np.array_equal(res.topk.scores, ws)
            # explicit clusters, duplicates included
            cl = [3, 5, 3, 60]
            got = laiv.search_clusters(dev, qo[t], cl, k)
            wi2, ws2 = ri.search_clusters(qo[t], cl, k)
            assert_topk_parity(metric, got.ids, got.scores, wi2, ws2)
        print(f"[wide] k={k} metric={metric} fetch={fetch}: {exact}/6 bit-identical")
        assert exact >= 5
        dev.close()


@pytest.mark.parametrize("metric", [IP, L2])
def test_large_k_batch(laiv, metric):
    ref = _ref()
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    ri = ref.index(cen, vecs, ids, off, metric)
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
    k, L = 700, 24
    for fetch in ("off", "auto", "all"):
        dev = laiv.Device(ix, BIG, miss_fetch=fetch, fetch_chunk_mb=2)
        _set(dev, np.arange(64) % 3 == 0)
        res, tm = laiv.hybrid_search_batch(dev, qo[:20], L, k)
        for q in range(20):
            wi, ws = ri.ivf_search(qo[q], L, k)
            n = res.counts[q]
            assert_topk_parity(metric, res.ids[q, :n], res.scores[q, :n], wi, ws)
        dev.close()


def test_exact_search_any_k(laiv):
    ref = _ref()
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    for metric in (IP, L2):
        ri = ref.index(cen, vecs, ids, off, metric)
        ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
        dev = laiv.Device(ix, BIG)
        _set(dev, np.arange(64) % 2)
        for k in (1, 10, 300, 19200, 25000):  # 19200 = every row; beyond returns all
            got = laiv.exact_search(dev, qo[0], k)
            wi, ws = ri.exact_search(qo[0], k)
            assert_topk_parity(metric, got.ids, got.scores, wi, ws)
        with pytest.raises(ValueError):
            laiv.exact_search(dev, qo[0], 0)
        dev.close()


def test_score_clusters(laiv):
    ref = _ref()
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    for metric in (IP, L2):
        ri = ref.index(cen, vecs, ids, off, metric)
        ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
        dev = laiv.Device(ix, BIG)
        _set(dev, np.arange(64) % 2)  # odd lists resident: GPU; even: host
        for cl in ([0], [1], [5, 2, 5, 63, 0], list(range(64)), []):
            gi, gs = laiv.score_clusters_arrays(dev, qo[1], cl)
            wi, ws = ri.score_clusters(qo[1], cl)
            assert np.array_equal(gi, wi)  # the reference's candidate order
            assert np.allclose(gs, ws, rtol=1e-6, atol=0)
            # fp64 accumulation rounded to f32: equal bits but for rare
            # rounding-boundary cases
            assert gs.size == 0 or np.mean(gs == ws) > 0.999
        with pytest.raises(ValueError):
            laiv.score_clusters(dev, qo[1], [64])
        dev.close()


def test_pairwise_l2_bit_identical(laiv):
    ref = _ref()
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.L2)
    dev = laiv.Device(ix, 1 << 24)
    rng = np.random.default_rng(3)
    for na, nb, d in ((1, 1, 1), (3, 3, 2), (37, 70, 768), (100, 33, 17)):
        a = rng.standard_normal((na, d)).astype(np.float32)
        b = rng.standard_normal((nb, d)).astype(np.float32)
        got = laiv.pairwise_l2(dev, a, b)
        want = ref.pairwise_l2(a, b)
        assert np.array_equal(got, want)
    a = np.array([[0, 0], [3, 4]], np.float32)  # test_vectorstore.cpp:131-137
    assert np.array_equal(laiv.pairwise_l2(dev, a, a), np.array([0, 5, 5, 0], np.float32))
    with pytest.raises(ValueError):
        laiv.pairwise_l2(dev, np.zeros((2, 3), np.float32), np.zeros((2, 4), np.float32))


@pytest.mark.parametrize("metric", [IP, L2])
def test_65536_lists(laiv, metric):
    """nc = 65,536 (4x the on-chip ranking limit): rankings, probes and
    searches equal the reference's."""
    ref = _ref()
    nc, per, d = 65536, 3, 16
    cen = laiv.synth_centroids(5, nc, d)
    vecs, ids = laiv.synth_lists(5, cen, per, 0.05)
    off = np.arange(0, nc * per + 1, per, dtype=np.uint64)
    qi, qo, _ = laiv.synth_queries(6, vecs, 24, 0.01)
    ri = ref.index(cen, vecs, ids, off, metric)
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
    dev = laiv.Device(ix, nc * per * (4 * d + 8) // 4, max_batch=32)
    _set(dev, np.arange(nc) % 4 == 0)
    for t in range(4):
        assert np.array_equal(laiv.rank_clusters(dev, qi[t]), ri.rank_clusters(qi[t]))
        assert np.array_equal(laiv.coarse_probe(dev, qi[t], 300), ri.coarse_probe(qi[t], 300))
        res, _ = laiv.hybrid_search(dev, qo[t], 200, 10)
        wi, ws = ri.ivf_search(qo[t], 200, 10)
        assert_topk_parity(metric, res.topk.ids, res.topk.scores, wi, ws, exact=True)
    # batched (coarse of 24 queries at once) and large k together
    res, _ = laiv.hybrid_search_batch(dev, qo, 128, 300)
    for q in range(24):
        wi, ws = ri.ivf_search(qo[q], 128, 300)
        n = res.counts[q]
        assert_topk_parity(metric, res.ids[q, :n], res.scores[q, :n], wi, ws)
    probes = laiv.coarse_probe(dev, qi, 64)
    for q in range(24):
        assert np.array_equal(probes[q], ri.coarse_probe(qi[q], 64))
