"""Parity of the CUDA path (through the C ABI) with the reference.

Against the golden fixtures recorded from the unmodified reference (bit-exact
for D = 8 / 16 where fp64 partial sums are exact), against the C oracle on the
planted D = 768 datastore (SURVEY §8c rule: ids bit-exact across gaps above
1e-5 relative, scores within 1e-5 relative), and through size-independent
properties (hybrid == monolithic under any residency, full probe == exact).
"""
import numpy as np
import pytest

from common import (IP, L2, accept1_case, assert_topk_parity, expected_row, golden,
                    hybrid_d8_case, planted_data, probe_parity)

pytestmark = pytest.mark.gpu
BIG = 1 << 34


def device_for(laiv, case, capacity=BIG, **kw):
    ix = laiv.IvfIndex(case.centroids, case.vecs, case.ids, case.list_off, laiv.Metric(case.metric))
    return ix, laiv.Device(ix, capacity, **kw)


def set_residency(dev, mask):
    dev.store.clear()
    for c in np.nonzero(mask)[0]:
        dev.store.insert(int(c))


@pytest.mark.parametrize("name", ["l2", "ip"])
def test_hybrid_d8_golden(orc, laiv, name):
    case, queries, g = hybrid_d8_case(orc, name)
    ix, dev = device_for(laiv, case)
    p = f"{name}_"
    for t in range(200):
        set_residency(dev, g[p + "masks"][t])
        L, k = int(g[p + "L"][t]), int(g[p + "k"][t])
        res, timing = laiv.hybrid_search(dev, queries[t], L, k)
        want_ids, want_sc = expected_row(g, p, t)
        assert_topk_parity(case.metric, res.topk.ids, res.topk.scores, want_ids, want_sc,
                           exact=True)
        ef, es = g[p + "exp_fast"][t], g[p + "exp_slow"][t]
        assert res.fast_clusters == [int(c) for c in ef[ef >= 0]]
        assert res.slow_clusters == [int(c) for c in es[es >= 0]]
        n = len(res.fast_clusters) + len(res.slow_clusters)
        assert res.hit_rate == (len(res.fast_clusters) / n if n else 0.0)
    for t in range(50):
        assert np.array_equal(laiv.rank_clusters(dev, queries[t]), g[p + "rank"][t])


def test_acceptance1_golden(orc, laiv):
    case, queries, masks, full_q, g = accept1_case(orc)
    ix, dev = device_for(laiv, case)
    for t in range(1000):
        set_residency(dev, masks[t])
        res, _ = laiv.hybrid_search(dev, queries[t], int(g["L"][t]), int(g["k"][t]))
        want_ids, want_sc = expected_row(g, "", t)
        assert_topk_parity(L2, res.topk.ids, res.topk.scores, want_ids, want_sc, exact=True)
    # full probe == exact search (acceptance.cpp:85-93), everything resident
    set_residency(dev, np.ones(64, np.uint8))
    for t in range(200):
        k = int(g["full_k"][t])
        got = laiv.ivf_search(dev, full_q[t], 64, k)
        assert_topk_parity(L2, got.ids, got.scores, g["full_ids"][t, :k], g["full_scores"][t, :k],
                           exact=True)


@pytest.mark.parametrize("name,metric", [("l2", L2), ("ip", IP)])
@pytest.mark.parametrize("acc_fp64", [True, False])
def test_planted_d768(orc, laiv, name, metric, acc_fp64):
    cen, vecs, ids, off, qi, qo, g = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
    dev = laiv.Device(ix, BIG, acc_fp64=acc_fp64)
    set_residency(dev, np.ones(64, np.uint8))
    exact = 0
    for t in range(40):
        got = laiv.ivf_search(dev, qo[t], 8, 10)
        want_ids, want_sc = g[f"{name}_ids"][t], g[f"{name}_scores"][t]
        assert_topk_parity(metric, got.ids, got.scores, want_ids, want_sc)
        exact += np.array_equal(got.ids, want_ids) and np.array_equal(got.scores, want_sc)
        order, scores = orc.rank_clusters(cen, metric, qi[t], with_scores=True)
        assert np.array_equal(order, g[f"{name}_rank"][t])
        gp = laiv.coarse_probe(dev, qi[t], 8)
        probe_parity(gp, order, scores, 8)
        assert laiv.coverage(dev, qi[t], qo[t], 8) == pytest.approx(g[f"{name}_coverage"][t])
    # fp64 accumulation, or fp32 accumulation + the exact fp64 re-score of the
    # survivors, reproduces the reference bit for bit on this datastore
    assert exact == 40


@pytest.mark.parametrize("metric", [L2, IP])
def test_random_residency_d768(orc, laiv, metric):
    # hybrid == monolithic on the planted datastore for random residency
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
    dev = laiv.Device(ix, BIG)
    rng = np.random.default_rng(5)
    for t in range(20):
        set_residency(dev, (rng.random(64) < rng.random()).astype(np.uint8))
        L = int(rng.integers(1, 65))
        k = int(rng.integers(1, 33))
        res, timing = laiv.hybrid_search(dev, qo[t], L, k)
        want = orc.ivf_search(cen, vecs, ids, off, metric, qo[t], L, k)
        assert_topk_parity(metric, res.topk.ids, res.topk.scores, *want)
        assert timing.scanned_vectors == 300 * len(res.fast_clusters)


@pytest.mark.parametrize("k", [1, 31, 32, 33, 64, 100, 129, 256])
def test_k_range(orc, laiv, k):
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.L2)
    dev = laiv.Device(ix, BIG)
    set_residency(dev, np.arange(64) % 2)
    for t in range(3):
        got = laiv.ivf_search(dev, qo[t], 16, k)
        want = orc.ivf_search(cen, vecs, ids, off, L2, qo[t], 16, k)
        assert_topk_parity(L2, got.ids, got.scores, *want)


def test_edge_cases(orc, laiv):
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
    dev = laiv.Device(ix, BIG)
    set_residency(dev, np.ones(64, np.uint8))
    # L = 0 / negative: empty probe, empty result
    assert laiv.ivf_search(dev, qo[0], 0, 5).entries == []
    assert laiv.ivf_search(dev, qo[0], -3, 5).entries == []
    # L > nc clamps to nc
    got = laiv.ivf_search(dev, qo[0], 1000, 5)
    want = orc.ivf_search(cen, vecs, ids, off, IP, qo[0], 64, 5)
    assert_topk_parity(IP, got.ids, got.scores, *want)
    # k larger than the candidate count returns everything, sorted
    got = laiv.search_clusters(dev, qo[0], [3], 300 if False else 256)
    want = orc.search_clusters(vecs, ids, off, IP, qo[0], [3], 256)
    assert_topk_parity(IP, got.ids, got.scores, *want)
    # errors mirror the reference exception classes
    with pytest.raises(ValueError):
        laiv.ivf_search(dev, qo[0], 8, 0)
    with pytest.raises(ValueError):
        laiv.search_clusters(dev, qo[0], [64], 3)
    with pytest.raises(ValueError):
        laiv.ivf_search(dev, qo[0][:10], 8, 3)
    # empty cluster list
    assert laiv.search_clusters(dev, qo[0], [], 3).entries == []


def test_ragged_lists_and_empty_lists(orc, laiv):
    # lists of very different sizes incl. empty ones; D not a multiple of 128
    rng = np.random.default_rng(3)
    nc, d = 40, 100
    sizes = rng.integers(0, 400, nc)
    sizes[[3, 17, 18]] = 0
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint64)
    n = int(off[-1])
    vecs = rng.standard_normal((n, d)).astype(np.float32)
    ids = rng.permutation(10 * n)[:n].astype(np.uint64)  # non-monotone ids
    cen = rng.standard_normal((nc, d)).astype(np.float32)
    for metric in (L2, IP):
        ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
        dev = laiv.Device(ix, BIG)
        for t in range(10):
            set_residency(dev, (rng.random(nc) < 0.6).astype(np.uint8))
            q = rng.standard_normal(d).astype(np.float32)
            L = int(rng.integers(1, nc + 1))
            k = int(rng.integers(1, 50))
            res, _ = laiv.hybrid_search(dev, q, L, k)
            want = orc.ivf_search(cen, vecs, ids, off, metric, q, L, k)
            assert_topk_parity(metric, res.topk.ids, res.topk.scores, *want)


def test_ties_break_by_id(orc, laiv):
    # duplicated vectors: equal scores must order by ascending id
    rng = np.random.default_rng(9)
    d, nc, per = 768, 4, 64
    base = rng.standard_normal((per // 4, d)).astype(np.float32)
    vecs = np.concatenate([np.repeat(base, 4, axis=0)] * nc)
    ids = rng.permutation(nc * per).astype(np.uint64) * 7
    off = np.arange(0, nc * per + 1, per, dtype=np.uint64)
    cen = rng.standard_normal((nc, d)).astype(np.float32)
    for metric in (L2, IP):
        ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
        dev = laiv.Device(ix, BIG)
        set_residency(dev, np.array([1, 0, 1, 0], np.uint8))
        q = rng.standard_normal(d).astype(np.float32)
        res, _ = laiv.hybrid_search(dev, q, 4, 40)
        want = orc.ivf_search(cen, vecs, ids, off, metric, q, 4, 40)
        assert_topk_parity(metric, res.topk.ids, res.topk.scores, *want, exact=True)


@pytest.mark.parametrize("nc", [1, 3, 33, 1000, 2048, 4096, 5000, 8192, 16384])
def test_rank_clusters_all_sort_sizes(orc, laiv, nc):
    # every on-chip sort geometry (1..16 elements per thread) vs the oracle
    rng = np.random.default_rng(nc)
    d = 64
    cen = rng.standard_normal((nc, d)).astype(np.float32)
    cen[nc // 2] = cen[0]  # an exact tie: must order by ascending cluster id
    vecs = rng.standard_normal((nc, d)).astype(np.float32)
    off = np.arange(nc + 1, dtype=np.uint64)
    for metric in (L2, IP):
        ix = laiv.IvfIndex(cen, vecs, np.arange(nc, dtype=np.uint64), off, laiv.Metric(metric))
        dev = laiv.Device(ix, 1 << 24)
        Q = rng.standard_normal((3, d)).astype(np.float32)
        got = laiv.rank_clusters(dev, Q)
        for t in range(3):
            assert np.array_equal(got[t], orc.rank_clusters(cen, metric, Q[t]))
        probe = laiv.coarse_probe(dev, Q, 17)
        for t in range(3):
            assert np.array_equal(probe[t], orc.coarse_probe(cen, metric, Q[t], 17))


@pytest.mark.parametrize("resident", [0, 1])
def test_search_clusters_duplicate_clusters(orc, laiv, resident):
    # score_clusters appends every member of every listed cluster, so a
    # cluster named twice contributes its members twice (ivf.cpp:301-323)
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
    dev = laiv.Device(ix, BIG)
    set_residency(dev, np.full(64, resident, np.uint8))
    for t in range(3):
        cl = [int(x) for x in laiv.coarse_probe(dev, qo[t], 3)]
        cl = [cl[0], cl[1], cl[0], cl[2], cl[0]]
        got = laiv.search_clusters(dev, qo[t], cl, 12)
        want = orc.search_clusters(vecs, ids, off, IP, qo[t], cl, 12)
        assert_topk_parity(IP, got.ids, got.scores, *want, exact=True)
