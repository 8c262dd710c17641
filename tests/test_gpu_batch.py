"""Batched retrieval on the GPU (SURVEY §8b extension point (2); north-star
subsystem (1): the coarse quantizer on tensor cores when queries batch).

* the tcgen05 tf32 coarse GEMM stays inside its error bound
  (|s~ - s| <= kTcErr ||q|| ||c||, kTcErr = 4e-3) against fp64 numpy;
* the batched probe (tensor-core scores + exact fp64 re-score of the
  boundary candidates) is bit-identical to the fp64 device ranking and meets
  the §8c rule against the C oracle;
* hybrid_search_batch / ivf_search_batch return, per query, exactly what the
  single-query path returns, and the reference's goldens (bit-exact at
  D = 8 / 16) under any residency (hybrid == monolithic, tiered.hpp:120-124).
"""
import numpy as np
import pytest

from common import (IP, L2, accept1_case, assert_topk_parity, expected_row, hybrid_d8_case,
                    planted_data, probe_parity)

pytestmark = pytest.mark.gpu
BIG = 1 << 34
TC_ERR = 4.0e-3


def set_residency(dev, mask):
    dev.store.clear()
    for c in np.nonzero(mask)[0]:
        dev.store.insert(int(c))


def synth_index(laiv, nc, per, d, metric, seed=3, nq=64, sigma=0.02):
    cen = laiv.synth_centroids(seed, nc, d)
    vecs, ids = laiv.synth_lists(seed, cen, per, 0.05)
    off = np.arange(0, nc * per + 1, per, dtype=np.uint64)
    qi, qo, _ = laiv.synth_queries(seed + 1, vecs, nq, sigma)
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
    return cen, vecs, ids, off, qi, qo, ix


@pytest.mark.parametrize("nc,d", [(300, 768), (4096, 768), (1000, 100), (77, 8)])
def test_tc_coarse_error_bound(laiv, nc, d):
    rng = np.random.default_rng(nc + d)
    cen = rng.standard_normal((nc, d)).astype(np.float32)
    vecs = rng.standard_normal((nc, d)).astype(np.float32)
    ids = np.arange(nc, dtype=np.uint64)
    off = np.arange(nc + 1, dtype=np.uint64)
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
    dev = laiv.Device(ix, 1 << 20)
    for nq in (8, 33, 256, 300):
        Q = rng.standard_normal((nq, d)).astype(np.float32) * rng.uniform(0.1, 10)
        approx = dev.coarse_approx(Q).astype(np.float64)
        exact = Q.astype(np.float64) @ cen.astype(np.float64).T
        bound = np.outer(np.linalg.norm(Q.astype(np.float64), axis=1),
                         np.linalg.norm(cen.astype(np.float64), axis=1))
        ratio = np.abs(approx - exact) / bound
        assert ratio.max() <= TC_ERR, ratio.max()
        # the bound carries a real margin (tf32 error ~ 2^-11 relative)
        assert ratio.max() < 0.75 * TC_ERR, ratio.max()


@pytest.fixture(params=["stream", "lm"])
def rescore(request, monkeypatch):
    """The batched selection's exact re-score: per (query, candidate) pair
    (default) or list-major (LAIVG_TC_RESCORE=lm)."""
    monkeypatch.setenv("LAIVG_TC_RESCORE", request.param)
    return request.param


@pytest.mark.parametrize("metric", [IP, L2])
@pytest.mark.parametrize("nc,d", [(300, 768), (4096, 768), (1000, 100)])
def test_tc_probe_bit_exact(orc, laiv, rescore, metric, nc, d):
    cen, vecs, ids, off, qi, qo, ix = synth_index(laiv, nc, 4, d, metric, nq=48)
    dev_tc = laiv.Device(ix, 1 << 20, coarse_impl="tensor")
    dev_64 = laiv.Device(ix, 1 << 20, coarse_impl="fp64")
    dev_auto = laiv.Device(ix, 1 << 20)
    Q = np.concatenate([qi, qo])
    for L in (1, 17, 128, nc - 1, nc, nc + 5):
        a = laiv.coarse_probe(dev_tc, Q, L)
        b = laiv.coarse_probe(dev_64, Q, L)
        c = laiv.coarse_probe(dev_auto, Q, L)
        assert np.array_equal(a, b), L
        assert np.array_equal(a, c), L
        Lc = min(L, nc)
        for t in range(0, Q.shape[0], 7):
            order, scores = orc.rank_clusters(cen, metric, Q[t], with_scores=True)
            probe_parity(a[t], order, scores, Lc)
    # single query forced onto the tensor cores
    for t in range(4):
        assert np.array_equal(laiv.coarse_probe(dev_tc, Q[t], 64),
                              laiv.coarse_probe(dev_64, Q[t], 64))


def test_tc_probe_exact_ties(laiv, rescore):
    # duplicated centroids: exact score ties ordered by ascending cluster id
    rng = np.random.default_rng(9)
    base = rng.standard_normal((50, 64)).astype(np.float32)
    cen = np.concatenate([base, base, base])  # 150 clusters, triples tie
    vecs = cen.copy()
    ids = np.arange(150, dtype=np.uint64)
    off = np.arange(151, dtype=np.uint64)
    for metric in (laiv.Metric.InnerProduct, laiv.Metric.L2):
        ix = laiv.IvfIndex(cen, vecs, ids, off, metric)
        dev_tc = laiv.Device(ix, 1 << 20, coarse_impl="tensor")
        dev_64 = laiv.Device(ix, 1 << 20, coarse_impl="fp64")
        Q = rng.standard_normal((16, 64)).astype(np.float32)
        for L in (1, 2, 3, 10, 149):
            assert np.array_equal(laiv.coarse_probe(dev_tc, Q, L), laiv.coarse_probe(dev_64, Q, L))


@pytest.mark.parametrize("name,metric", [("l2", L2), ("ip", IP)])
@pytest.mark.parametrize("fetch,chunk_mb", [("off", 0), ("auto", 0), ("all", 1), ("all", 3)])
def test_batch_matches_single_planted(orc, laiv, name, metric, fetch, chunk_mb):
    # misses on the host, adaptively split, or fetched on demand through a
    # 1-list / 3-list ring (many chunks, the 32-chunk cap, three-way merge)
    cen, vecs, ids, off, qi, qo, g = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
    dev = laiv.Device(ix, BIG, miss_fetch=fetch, fetch_chunk_mb=chunk_mb)
    rng = np.random.default_rng(17)
    for trial in range(4):
        set_residency(dev, (rng.random(64) < [0.0, 1.0, 0.5, 0.2][trial]).astype(np.uint8))
        L, k = [8, 16, 64, 5][trial], [10, 32, 7, 100][trial]
        res, timing = laiv.hybrid_search_batch(dev, qo, L, k)
        for t in range(40):
            single, _ = laiv.hybrid_search(dev, qo[t], L, k)
            got = res.topk(t)
            assert np.array_equal(got.ids, single.topk.ids), t
            assert np.array_equal(got.scores, single.topk.scores), t
            assert res.nfast[t] == len(single.fast_clusters)
            want = orc.ivf_search(cen, vecs, ids, off, metric, qo[t], L, k)
            assert_topk_parity(metric, got.ids, got.scores, *want)
        assert timing.scanned_vectors == 300 * int(res.nfast.sum())
        if fetch == "off":
            assert timing.fetched_lists == 0
        if fetch == "all" and trial in (0, 3):
            assert timing.fetched_lists > 0
            assert timing.fetched_bytes == timing.fetched_lists * 300 * 768 * 4


@pytest.mark.parametrize("name", ["l2", "ip"])
@pytest.mark.parametrize("fetch", ["off", "all"])
def test_batch_d8_golden(orc, laiv, name, fetch):
    # reference goldens are residency-independent (hybrid == monolithic):
    # replay them through the batch path under three residencies
    case, queries, g = hybrid_d8_case(orc, name)
    ix = laiv.IvfIndex(case.centroids, case.vecs, case.ids, case.list_off,
                       laiv.Metric(case.metric))
    dev = laiv.Device(ix, BIG, max_batch=32, miss_fetch=fetch, fetch_chunk_mb=1)
    p = f"{name}_"
    Ls, ks = g[p + "L"], g[p + "k"]
    for mask in (np.zeros(case.nc, np.uint8), np.ones(case.nc, np.uint8), g[p + "masks"][0]):
        set_residency(dev, mask)
        for L, k in sorted(set(zip(Ls.tolist(), ks.tolist()))):
            sel = [t for t in range(200) if Ls[t] == L and ks[t] == k]
            got = laiv.ivf_search_batch(dev, queries[sel], L, k)
            for t, tk in zip(sel, got):
                want_ids, want_sc = expected_row(g, p, t)
                assert_topk_parity(case.metric, tk.ids, tk.scores, want_ids, want_sc, exact=True)


def test_batch_accept1_golden(orc, laiv):
    case, queries, masks, full_q, g = accept1_case(orc)
    ix = laiv.IvfIndex(case.centroids, case.vecs, case.ids, case.list_off, laiv.Metric.L2)
    dev = laiv.Device(ix, BIG)
    set_residency(dev, masks[0])
    Ls, ks = g["L"], g["k"]
    for L, k in sorted(set(zip(Ls.tolist(), ks.tolist()))):
        sel = [t for t in range(1000) if Ls[t] == L and ks[t] == k]
        got = laiv.ivf_search_batch(dev, queries[sel], L, k)
        for t, tk in zip(sel, got):
            want_ids, want_sc = expected_row(g, "", t)
            assert_topk_parity(L2, tk.ids, tk.scores, want_ids, want_sc, exact=True)


def test_batch_edges(orc, laiv):
    cen, vecs, ids, off, qi, qo, g = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
    dev = laiv.Device(ix, BIG, max_batch=16)
    set_residency(dev, np.arange(64) % 3 == 0)
    # L = 0 / negative: empty results
    res, _ = laiv.hybrid_search_batch(dev, qo[:8], 0, 5)
    assert (res.counts == 0).all()
    res, _ = laiv.hybrid_search_batch(dev, qo[:8], -2, 5)
    assert (res.counts == 0).all()
    # L > nc clamps; more queries than max_batch chunk through ivf_search_batch
    got = laiv.ivf_search_batch(dev, qo, 1000, 12)
    for t in range(40):
        want = orc.ivf_search(cen, vecs, ids, off, IP, qo[t], 64, 12)
        assert_topk_parity(IP, got[t].ids, got[t].scores, *want)
    with pytest.raises(ValueError):
        laiv.hybrid_search_batch(dev, qo[:17], 8, 5)  # > max_batch
    with pytest.raises(ValueError):
        laiv.hybrid_search_batch(dev, qo[:4], 8, 0)


def test_prefetch_batch_matches_sequential(laiv):
    # pipeline.cpp:357-371: query i plans against the store holding the earlier
    # plans with budget min(budget_i, free bytes); shared lists travel once
    cen, vecs, ids, off, qi, qo, g = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
    cb = 300 * (4 * 768 + 8)
    cap = 20 * cb
    dev_a = laiv.Device(ix, cap)
    dev_b = laiv.Device(ix, cap)
    chan = laiv.TransferChannel(50e9, laiv.ChannelMode.Device)
    for trial, (nq, per_q) in enumerate([(8, 3 * cb), (6, 5 * cb + 7), (12, 2 * cb - 1)]):
        Q = qi[trial * 12: trial * 12 + nq]
        budgets = laiv.split_budget(per_q * nq, laiv.MicroBatch(list(range(nq))))
        dev_a.store.clear()
        dev_b.store.clear()
        dev_a.store.insert(int(laiv.coarse_probe(dev_a, Q[0], 1)[0]))  # one already resident
        dev_b.store.insert(int(laiv.coarse_probe(dev_b, Q[0], 1)[0]))
        rep, npl = laiv.prefetch_batch(dev_a, Q, budgets, chan, 0.001)
        want = []
        for i in range(nq):
            b = min(budgets[i], dev_b.store.free_bytes())
            plan = laiv.plan_prefetch(dev_b, Q[i], b)
            laiv.execute_prefetch(dev_b, plan, chan)
            assert npl[i] == len(plan.clusters)
            want += plan.clusters
        assert rep.transferred == want
        assert rep.bytes == len(want) * cb
        assert dev_a.store.resident() == dev_b.store.resident()
        assert rep.window_s >= 0.001 and rep.t_p > 0
        # the prefetched lists are scanned from HBM: batch search still exact
        res, _ = laiv.hybrid_search_batch(dev_a, qo[trial * 12: trial * 12 + nq], 8, 10)
        for t in range(nq):
            single, _ = laiv.hybrid_search(dev_b, qo[trial * 12 + t], 8, 10)
            assert np.array_equal(res.topk(t).ids, single.topk.ids)


# ---- GPU schedulers ----------------------------------------
def test_group_microbatches_gpu_golden(orc, laiv):
    # acceptance.cpp:408-417 fixture: 256 x 768 queries, m = 4
    from common import golden, sha

    g = golden("sched.npz")
    q = orc.random_matrix(256, 768, 717)
    assert sha(q) == str(g["group_sha"])
    cen = laiv.synth_centroids(0, 16, 768)
    vecs, ids = laiv.synth_lists(0, cen, 2, 0.05)
    ix = laiv.IvfIndex(cen, vecs, ids, np.arange(0, 33, 2, dtype=np.uint64),
                       laiv.Metric.InnerProduct)
    dev = laiv.Device(ix, 1 << 20)
    got = laiv.group_microbatches_gpu(dev, q, 4)
    want = laiv.group_microbatches(q, 4)
    assert [b.queries for b in got] == [b.queries for b in want]
    ref = orc.group_microbatches(q, 4)
    assert [b.queries for b in got] == [list(b) for b in ref]


@pytest.mark.parametrize("n,m,d", [(1, 4, 8), (5, 3, 8), (37, 4, 16), (300, 7, 64),
                                   (1000, 4, 32), (64, 1, 8)])
def test_group_microbatches_gpu_matches_host(laiv, n, m, d):
    rng = np.random.default_rng(n * 31 + m)
    q = rng.standard_normal((n, d)).astype(np.float32)
    if n >= 37:  # exact distance ties: duplicated rows
        q[n // 2: n // 2 + 5] = q[3]
    cen = rng.standard_normal((8, d)).astype(np.float32)
    ix = laiv.IvfIndex(cen, cen.copy(), np.arange(8, dtype=np.uint64),
                       np.arange(9, dtype=np.uint64), laiv.Metric.L2)
    dev = laiv.Device(ix, 1 << 20)
    got = laiv.group_microbatches_gpu(dev, q, m)
    want = laiv.group_microbatches(q, m)
    assert [b.queries for b in got] == [b.queries for b in want]


@pytest.mark.parametrize("n,m,d", [(8193, 4, 16), (12000, 3, 64), (9000, 1, 8)])
def test_group_microbatches_gpu_streaming(laiv, n, m, d):
    """n above the one-CTA kernel's 8192: the persistent streaming grouping
    (no n x n matrix) equals the host scheduler bit for bit."""
    rng = np.random.default_rng(n + m)
    q = rng.standard_normal((n, d)).astype(np.float32)
    q[n // 3: n // 3 + 7] = q[11]  # exact ties
    cen = rng.standard_normal((8, d)).astype(np.float32)
    ix = laiv.IvfIndex(cen, cen.copy(), np.arange(8, dtype=np.uint64),
                       np.arange(9, dtype=np.uint64), laiv.Metric.L2)
    dev = laiv.Device(ix, 1 << 20)
    got = laiv.group_microbatches_gpu(dev, q, m)
    want = laiv.group_microbatches(q, m)
    assert [b.queries for b in got] == [b.queries for b in want]
    # and the smaller path still works on the same context afterwards
    got = laiv.group_microbatches_gpu(dev, q[:300], m)
    assert [b.queries for b in got] == [b.queries for b in laiv.group_microbatches(q[:300], m)]


@pytest.mark.parametrize("nw", [1, 2, 3, 8])
def test_schedule_matches_oracle(orc, laiv, nw):
    from paper_2502_20969_b200 import shard

    rng = np.random.default_rng(nw)
    nc, d, nq, L = 64, 16, 40, 6
    cen = orc.random_matrix(nc, d, 5)
    queries = orc.random_matrix(nq, d, 6)
    ix = laiv.IvfIndex(cen, cen.copy(), np.arange(nc, dtype=np.uint64),
                       np.arange(nc + 1, dtype=np.uint64), laiv.Metric.L2)
    dev = laiv.Device(ix, 1 << 20)
    resident = (rng.random((nw, nc)) < 0.3).astype(np.uint8)
    batches, assign, ov = laiv.schedule(dev, queries, 4, L, resident)
    want_b = laiv.group_microbatches(queries, 4)
    assert [b.queries for b in batches] == [b.queries for b in want_b]
    probes = np.array([orc.coarse_probe(cen, 1, qv, L) for qv in queries])
    want_ov = shard.overlap_matrix(shard.probe_union_masks(probes, want_b, nc), resident)
    assert np.array_equal(ov, want_ov)
    want = orc.assign_cache_aware([b.queries for b in want_b], resident, cen, 1, queries, L)
    assert assign == list(want)


def test_batch_single_query_and_fetch_metrics(orc, laiv):
    # a batch of one, and the fetch path's accounting under both metrics
    cen, vecs, ids, off, qi, qo, g = planted_data()
    for metric in (laiv.Metric.InnerProduct, laiv.Metric.L2):
        ix = laiv.IvfIndex(cen, vecs, ids, off, metric)
        dev = laiv.Device(ix, BIG, miss_fetch="all", fetch_chunk_mb=2)
        set_residency(dev, np.arange(64) % 4 == 0)
        res, tm = laiv.hybrid_search_batch(dev, qo[:1], 24, 10)
        single, _ = laiv.hybrid_search(dev, qo[0], 24, 10)
        assert np.array_equal(res.topk(0).ids, single.topk.ids)
        assert np.array_equal(res.topk(0).scores, single.topk.scores)
        want = orc.ivf_search(cen, vecs, ids, off, int(metric), qo[0], 24, 10)
        assert_topk_parity(int(metric), res.topk(0).ids, res.topk(0).scores, *want)
        assert tm.fetched_lists + tm.cpu_lists == 24 - int(res.nfast[0])


@pytest.mark.parametrize("name,metric", [("l2", L2), ("ip", IP)])
def test_microbatches_match_single(orc, laiv, name, metric):
    # micro-batches of 2-4 queries (the C4 micro-batch size): the batch path
    # must equal the single-query path under every residency and k
    cen, vecs, ids, off, qi, qo, g = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
    dev = laiv.Device(ix, BIG)
    rng = np.random.default_rng(5)
    for frac in (0.0, 1.0, 0.5):
        set_residency(dev, (rng.random(64) < frac).astype(np.uint8))
        for nq in (2, 3, 4):
            for L, k in ((8, 10), (32, 32), (16, 33), (64, 1)):
                sel = rng.choice(40, nq, replace=False)
                res, timing = laiv.hybrid_search_batch(dev, qo[sel], L, k)
                for i, t in enumerate(sel):
                    single, _ = laiv.hybrid_search(dev, qo[t], L, k)
                    got = res.topk(i)
                    assert np.array_equal(got.ids, single.topk.ids), (nq, L, k, t)
                    assert np.array_equal(got.scores, single.topk.scores), (nq, L, k, t)
                    assert res.nfast[i] == len(single.fast_clusters)
                    want = orc.ivf_search(cen, vecs, ids, off, metric, qo[t], L, k)
                    assert_topk_parity(metric, got.ids, got.scores, *want)
                assert timing.scanned_vectors == 300 * int(res.nfast.sum())
