"""The fused single-query kernel (query fetch -> coarse scores -> top-L ->
residency split -> TMA scan in one cooperative launch) against the
multi-kernel chain it replaces and against the C oracle.

Both paths run the same per-term fp64 arithmetic, so every result (ids,
scores, probe, fast/slow split) must be bit-identical between them; the
oracle checks the §8c rule (ivf.cpp:269-343, tiered.cpp:148-185).
"""
import numpy as np
import pytest

from common import IP, L2, assert_topk_parity, planted_data

pytestmark = pytest.mark.gpu
BIG = 1 << 30


def pair(laiv, cen, vecs, ids, off, metric, **kw):
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
    fused = laiv.Device(ix, BIG, single_query="fused", **kw)
    chain = laiv.Device(ix, BIG, single_query="chain", **kw)
    return ix, fused, chain


def set_res(devs, mask):
    for dev in devs:
        dev.store.clear()
        for c in np.nonzero(mask)[0]:
            dev.store.insert(int(c))


def same(a, b):
    (ra, ta), (rb, tb) = a, b
    assert np.array_equal(ra.topk.ids, rb.topk.ids), (ra.topk.ids, rb.topk.ids)
    assert np.array_equal(ra.topk.scores, rb.topk.scores)
    assert ra.fast_clusters == rb.fast_clusters
    assert ra.slow_clusters == rb.slow_clusters
    assert ta.t_kernel > 0.0 and tb.t_kernel == 0.0
    assert ta.scanned_vectors == tb.scanned_vectors


@pytest.mark.parametrize("metric", [IP, L2])
@pytest.mark.parametrize("acc_fp64", [True, False])
def test_fused_equals_chain_planted(orc, laiv, metric, acc_fp64):
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    ix, fused, chain = pair(laiv, cen, vecs, ids, off, metric, acc_fp64=acc_fp64)
    rng = np.random.default_rng(21 + metric)
    for t in range(40):
        set_res((fused, chain), (rng.random(64) < rng.random()).astype(np.uint8))
        L = int(rng.choice([1, 2, 7, 8, 31, 63, 64, 100]))
        k = int(rng.choice([1, 10, 32, 33, 100, 239 if acc_fp64 else 200, 256]))
        a = laiv.hybrid_search(fused, qo[t], L, k)
        b = laiv.hybrid_search(chain, qo[t], L, k)
        same(a, b)
        want = orc.ivf_search(cen, vecs, ids, off, metric, qo[t], min(L, 64), k)
        assert_topk_parity(metric, a[0].topk.ids, a[0].topk.scores, *want)


@pytest.mark.parametrize("metric", [IP, L2])
def test_fused_probe_ties_and_all_equal(orc, laiv, metric):
    # duplicated centroids give exactly equal coarse keys: the selection must
    # take the smaller cluster id at the boundary (radix select's tie path),
    # including the case where every key is equal
    rng = np.random.default_rng(5)
    d, nc, per = 64, 96, 40
    base = rng.standard_normal((nc // 8, d)).astype(np.float32)
    cen = np.repeat(base, 8, axis=0)
    vecs = rng.standard_normal((nc * per, d)).astype(np.float32)
    ids = rng.permutation(nc * per).astype(np.uint64)
    off = np.arange(0, nc * per + 1, per, dtype=np.uint64)
    ix, fused, chain = pair(laiv, cen, vecs, ids, off, metric)
    set_res((fused, chain), np.ones(nc, np.uint8))
    for t in range(12):
        q = rng.standard_normal(d).astype(np.float32)
        L = int(rng.integers(1, nc + 1))
        a = laiv.hybrid_search(fused, q, L, 10)
        b = laiv.hybrid_search(chain, q, L, 10)
        same(a, b)
        assert a[0].fast_clusters == [int(c) for c in orc.coarse_probe(cen, metric, q, L)]
    # every centroid identical: the probe is clusters 0..L-1
    cen1 = np.repeat(base[:1], nc, axis=0)
    ix1, f1, c1 = pair(laiv, cen1, vecs, ids, off, metric)
    set_res((f1, c1), np.ones(nc, np.uint8))
    q = rng.standard_normal(d).astype(np.float32)
    for L in (1, 5, 95, 96, 500):
        a = laiv.hybrid_search(f1, q, L, 7)
        same(a, laiv.hybrid_search(c1, q, L, 7))
        assert a[0].fast_clusters == list(range(min(L, nc)))


def test_fused_empty_lists_and_no_resident(orc, laiv):
    rng = np.random.default_rng(8)
    d, nc = 768, 50
    sizes = rng.integers(0, 120, nc)
    sizes[[0, 5, 6, 49]] = 0
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint64)
    n = int(off[-1])
    vecs = rng.standard_normal((n, d)).astype(np.float32)
    ids = rng.permutation(5 * n)[:n].astype(np.uint64)
    cen = rng.standard_normal((nc, d)).astype(np.float32)
    for metric in (IP, L2):
        ix, fused, chain = pair(laiv, cen, vecs, ids, off, metric)
        for t, frac in enumerate([0.0, 0.3, 1.0, 0.7]):
            set_res((fused, chain), (rng.random(nc) < frac).astype(np.uint8))
            q = rng.standard_normal(d).astype(np.float32)
            for L, k in ((1, 5), (13, 40), (50, 256)):
                a = laiv.hybrid_search(fused, q, L, k)
                same(a, laiv.hybrid_search(chain, q, L, k))
                want = orc.ivf_search(cen, vecs, ids, off, metric, q, L, k)
                assert_topk_parity(metric, a[0].topk.ids, a[0].topk.scores, *want)
        # L <= 0: empty probe
        assert laiv.ivf_search(fused, q, 0, 5).entries == []


@pytest.mark.parametrize("miss_fetch", ["off", "auto", "all"])
def test_fused_staged_misses_every_path(orc, laiv, miss_fetch):
    # staged rows with a third of the lists missing: the misses go to the
    # host, to the runtime fetch ring (chunk scans after the fused kernel read
    # the query from dQ), or are split between them; every path is exact
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
    dev = laiv.Device(ix, BIG, miss_fetch=miss_fetch, fetch_chunk_mb=4)
    set_res((dev,), np.arange(64) % 3 != 0)
    dev.stage_queries(qo)
    for t in range(40):
        want = orc.ivf_search(cen, vecs, ids, off, IP, qo[t], 16, 10)
        i, s, n, tm = dev.hybrid_search_staged(t, 16, 10)
        assert tm.t_kernel > 0.0
        assert_topk_parity(IP, i, s, *want)
        res, _ = laiv.hybrid_search(dev, qo[t], 16, 10)
        assert_topk_parity(IP, res.topk.ids, res.topk.scores, *want)


def test_fused_staged_queries_and_repeats(laiv):
    # the staged-row entry (mapped slot) and back-to-back calls: the grid
    # barrier word and the probe sequence number carry across launches
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    ix, fused, chain = pair(laiv, cen, vecs, ids, off, IP)
    set_res((fused, chain), np.arange(64) % 3 != 0)
    fused.stage_queries(qo)
    chain.stage_queries(qo)
    for rep in range(3):
        for t in range(40):
            ia, sa, na, ta = fused.hybrid_search_staged(t, 16, 10)
            ib, sb, nb, tb = chain.hybrid_search_staged(t, 16, 10)
            assert np.array_equal(ia, ib) and np.array_equal(sa, sb) and na == nb
            assert ta.t_kernel > 0.0 and tb.t_kernel == 0.0
            c = laiv.hybrid_search(fused, qo[t], 16, 10)
            assert np.array_equal(c[0].topk.ids, ib)
            assert np.array_equal(c[0].topk.scores, sb)


def test_fused_large_nc_shapes(orc, laiv):
    # nc where the ranking spans many radix digits; nc whose keys no longer fit
    # the ring (the chain runs instead, same results)
    rng = np.random.default_rng(3)
    d = 768
    for nc in (4096, 16384):
        cen = rng.standard_normal((nc, d)).astype(np.float32)
        vecs = rng.standard_normal((nc * 2, d)).astype(np.float32)
        off = np.arange(0, 2 * nc + 1, 2, dtype=np.uint64)
        ids = np.arange(2 * nc, dtype=np.uint64)
        for metric in (IP, L2):
            ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
            fused = laiv.Device(ix, BIG, single_query="fused")
            chain = laiv.Device(ix, BIG, single_query="chain")
            set_res((fused, chain), (rng.random(nc) < 0.5).astype(np.uint8))
            for t in range(3):
                q = rng.standard_normal(d).astype(np.float32)
                L = int(rng.choice([1, 128, 1000]))
                a = laiv.hybrid_search(fused, q, L, 10)
                b = laiv.hybrid_search(chain, q, L, 10)
                assert np.array_equal(a[0].topk.ids, b[0].topk.ids)
                assert np.array_equal(a[0].topk.scores, b[0].topk.scores)
                assert a[0].fast_clusters == b[0].fast_clusters
                assert a[0].slow_clusters == b[0].slow_clusters
                probe = orc.coarse_probe(cen, metric, q, L)
                got = sorted(a[0].fast_clusters + a[0].slow_clusters)
                assert got == sorted(int(c) for c in probe)


def test_plain_call_without_timing(laiv):
    # laivg_hybrid_search with no timing struct (the library skips its event
    # queries) returns the same result; the cumulative link counters count
    # the call's host-link bytes (laivg_link_bytes)
    import ctypes as C

    from paper_2502_20969_b200._lib import CostModelC, check

    cen, vecs, ids, off, qi, qo, _ = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
    dev = laiv.Device(ix, BIG)
    set_res((dev,), np.arange(64) % 2)
    k, L = 10, 16
    e_ids = np.empty(k, np.uint64)
    e_sc = np.empty(k, np.float32)
    fast = np.empty(64, np.uint32)
    slow = np.empty(64, np.uint32)
    cnt, nf, ns, hr = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_double()
    cm = CostModelC(32e9, 1e-3, 1e-5, 1)
    h, d = C.c_uint64(), C.c_uint64()
    for t in range(6):
        q = np.ascontiguousarray(qo[t], np.float32)
        check(laiv.lib().laivg_link_bytes(dev.h, C.byref(h), C.byref(d)))
        h0, d0 = h.value, d.value
        check(laiv.lib().laivg_hybrid_search(dev.h, q.ctypes.data, L, k, C.byref(cm),
                                             e_ids.ctypes.data, e_sc.ctypes.data, C.byref(cnt),
                                             fast.ctypes.data, C.byref(nf), slow.ctypes.data,
                                             C.byref(ns), C.byref(hr), None))
        check(laiv.lib().laivg_link_bytes(dev.h, C.byref(h), C.byref(d)))
        assert h.value - h0 >= 768 * 4 and d.value > d0
        res, tm = laiv.hybrid_search(dev, q, L, k)
        assert np.array_equal(res.topk.ids, e_ids[: cnt.value])
        assert np.array_equal(res.topk.scores, e_sc[: cnt.value])
        assert res.fast_clusters == fast[: nf.value].tolist()
        assert tm.t_kernel > 0.0


@pytest.mark.parametrize("metric", [IP, L2])
def test_fused_odd_shapes(orc, laiv, metric):
    # odd nc (the key loader's tail), d = 764 (the generic consumer path, not
    # the d = 768 specialisation), k across the register top-k widths, a
    # probe capped by max_probe
    rng = np.random.default_rng(17 + metric)
    nc, d = 77, 764
    sizes = rng.integers(1, 90, nc)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint64)
    n = int(off[-1])
    vecs = rng.standard_normal((n, d)).astype(np.float32)
    ids = rng.permutation(3 * n)[:n].astype(np.uint64)
    cen = rng.standard_normal((nc, d)).astype(np.float32)
    ix, fused, chain = pair(laiv, cen, vecs, ids, off, metric, max_probe=40)
    set_res((fused, chain), (rng.random(nc) < 0.6).astype(np.uint8))
    for t in range(10):
        q = rng.standard_normal(d).astype(np.float32)
        L = int(rng.choice([1, 9, 40]))
        k = int(rng.choice([1, 31, 33, 64, 65, 128, 129, 256]))
        a = laiv.hybrid_search(fused, q, L, k)
        same(a, laiv.hybrid_search(chain, q, L, k))
        want = orc.ivf_search(cen, vecs, ids, off, metric, q, L, k)
        assert_topk_parity(metric, a[0].topk.ids, a[0].topk.scores, *want)
