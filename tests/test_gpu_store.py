"""Tiered store = the GPU cluster cache; lookahead prefetch; hotness policy.

Known answers from the reference's own tests (test_tiered.cpp, test_cache.cpp,
the hotness.json scripts recorded from the reference) run against the device
store, plus device-only behaviour (window kernel, measured overlap,
compaction keeps search results exact).
"""
import numpy as np
import pytest

from common import IP, L2, Case, assert_topk_parity, golden, hybrid_d8_case, planted_data

pytestmark = pytest.mark.gpu
KMEMBER = 12  # 4 * 1 + 8 bytes (test_tiered.cpp:23)


def fixture_1d(laiv):
    # test_tiered.cpp:21-46: clusters of 5, 3, 4 members at 0, 1, 2
    cen = np.array([[0.0], [1.0], [2.0]], np.float32)
    sizes = [5, 3, 4]
    vecs, ids = [], []
    i = 0
    for c, n in enumerate(sizes):
        for j in range(n):
            vecs.append([c + 0.01 * j])
            ids.append(i)
            i += 1
    off = np.array([0, 5, 8, 12], np.uint64)
    ix = laiv.IvfIndex(cen, np.array(vecs, np.float32), np.array(ids, np.uint64), off,
                       laiv.Metric.L2)
    return ix


Q = np.array([-1.0], np.float32)


def test_plan_known_answers(laiv):
    ix = fixture_1d(laiv)
    dev = laiv.Device(ix, 1 << 20)
    p = laiv.plan_prefetch(dev, Q, 8 * KMEMBER)
    assert (p.clusters, p.planned_bytes, p.skipped) == ([0, 1], 8 * KMEMBER, [2])
    p = laiv.plan_prefetch(dev, Q, 7 * KMEMBER)
    assert (p.clusters, p.planned_bytes, p.skipped) == ([0], 5 * KMEMBER, [1, 2])
    p = laiv.plan_prefetch(dev, Q, 4 * KMEMBER)
    assert (p.clusters, p.skipped) == ([1], [0, 2])
    p = laiv.plan_prefetch(dev, Q, 0)
    assert (p.clusters, p.planned_bytes, p.skipped) == ([], 0, [0, 1, 2])
    dev.store.insert(0, laiv.Residency.Cached)
    assert laiv.plan_prefetch(dev, Q, 100 * KMEMBER).clusters == [1, 2]


def test_execute_prefetch_modes(laiv):
    ix = fixture_1d(laiv)
    dev = laiv.Device(ix, 1 << 20)
    chan = laiv.TransferChannel(12.0, laiv.ChannelMode.SimulatedClock)
    rep = laiv.execute_prefetch(dev, laiv.PrefetchPlan(), chan, 0.0)
    assert rep.t_p == 0.0 and dev.store.resident_count() == 0
    plan = laiv.plan_prefetch(dev, Q, 8 * KMEMBER)
    rep = laiv.execute_prefetch(dev, plan, chan, 0.0)
    assert rep.t_p == float(8 * KMEMBER) / 12.0 and rep.bytes == 8 * KMEMBER
    assert dev.store.contains(0) and dev.store.contains(1) and not dev.store.contains(2)
    assert dev.store.used_bytes() == 8 * KMEMBER
    assert dev.store.resident()[0][0] == laiv.Residency.Prefetched
    # capacity violations throw std::runtime_error
    tiny = laiv.Device(ix, 3 * KMEMBER)
    with pytest.raises(RuntimeError):
        laiv.execute_prefetch(tiny, laiv.PrefetchPlan([0], 60, []), chan, 0.0)
    # device mode: copies on the copy stream, window kernel on the compute stream
    dev.store.clear()
    plan = laiv.plan_prefetch(dev, Q, 12 * KMEMBER)
    rep = laiv.execute_prefetch(dev, plan, laiv.TransferChannel(1e9, laiv.ChannelMode.Device),
                                0.01)
    assert rep.transferred == [0, 1, 2] and dev.store.resident_count() == 3
    assert 0.009 <= rep.window_s <= 0.05
    assert rep.overshoot_s >= 0.0
    res, _ = laiv.hybrid_search(dev, Q, 3, 12)
    assert res.hit_rate == 1.0 and len(res.topk.entries) == 12


def test_incremental_prefetch(laiv):
    ix = fixture_1d(laiv)
    dev = laiv.Device(ix, 1 << 20)
    chan = laiv.TransferChannel(1e6, laiv.ChannelMode.SimulatedClock)
    r1 = laiv.incremental_prefetch(dev, Q, 12 * KMEMBER, chan)
    assert len(r1.transferred) == 3
    r2 = laiv.incremental_prefetch(dev, Q, 12 * KMEMBER, chan)
    assert r2.transferred == [] and r2.t_p == 0.0
    laiv.incremental_prefetch(dev, np.array([5.0], np.float32), 12 * KMEMBER, chan)
    assert dev.store.resident_count() == 3
    dev.store.clear()
    dev.store.insert(0)
    rep = laiv.incremental_prefetch(dev, Q, 7 * KMEMBER, chan)
    assert rep.transferred == [1, 2] and rep.bytes == 7 * KMEMBER


def test_store_errors_and_accounting(laiv):
    ix = fixture_1d(laiv)
    dev = laiv.Device(ix, 100)
    dev.store.insert(1)  # 36 bytes
    with pytest.raises(laiv.LogicError):
        dev.store.insert(1)
    with pytest.raises(RuntimeError):
        dev.store.insert(0)  # 60 + 36 fits, then 2 (48) would not
        dev.store.insert(2)
    with pytest.raises(laiv.LogicError):
        dev.store.evict(2)
    rng = np.random.default_rng(71)
    dev2 = laiv.Device(ix, 1 << 20)
    for _ in range(300):
        c = int(rng.integers(0, 3))
        if dev2.store.contains(c):
            dev2.store.evict(c)
        else:
            dev2.store.insert(c, laiv.Residency(int(rng.integers(0, 2))))
        assert dev2.store.recompute_used_bytes() == dev2.store.used_bytes()
        assert dev2.store.used_bytes() <= dev2.store.capacity_bytes()


def test_fragmentation_and_compaction_keep_results_exact(orc, laiv):
    # ragged lists in a slab sized to force holes and compaction
    rng = np.random.default_rng(11)
    nc, d = 32, 256
    sizes = rng.integers(50, 500, nc)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint64)
    n = int(off[-1])
    vecs = rng.standard_normal((n, d)).astype(np.float32)
    ids = np.arange(n, dtype=np.uint64)
    cen = rng.standard_normal((nc, d)).astype(np.float32)
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.L2)
    cap = int(sizes.sum() * 0.45) * (4 * d + 8)
    dev = laiv.Device(ix, cap)
    for step in range(200):
        c = int(rng.integers(0, nc))
        if dev.store.contains(c):
            dev.store.evict(c)
        elif dev.store.free_bytes() >= ix.cluster_bytes(c):
            dev.store.insert(c)
        if step % 20 == 0:
            q = rng.standard_normal(d).astype(np.float32)
            res, _ = laiv.hybrid_search(dev, q, 12, 10)
            want = orc.ivf_search(cen, vecs, ids, off, L2, q, 12, 10)
            assert_topk_parity(L2, res.topk.ids, res.topk.scores, *want)
    dev.store.compact()
    q = rng.standard_normal(d).astype(np.float32)
    res, _ = laiv.hybrid_search(dev, q, 32, 10)
    want = orc.ivf_search(cen, vecs, ids, off, L2, q, 32, 10)
    assert_topk_parity(L2, res.topk.ids, res.topk.scores, *want)


def test_hotness_scripts_on_device_store(orc, laiv):
    case, _, _ = hybrid_d8_case(orc, "l2")
    ix = laiv.IvfIndex(case.centroids, case.vecs, case.ids, case.list_off, laiv.Metric.L2)
    for s in golden("hotness.json"):
        h_init, h_inc, decay, frac = s["params"]
        dev = laiv.Device(ix, s["cap"])
        hot = laiv.HotnessTable(laiv.CacheParams(h_init, h_inc, decay, frac))
        for (ins, used), want in zip(s["ops"], s["evicted"]):
            for c in ins:
                dev.store.insert(c)
                hot.on_fetch(c)
            hot.end_of_round(set(used))
            assert hot.evict_to_fraction(dev) == want
            assert all(t == laiv.Residency.Cached for t, _ in dev.store.resident().values())
        final = {c: hot.hotness(c) for c in dev.store.resident()}
        assert final == {int(k): v for k, v in s["final"].items()}


def test_window_kernel(laiv):
    ix = fixture_1d(laiv)
    dev = laiv.Device(ix, 1 << 20)
    for w in (0.001, 0.02):
        got = dev.window(w)
        assert w * 0.95 <= got <= w + 0.01


def test_device_prefetch_overlap_planted(laiv):
    # lookahead: the copy of the planned lists hides behind the window
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
    dev = laiv.Device(ix, 64 * 300 * (4 * 768 + 8))
    chan = laiv.TransferChannel(50e9, laiv.ChannelMode.Device)
    plan = laiv.plan_prefetch(dev, qi[0], 16 * 300 * (4 * 768 + 8))
    assert len(plan.clusters) == 16
    rep = laiv.execute_prefetch(dev, plan, chan, 0.05)
    assert rep.overshoot_s == 0.0  # 14.8 MB at tens of GB/s is far below 50 ms
    assert rep.h2d_gbps > 5.0
    res, t = laiv.hybrid_search(dev, qo[0], 8, 10)
    assert res.hit_rate > 0.5
    assert t.t_scan > 0.0 and t.scanned_bytes == len(res.fast_clusters) * 300 * (4 * 768 + 8)
