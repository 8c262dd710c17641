"""List-major batched scan on the tensor cores (listscan.cu).

A batch's resident lists are read once per group of 16 queries probing them
and scored with tcgen05 tf32 MMAs; error bounds keep every possible top-k
member, which is then re-scored with the reference's fp64 arithmetic
(vectorstore.cpp:93-115) and ranked on (score, id) (vectorstore.hpp:34-39).
The batch result must equal the per-query scan's bit for bit and meet the
§8c rule against the C oracle, under any residency, list length (partial
row-blocks, multi-chunk lists, empty lists), query sharing (one to many
groups per list), d not a multiple of the 32-float k-block, both metrics.
"""
import numpy as np
import pytest

from common import IP, L2, assert_topk_parity, planted_data

pytestmark = pytest.mark.gpu
BIG = 1 << 34


def set_residency(dev, mask):
    dev.store.clear()
    for c in np.nonzero(mask)[0]:
        dev.store.insert(int(c))


def both_paths(laiv, dev, Q, L, k, monkeypatch):
    monkeypatch.setenv("LAIVG_LIST_SCAN", "0")
    base, _ = laiv.hybrid_search_batch(dev, Q, L, k)
    r0, f0, _ = dev.list_scan_stats()
    monkeypatch.setenv("LAIVG_LIST_SCAN", "1")
    got, timing = laiv.hybrid_search_batch(dev, Q, L, k)
    r1, f1, _ = dev.list_scan_stats()
    monkeypatch.delenv("LAIVG_LIST_SCAN")
    return base, got, timing, r1 - r0, f1 - f0


def assert_same(base, got, nq):
    for t in range(nq):
        a, b = base.topk(t), got.topk(t)
        assert np.array_equal(a.ids, b.ids), t
        assert np.array_equal(a.scores, b.scores), t
    assert np.array_equal(base.nfast, got.nfast)


@pytest.fixture(params=[16, 32], ids=["g16", "g32"])
def group(request, monkeypatch):
    """Queries per work item (UMMA N): 16, or 32 for heavily shared lists."""
    monkeypatch.setenv("LAIVG_LIST_SCAN_N", str(request.param))
    return request.param


@pytest.mark.parametrize("metric", [IP, L2])
@pytest.mark.parametrize("k", [1, 10, 32, 64])
def test_list_scan_planted(orc, laiv, monkeypatch, group, metric, k):
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
    dev = laiv.Device(ix, BIG, miss_fetch="off")
    rng = np.random.default_rng(5 + k)
    for frac, L in ((1.0, 8), (0.5, 16), (1.0, 64)):
        set_residency(dev, (rng.random(64) < frac).astype(np.uint8))
        base, got, _, runs, fb = both_paths(laiv, dev, qo, L, k, monkeypatch)
        assert runs == 1 and fb == 0
        assert_same(base, got, len(qo))
        for t in range(0, len(qo), 4):
            want = orc.ivf_search(cen, vecs, ids, off, metric, qo[t], L, k)
            assert_topk_parity(metric, got.topk(t).ids, got.topk(t).scores, *want)


@pytest.mark.parametrize("metric", [IP, L2])
def test_list_scan_shapes(orc, laiv, monkeypatch, group, metric):
    # ragged lists: empty, shorter than one row-block, multi-chunk (> 1024
    # rows); d = 100 (the last k-block is partial); 200 queries on 24 lists
    # (many 16-query groups per list)
    rng = np.random.default_rng(11)
    d, nc = 100, 24
    lens = rng.integers(0, 2600, nc)
    lens[3] = 0
    lens[5] = 1
    lens[7] = 127
    lens[8] = 129
    lens[9] = 1024
    lens[10] = 1025
    off = np.zeros(nc + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    n = int(off[-1])
    cen = rng.standard_normal((nc, d)).astype(np.float32)
    lab = np.repeat(np.arange(nc), lens)
    vecs = (cen[lab] + 0.3 * rng.standard_normal((n, d))).astype(np.float32)
    ids = rng.permutation(n).astype(np.uint64) * 3 + 7
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
    dev = laiv.Device(ix, BIG, miss_fetch="off")
    Q = (cen[rng.integers(0, nc, 200)] + 0.3 * rng.standard_normal((200, d))).astype(np.float32)
    for frac, L, k in ((1.0, 6, 10), (0.6, 24, 5), (1.0, 3, 32)):
        set_residency(dev, (rng.random(nc) < frac).astype(np.uint8))
        base, got, _, runs, fb = both_paths(laiv, dev, Q, L, k, monkeypatch)
        assert runs == 1 and fb == 0
        assert_same(base, got, len(Q))
        for t in range(0, len(Q), 25):
            want = orc.ivf_search(cen, vecs, ids, off, metric, Q[t], L, k)
            assert_topk_parity(metric, got.topk(t).ids, got.topk(t).scores, *want)


def test_list_scan_ties_fall_back(orc, laiv, monkeypatch, group):
    # every member of a list equal: all scores tie, the candidate buffers
    # overflow, the batch is re-run on the per-query scan (same answer)
    d, nc, per = 64, 8, 700
    rng = np.random.default_rng(2)
    cen = rng.standard_normal((nc, d)).astype(np.float32)
    vecs = np.repeat(cen, per, axis=0)
    ids = rng.permutation(nc * per).astype(np.uint64)
    off = np.arange(0, nc * per + 1, per, dtype=np.uint64)
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
    dev = laiv.Device(ix, BIG, miss_fetch="off")
    set_residency(dev, np.ones(nc, np.uint8))
    Q = rng.standard_normal((40, d)).astype(np.float32)
    base, got, _, runs, fb = both_paths(laiv, dev, Q, 4, 10, monkeypatch)
    assert runs == 1 and fb == 1
    assert_same(base, got, len(Q))
    want = orc.ivf_search(cen, vecs, ids, off, IP, Q[0], 4, 10)
    assert_topk_parity(IP, got.topk(0).ids, got.topk(0).scores, *want, exact=True)


def test_list_scan_with_misses_and_fetch(orc, laiv, monkeypatch):
    # the list scan covers the hits; misses go to the host or the runtime
    # fetch as before, and the merge is unchanged
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    for fetch in ("off", "all"):
        ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
        dev = laiv.Device(ix, BIG, miss_fetch=fetch, fetch_chunk_mb=3)
        set_residency(dev, (np.arange(64) % 3 == 0).astype(np.uint8))
        base, got, timing, runs, fb = both_paths(laiv, dev, qo, 16, 10, monkeypatch)
        assert runs == 1 and fb == 0
        assert_same(base, got, len(qo))
        for t in range(0, len(qo), 5):
            want = orc.ivf_search(cen, vecs, ids, off, IP, qo[t], 16, 10)
            assert_topk_parity(IP, got.topk(t).ids, got.topk(t).scores, *want)


def test_list_scan_unsupported_k_uses_per_query_scan(laiv, monkeypatch):
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
    dev = laiv.Device(ix, BIG, miss_fetch="off")
    set_residency(dev, np.ones(64, np.uint8))
    base, got, _, runs, fb = both_paths(laiv, dev, qo, 8, 100, monkeypatch)
    assert runs == 0 and fb == 0
    assert_same(base, got, len(qo))


def test_list_scan_auto_policy(laiv, monkeypatch):
    # auto: the list scan once the batches' queries per resident list reach
    # the threshold (EMA over batches)
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
    dev = laiv.Device(ix, BIG, miss_fetch="off")
    set_residency(dev, np.ones(64, np.uint8))
    monkeypatch.delenv("LAIVG_LIST_SCAN", raising=False)
    monkeypatch.setenv("LAIVG_LIST_SCAN_QPL", "4")
    laiv.hybrid_search_batch(dev, qo[:6], 32, 10)   # prior 6 x 32 / 64 = 3 < 4
    r, f, qpl = dev.list_scan_stats()
    assert r == 0 and qpl > 1
    laiv.hybrid_search_batch(dev, qo, 32, 10)       # EMA of 6 and 40 queries
    r, f, qpl = dev.list_scan_stats()
    assert qpl > 4
    laiv.hybrid_search_batch(dev, qo, 32, 10)
    r, f, _ = dev.list_scan_stats()
    assert r >= 1 and f == 0
    monkeypatch.setenv("LAIVG_LIST_SCAN_QPL", "1000")
    laiv.hybrid_search_batch(dev, qo, 32, 10)
    assert dev.list_scan_stats()[0] == r
    # a fresh context decides its first batch on the prior nq * L / nc
    dev2 = laiv.Device(ix, BIG, miss_fetch="off")
    set_residency(dev2, np.ones(64, np.uint8))
    monkeypatch.setenv("LAIVG_LIST_SCAN_QPL", "4")
    laiv.hybrid_search_batch(dev2, qo, 32, 10)      # prior 40 x 32 / 64 = 20
    assert dev2.list_scan_stats()[0] == 1


def test_list_scan_in_fp32_accumulation_contexts(orc, laiv, monkeypatch):
    # a context in fp32 + re-score mode: the list scan's exact answer equals
    # the per-query scan's (whose survivors are re-scored in fp64)
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    for metric in (IP, L2):
        ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
        dev = laiv.Device(ix, BIG, miss_fetch="off", acc_fp64=False)
        set_residency(dev, np.ones(64, np.uint8))
        base, got, _, runs, fb = both_paths(laiv, dev, qo, 16, 10, monkeypatch)
        assert runs == 1 and fb == 0
        assert_same(base, got, len(qo))
        for t in range(0, len(qo), 8):
            want = orc.ivf_search(cen, vecs, ids, off, metric, qo[t], 16, 10)
            assert_topk_parity(metric, got.topk(t).ids, got.topk(t).scores, *want)


@pytest.mark.parametrize("chunk", [128, 384, 4096])
def test_list_scan_chunk_lengths(orc, laiv, monkeypatch, chunk):
    # rows per work item from one row-block to whole lists: same answers
    rng = np.random.default_rng(23)
    d, nc = 64, 12
    lens = rng.integers(0, 3000, nc)
    lens[2] = 0
    lens[4] = 129
    off = np.zeros(nc + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    n = int(off[-1])
    cen = rng.standard_normal((nc, d)).astype(np.float32)
    vecs = (cen[np.repeat(np.arange(nc), lens)] +
            0.3 * rng.standard_normal((n, d))).astype(np.float32)
    ids = rng.permutation(n).astype(np.uint64)
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
    dev = laiv.Device(ix, BIG, miss_fetch="off")
    set_residency(dev, np.ones(nc, np.uint8))
    Q = (cen[rng.integers(0, nc, 60)] + 0.3 * rng.standard_normal((60, d))).astype(np.float32)
    monkeypatch.setenv("LAIVG_LIST_SCAN_CHUNK", str(chunk))
    base, got, _, runs, fb = both_paths(laiv, dev, Q, 5, 10, monkeypatch)
    assert runs == 1 and fb == 0
    assert_same(base, got, len(Q))
    for t in range(0, len(Q), 10):
        want = orc.ivf_search(cen, vecs, ids, off, IP, Q[t], 5, 10)
        assert_topk_parity(IP, got.topk(t).ids, got.topk(t).scores, *want)
