"""Parity at BASELINE scale, through the C ABI, against
the UNMODIFIED reference core (`laiv::ivf_search`, oracle/_ref/libref.so,
/root/reference/proj/core/src/ivf.cpp:345-349) on the same box and inputs.

* C1 = 1M x 768, 1024 lists, nprobe 32, k 10: 1000 queries per metric (IP,
  L2), under fp64 accumulation and under fp32 accumulation + the exact fp64
  re-score, with every list resident (pure GPU path) and with a 10% cache
  filled by the lookahead prefetch of q_in (hybrid path, misses on the GPU
  ring or the host), plus the batched path.
* C2 = 10M x 768, 4096 lists, nprobe 128, k 10: 200 queries per metric,
  lookahead prefetch into a 10% cache then hybrid_search (the bench step),
  both accumulation modes; coarse probes of 100 queries vs the reference.
* Batched C2: one 256-query batch at nprobe 256 (tensor-core coarse
  quantizer, batched scan, runtime fetch of misses through the HBM ring).

Comparison: bit-for-bit (ids and f32 scores); the SURVEY §8c rule is applied
only where the reference's adjacent scores are within 1e-5 relative. Match
counts are printed (`-s`) and asserted.
"""
import os

import numpy as np
import pytest

from common import assert_topk_parity

pytestmark = pytest.mark.gpu

SEED, QSEED, SPREAD, SIGMA = 0, 1, 0.05, 0.008
THREADS = os.cpu_count() or 1


def _need_ref():
    from oracle.oracle import RefLib

    if not RefLib.available():
        pytest.skip("oracle/_ref/libref.so not built")
    return RefLib()


def _store(laiv, nc, per, d=768):
    cen = laiv.synth_centroids(SEED, nc, d)
    n = nc * per
    vecs = laiv.pinned_empty((n, d), np.float32)
    ids = np.empty(n, np.uint64)
    laiv.synth_lists(SEED, cen, per, SPREAD, vecs=vecs, ids=ids)
    off = np.arange(0, n + 1, per, dtype=np.uint64)
    return cen, vecs, ids, off


def _compare(tag, metric, got, want):
    """got / want: lists of (ids, scores). Asserts the §8c rule on every
    query; returns the bit-identical count (printed)."""
    exact = 0
    for (gi, gs), (wi, ws) in zip(got, want):
        gi, gs = np.asarray(gi, np.uint64), np.asarray(gs, np.float32)
        assert_topk_parity(metric, gi, gs, wi, ws)
        exact += bool(np.array_equal(gi, wi) and np.array_equal(gs, ws))
    print(f"[scale parity] {tag}: {exact}/{len(got)} bit-identical to laiv::ivf_search")
    return exact


class _C1:
    nc, per, L, k, nq = 1024, 977, 32, 10, 1000


@pytest.fixture(scope="module")
def c1(laiv):
    ref = _need_ref()
    cen, vecs, ids, off = _store(laiv, _C1.nc, _C1.per)
    qi, qo, _ = laiv.synth_queries(QSEED, vecs, _C1.nq, SIGMA)
    want = {}
    for metric in (0, 1):
        ri = ref.index(cen, vecs, ids, off, metric)
        wi, ws, _ = ri.search_many(qo, _C1.L, _C1.k, THREADS)
        want[metric] = list(zip(wi, ws))
        ri.close()
        del ri
    return cen, vecs, ids, off, qi, qo, want


@pytest.mark.parametrize("metric", [0, 1], ids=["ip", "l2"])
@pytest.mark.parametrize("acc_fp64", [True, False], ids=["fp64", "fp32"])
def test_c1_all_resident(laiv, c1, metric, acc_fp64):
    cen, vecs, ids, off, qi, qo, want = c1
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric), borrow=True, trust=True)
    dev = laiv.Device(ix, ix.total_payload_bytes(), acc_fp64=acc_fp64)
    for c in range(_C1.nc):
        dev.store.insert(c)
    got = []
    for t in range(_C1.nq):
        r = laiv.ivf_search(dev, qo[t], _C1.L, _C1.k)
        got.append((r.ids, r.scores))
    exact = _compare(f"C1 {'ip' if metric == 0 else 'l2'} acc={'fp64' if acc_fp64 else 'fp32'} "
                     "all resident", metric, got, want[metric])
    assert exact >= _C1.nq - 2  # fp64: identical arithmetic; near-ties only may differ
    dev.close()
    ix.close()


@pytest.mark.parametrize("metric", [0, 1], ids=["ip", "l2"])
@pytest.mark.parametrize("acc_fp64", [True, False], ids=["fp64", "fp32"])
def test_c1_lookahead_hybrid(laiv, c1, metric, acc_fp64):
    cen, vecs, ids, off, qi, qo, want = c1
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric), borrow=True, trust=True)
    member = 4 * 768 + 8
    cap = int(0.10 * _C1.nc) * _C1.per * member
    dev = laiv.Device(ix, cap, acc_fp64=acc_fp64)
    chan = laiv.TransferChannel(50e9, laiv.ChannelMode.Device)
    got, hits = [], 0
    for t in range(_C1.nq):
        dev.store.clear()
        plan = laiv.plan_prefetch(dev, qi[t], cap)
        laiv.execute_prefetch(dev, plan, chan, 0.0)
        res, _ = laiv.hybrid_search(dev, qo[t], _C1.L, _C1.k)
        hits += len(res.fast_clusters)
        got.append((res.topk.ids, res.topk.scores))
    exact = _compare(f"C1 {'ip' if metric == 0 else 'l2'} acc={'fp64' if acc_fp64 else 'fp32'} "
                     f"lookahead 10% cache (hit rate {hits / (_C1.nq * _C1.L):.2f})", metric,
                     got, want[metric])
    assert exact >= _C1.nq - 2
    dev.close()
    ix.close()


@pytest.mark.parametrize("metric", [0, 1], ids=["ip", "l2"])
def test_c1_batched(laiv, c1, metric):
    cen, vecs, ids, off, qi, qo, want = c1
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric), borrow=True, trust=True)
    member = 4 * 768 + 8
    cap = int(0.25 * _C1.nc) * _C1.per * member
    dev = laiv.Device(ix, cap, max_batch=64)
    chan = laiv.TransferChannel(50e9, laiv.ChannelMode.Device)
    got = []
    for b in range(0, _C1.nq, 64):
        sel = slice(b, min(b + 64, _C1.nq))
        n = sel.stop - sel.start
        dev.store.clear()
        laiv.prefetch_batch(dev, qi[sel], np.full(n, cap // n, np.uint64), chan, 0.0)
        res, _ = laiv.hybrid_search_batch(dev, qo[sel], _C1.L, _C1.k)
        got += [(res.ids[q, : res.counts[q]], res.scores[q, : res.counts[q]]) for q in range(n)]
    runs, fallbacks, qpl = dev.list_scan_stats()
    exact = _compare(f"C1 {'ip' if metric == 0 else 'l2'} batched (64/call, 25% cache; hits on "
                     f"the list-major scan in {runs} of {(_C1.nq + 63) // 64} batches, "
                     f"{qpl:.1f} queries per list)", metric, got, want[metric])
    assert exact >= _C1.nq - 2
    assert runs > 0 and fallbacks == 0
    dev.close()
    ix.close()


class _C2:
    nc, per, L, k, nq = 4096, 2442, 128, 10, 200


@pytest.fixture(scope="module")
def c2(laiv):
    ref = _need_ref()
    cen, vecs, ids, off = _store(laiv, _C2.nc, _C2.per)
    qi, qo, _ = laiv.synth_queries(QSEED, vecs, 256, SIGMA)
    return ref, cen, vecs, ids, off, qi, qo


@pytest.mark.parametrize("metric", [0, 1], ids=["ip", "l2"])
def test_c2_lookahead_and_batch(laiv, c2, metric):
    ref, cen, vecs, ids, off, qi, qo = c2
    name = "ip" if metric == 0 else "l2"
    ri = ref.index(cen, vecs, ids, off, metric)
    wi, ws, _ = ri.search_many(qo[: _C2.nq], _C2.L, _C2.k, THREADS)
    want = list(zip(wi, ws))
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric), borrow=True, trust=True)
    member = 4 * 768 + 8
    cap = int(0.10 * _C2.nc) * _C2.per * member
    chan = laiv.TransferChannel(50e9, laiv.ChannelMode.Device)

    # coarse probes: the GPU's fp64 ranking prefix vs laiv::coarse_probe
    dev = laiv.Device(ix, cap, max_batch=256)
    probes = laiv.coarse_probe(dev, qi[:100], _C2.L)
    same = sum(np.array_equal(probes[t], ri.coarse_probe(qi[t], _C2.L)) for t in range(100))
    print(f"[scale parity] C2 {name} coarse_probe: {same}/100 identical")
    assert same == 100

    # the bench step: lookahead prefetch of q_in into a 10% cache, then
    # hybrid_search of q_out, both accumulation modes
    for acc in (True, False):
        if not acc:
            dev.close()
            dev = laiv.Device(ix, cap, max_batch=256, acc_fp64=False)
        got = []
        for t in range(_C2.nq):
            dev.store.clear()
            plan = laiv.plan_prefetch(dev, qi[t], cap)
            laiv.execute_prefetch(dev, plan, chan, 0.0)
            res, _ = laiv.hybrid_search(dev, qo[t], _C2.L, _C2.k)
            got.append((res.topk.ids, res.topk.scores))
        exact = _compare(f"C2 {name} acc={'fp64' if acc else 'fp32'} lookahead 10% cache",
                         metric, got, want)
        assert exact >= _C2.nq - 1

    # one 256-query batch at nprobe 256: tensor-core coarse quantizer,
    # batched scan of the hits, misses through the runtime-fetch ring
    # (IP: adaptive GPU/host split; L2: every fetchable miss on the GPU)
    dev.close()
    dev = laiv.Device(ix, cap, max_batch=256, miss_fetch="auto" if metric == 0 else "all")
    wi2, ws2, _ = ri.search_many(qo, 256, _C2.k, THREADS)
    dev.store.clear()
    laiv.prefetch_batch(dev, qi, np.full(256, cap // 256, np.uint64), chan, 0.0)
    os.environ["LAIVG_LIST_SCAN"] = "0"  # hits on the per-query scan
    try:
        res, tm = laiv.hybrid_search_batch(dev, qo, 256, _C2.k)
    finally:
        os.environ.pop("LAIVG_LIST_SCAN", None)
    assert dev.list_scan_stats()[0] == 0
    got = [(res.ids[q, : res.counts[q]], res.scores[q, : res.counts[q]]) for q in range(256)]
    exact = _compare(f"C2 {name} batch 256 x nprobe 256 (fetched lists {tm.fetched_lists}, "
                     f"host lists {tm.cpu_lists})", metric, got, list(zip(wi2, ws2)))
    assert exact >= 255
    assert tm.fetched_lists > 0
    # the same batch with the hits on the list-major tensor-core scan
    os.environ["LAIVG_LIST_SCAN"] = "1"
    try:
        res2, _ = laiv.hybrid_search_batch(dev, qo, 256, _C2.k)
    finally:
        os.environ.pop("LAIVG_LIST_SCAN", None)
    assert dev.list_scan_stats()[0] == 1
    got2 = [(res2.ids[q, : res2.counts[q]], res2.scores[q, : res2.counts[q]]) for q in range(256)]
    exact2 = _compare(f"C2 {name} batch 256 x nprobe 256, list-major scan", metric, got2,
                      list(zip(wi2, ws2)))
    assert exact2 >= 255
    assert all(np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
               for a, b in zip(got, got2))
    dev.close()
    ix.close()
    ri.close()
