"""Peer-GPU cache hits: a miss of one context that another
context caches is copied out of that context's slab and scanned locally.

Results must not depend on where a list was scanned (hybrid == monolithic,
tiered.hpp:120-124); the epoch protocol must keep every published list intact
(quarantined evictions, no compaction) until the epoch closes. The peers here
share cuda:0 (one GPU per test box): in one process through
laivg_peer_attach_local, across two processes through CUDA IPC.
"""
import os
import socket

import numpy as np
import pytest

from common import assert_topk_parity, planted_data

pytestmark = pytest.mark.gpu
CB = 300 * (4 * 768 + 8)  # cluster bytes of the planted lists


def cache(dev, lists):
    dev.store.clear()
    for c in lists:
        dev.store.insert(int(c))


@pytest.mark.parametrize("metric", [0, 1])
def test_peer_hits_in_process(orc, laiv, metric):
    cen, vecs, ids, off, qi, qo, g = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
    a = laiv.Device(ix, 64 * CB, fetch_chunk_mb=2)
    b = laiv.Device(ix, 64 * CB)
    ref = laiv.Device(ix, 64 * CB, miss_fetch="off")
    cache(a, range(40, 48))
    cache(b, range(0, 32))
    cache(ref, range(40, 48))
    a.peer_attach(0, other=b)
    for dv in (a, b):
        dv.epoch_open()
    a.peer_publish(0, b.store_offsets())
    res, tm = laiv.hybrid_search_batch(a, qo, 16, 10)
    want, _ = laiv.hybrid_search_batch(ref, qo, 16, 10)
    assert np.array_equal(res.ids, want.ids) and np.array_equal(res.scores, want.scores)
    for t in range(0, 40, 7):
        w = orc.ivf_search(cen, vecs, ids, off, metric, qo[t], 16, 10)
        assert_topk_parity(metric, res.topk(t).ids, res.topk(t).scores, *w)
    assert tm.peer_lists > 0 and tm.peer_bytes == tm.peer_lists * 300 * 768 * 4
    for dv in (a, b):
        dv.epoch_close()
    # outside an epoch nothing is published
    with pytest.raises(laiv.LogicError):
        a.peer_publish(0, b.store_offsets())


def test_epoch_quarantine_keeps_published_lists(orc, laiv):
    cen, vecs, ids, off, qi, qo, g = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
    a = laiv.Device(ix, 64 * CB, fetch_chunk_mb=2)
    b = laiv.Device(ix, 12 * CB)
    cache(a, [])
    cache(b, range(0, 12))
    a.peer_attach(0, other=b)
    b.epoch_open()
    a.epoch_open()
    a.peer_publish(0, b.store_offsets())
    # b evicts everything it published and refills its slab with other lists:
    # the quarantined ranges must not be reused while the epoch is open
    for c in range(0, 12):
        b.store.evict(c)
    assert b.store.free_bytes() == 0  # quarantined bytes still count
    with pytest.raises(RuntimeError):
        b.store.insert(20)
    with pytest.raises(laiv.LogicError):
        b.store.compact()
    res, tm = laiv.hybrid_search_batch(a, qo, 64, 10)
    assert tm.peer_lists == 12
    for t in range(40):
        w = orc.ivf_search(cen, vecs, ids, off, 0, qo[t], 64, 10)
        assert_topk_parity(0, res.topk(t).ids, res.topk(t).scores, *w, exact=True)
    a.epoch_close()
    b.epoch_close()
    assert b.store.free_bytes() == 12 * CB
    for c in range(20, 32):
        b.store.insert(c)
    assert b.store.resident_count() == 12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    try:
        import torch.distributed as dist

        from common import planted_data as pdata
        from paper_2502_20969_b200 import laiv as L

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=2)
        cen, vecs, ids, off, qi, qo, g = pdata()
        ix = L.IvfIndex(cen, vecs, ids, off, L.Metric.InnerProduct)
        dev = L.Device(ix, 64 * CB, fetch_chunk_mb=2)
        dev.store.clear()
        for c in (range(0, 24) if rank == 1 else range(50, 54)):
            dev.store.insert(int(c))
        handles = [None, None]
        dist.all_gather_object(handles, dev.slab_ipc_handle())
        dev.peer_attach(0, ipc_handle=handles[1 - rank])
        dev.epoch_open()
        offs = [None, None]
        dist.all_gather_object(offs, dev.store_offsets().tolist())
        dev.peer_publish(0, np.array(offs[1 - rank], np.int64))
        out = None
        if rank == 0:
            res, tm = L.hybrid_search_batch(dev, qo, 16, 10)
            out = (res.ids.tolist(), res.scores.tolist(), tm.peer_lists)
        dist.barrier()  # the peer keeps its epoch open until rank 0 is done
        dev.epoch_close()
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error: " + repr(e)))


def test_peer_hits_across_processes_ipc(orc, laiv):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert not isinstance(out[1], str), out[1]
    assert not isinstance(out[0], str), out[0]
    ids_, scores, peer_lists = out[0]
    assert peer_lists > 0
    cen, vecs, ids, off, qi, qo, g = planted_data()
    for t in range(40):
        w = orc.ivf_search(cen, vecs, ids, off, 0, qo[t], 16, 10)
        assert_topk_parity(0, np.array(ids_[t], np.uint64), np.array(scores[t], np.float32), *w)


def test_epoch_publishes_only_pinned_lists(laiv):
    cen, vecs, ids, off, qi, qo, g = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
    b = laiv.Device(ix, 16 * CB)
    cache(b, range(0, 8))
    b.epoch_open()
    b.store.insert(30)  # during the epoch: not published
    offs = b.store_offsets()
    assert (offs[:8] >= 0).all() and offs[30] == -1
    b.store.evict(30)   # unpublished: released at once
    assert b.store.free_bytes() == 8 * CB
    b.store.evict(3)    # published: quarantined until the epoch closes
    assert b.store.free_bytes() == 8 * CB
    h = laiv.HotnessTable(laiv.CacheParams(cache_fraction=0.25))
    assert h.evict_to_fraction(b) == []  # pinned lists are passed over
    b.epoch_close()
    assert b.store.free_bytes() == 9 * CB
    assert len(h.evict_to_fraction(b)) == 3  # 7 resident -> 4 (25% of 16)
