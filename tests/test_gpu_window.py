"""Decode-like generation windows (laivg_window_load) and the independent
host-link probe (laivg_link_peak).

The lookahead prefetch (tiered.cpp:86-136) overlaps its copies with the
generation window; with a load buffer set the window streams HBM like a
memory-bound decode, so the copies compete with it. The copied lists and the
retrieval results must be unaffected, and the report carries the window's
measured read rate.
"""
import numpy as np
import pytest

from common import IP, assert_topk_parity, planted_data

pytestmark = pytest.mark.gpu


def test_link_peak(laiv):
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
    dev = laiv.Device(ix, 1 << 28)
    h2d, d2h = dev.link_peak(256 << 20)
    # any PCIe Gen4/5 or C2C host link: well above 5 GB/s, below 1 TB/s
    assert 5.0 < h2d < 1000.0 and 5.0 < d2h < 1000.0
    with pytest.raises(ValueError):
        dev.link_peak(0)


def test_decode_window_prefetch(orc, laiv):
    cen, vecs, ids, off, qi, qo, _ = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
    per = 300 * (4 * 768 + 8)
    dev = laiv.Device(ix, 64 * per)
    chan = laiv.TransferChannel(50e9, laiv.ChannelMode.Device)
    # idle window: no read rate
    plan = laiv.plan_prefetch(dev, qi[0], 16 * per)
    rep = laiv.execute_prefetch(dev, plan, chan, 0.01)
    assert rep.window_read_gbps == 0.0 and rep.window_s >= 0.0099
    # decode-like: 1 GB per token at 2 TB/s -> one token every 0.5 ms
    dev.window_load(1 << 30, 2000.0)
    for t in range(4):
        dev.store.clear()
        plan = laiv.plan_prefetch(dev, qi[t], 16 * per)
        rep = laiv.execute_prefetch(dev, plan, chan, 0.02)
        assert rep.window_s >= 0.0199
        assert 1000.0 < rep.window_read_gbps < 2600.0, rep.window_read_gbps
        assert rep.transferred == plan.clusters
        res, _ = laiv.hybrid_search(dev, qo[t], 8, 10)
        want = orc.ivf_search(cen, vecs, ids, off, IP, qo[t], 8, 10)
        assert_topk_parity(IP, res.topk.ids, res.topk.scores, *want)
    # prefetch_batch shares the window
    dev.store.clear()
    rep, _ = laiv.prefetch_batch(dev, qi[:4], [8 * per] * 4, chan, 0.02)
    assert rep.window_read_gbps > 1000.0
    # back to idle
    dev.window_load(0, 0.0)
    assert dev.window(0.005) >= 0.0049
    with pytest.raises(ValueError):
        dev.window_load(1 << 20, -1.0)
