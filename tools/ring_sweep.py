#!/usr/bin/env python
"""TMA ring geometry of the fused single-query kernel at the C1 / C2 shapes
(every list resident): median kernel event time and in-kernel scan phase per
(rows per stage, stages). Usage: python tools/ring_sweep.py [c1|c2]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_20969_b200 import laiv  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
nc, per, L = (4096, 2442, 128) if cfg == "c2" else (1024, 977, 32)
d = 768
cen = laiv.synth_centroids(0, nc, d)
vecs, ids = laiv.synth_lists(0, cen, per, 0.05)
off = np.arange(0, nc * per + 1, per, dtype=np.uint64)
ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct, borrow=True, trust=True)
qi, qo, _ = laiv.synth_queries(1, vecs, 64, 0.01)
# a cache of 2 x the probe: the lists each query probes are made resident
for tile, stages in ((32, 2), (16, 4), (8, 8), (20, 3), (64, 1), (32, 2)):
    dev = laiv.Device(ix, 2 * L * per * (4 * d + 8), tma_tile=tile, tma_stages=stages)
    dev.stage_queries(qo)
    rows = []
    for rep in range(16):
        q = rep % 8
        dev.store.clear()
        for c in laiv.coarse_probe(dev, qo[q], L).reshape(-1):
            dev.store.insert(int(c))
        _, _, nf, tm = dev.hybrid_search_staged(q, L, 10)
        if rep >= 4:
            rows.append((tm.t_kernel, tm.t_scan, tm.t_2, tm.scanned_bytes))
    r = np.median(np.array(rows), axis=0)
    print(json.dumps({"cfg": cfg, "tile": tile, "stages": stages, "kernel_us": r[0] * 1e6,
                      "scan_phase_us": r[1] * 1e6, "t2_us": r[2] * 1e6,
                      "scan_phase_tbps": r[3] / r[1] / 1e12}), flush=True)
    dev.close()
