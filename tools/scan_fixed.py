#!/usr/bin/env python
"""Scan kernel fixed cost vs streaming rate: t_scan (CUDA events) against the
bytes scanned for L = 1..128 resident lists of 2442 x 768 fp32 (C2 list size).
Prints the least-squares intercept (fixed cost per launch) and slope (GB/s)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_20969_b200 import laiv  # noqa: E402

nc, per, d = 160, 2442, 768
cen = laiv.synth_centroids(0, nc, d)
vecs, ids = laiv.synth_lists(0, cen, per, 0.05)
off = np.arange(0, nc * per + 1, per, dtype=np.uint64)
ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
dev = laiv.Device(ix, nc * per * (4 * d + 8), scan_impl=os.environ.get("SCAN", "tma"),
                  tma_tile=int(os.environ.get("TILE", 0)), tma_stages=int(os.environ.get("STAGES", 0)),
                  ctas_per_sm=int(os.environ.get("CPS", 0)))
for c in range(nc):
    dev.store.insert(c)
qi, qo, _ = laiv.synth_queries(1, vecs, 64, 0.01)
dev.stage_queries(qo)
pts = []
for L in [int(x) for x in os.environ.get("LS", "1,2,4,8,16,32,64,96,128").split(",")]:
    ts = []
    for rep in range(12):
        _, _, nf, tm = dev.hybrid_search_staged(rep % 64, L, 10)
        if rep >= 2:
            ts.append(tm.t_scan)
    t = float(np.median(ts))
    b = L * per * d * 4
    pts.append((b, t))
    print(json.dumps({"L": L, "bytes": b, "t_scan_us": t * 1e6, "GBps": b / t / 1e9}), flush=True)
B = np.array([p[0] for p in pts], float)
T = np.array([p[1] for p in pts], float)
A = np.vstack([B, np.ones_like(B)]).T
slope, icpt = np.linalg.lstsq(A, T, rcond=None)[0]
print(json.dumps({"fixed_us": icpt * 1e6, "marginal_GBps": 1 / slope / 1e9}))
