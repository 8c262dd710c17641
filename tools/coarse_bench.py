#!/usr/bin/env python
"""Batched coarse_probe: fp64 SIMT path vs tcgen05 tf32 path, per batch size
(nc 4096, d 768, L 256). Prints one JSON line per (impl, nq) with the mean
wall time of laivg_coarse_probe (H2D of the queries and D2H of the probes
included) and the device time of the selection chain from ncu-free events is
not available here, so compare impls at equal nq."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_20969_b200 import laiv  # noqa: E402

nc, d, L = 4096, 768, int(os.environ.get("L", 256))
cen = laiv.synth_centroids(0, nc, d)
vecs, ids = laiv.synth_lists(0, cen, 2, 0.05)
off = np.arange(0, nc * 2 + 1, 2, dtype=np.uint64)
ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
qi, qo, _ = laiv.synth_queries(1, vecs, 256, 0.01)
for impl in ("fp64", "tensor"):
    dev = laiv.Device(ix, 1 << 20, coarse_impl=impl)
    for nq in (8, 32, 64, 128, 256):
        Q = qo[:nq]
        for _ in range(5):
            laiv.coarse_probe(dev, Q, L)
        t0 = time.perf_counter()
        n = 50
        for _ in range(n):
            laiv.coarse_probe(dev, Q, L)
        dt = (time.perf_counter() - t0) / n
        print(json.dumps({"impl": impl, "nq": nq, "L": L, "ms": dt * 1e3}), flush=True)
    dev.close()
