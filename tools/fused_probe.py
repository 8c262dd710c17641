#!/usr/bin/env python
"""Phase breakdown of the fused single-query kernel against the multi-kernel
chain: C1 / C2 coarse shapes (nc 1024 / 4096, d 768) with short lists, every
list resident. Per mode, the staged-row entry (query in HBM) and the host-row
entry (laivg_hybrid_search on a host buffer) are timed. With LAIVG_TRACE=1 the
library prints CTA 0's globaltimer stamps per call.
Usage: LAIVG_TRACE=1 python tools/fused_probe.py"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_20969_b200 import laiv  # noqa: E402

d = 768
SHAPES = [(1024, 32, int(os.environ.get("PER1", 977))), (4096, 128, int(os.environ.get("PER2", 600)))]
if os.environ.get("ONLY"):  # e.g. ONLY=4096 (one coarse shape)
    SHAPES = [s for s in SHAPES if s[0] == int(os.environ["ONLY"])]
MODES = os.environ.get("MODES", "chain,fused,chain,fused").split(",")
ENTRIES = os.environ.get("ENTRIES", "staged,host").split(",")
for nc, L, per in SHAPES:
    cen = laiv.synth_centroids(0, nc, d)
    vecs, ids = laiv.synth_lists(0, cen, per, 0.05)
    off = np.arange(0, nc * per + 1, per, dtype=np.uint64)
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
    qi, qo, _ = laiv.synth_queries(1, vecs, 64, 0.01)
    for mode in MODES:
        dev = laiv.Device(ix, nc * per * (4 * d + 8), single_query=mode)
        for c in range(nc):
            dev.store.insert(c)
        dev.stage_queries(qo)
        for entry in ENTRIES:
            rows = []
            for rep in range(24):
                t0 = time.perf_counter()
                if entry == "staged":
                    _, _, nf, tm = dev.hybrid_search_staged(rep % 64, L, 10)
                else:
                    _, tm = laiv.hybrid_search(dev, qo[rep % 64], L, 10)
                wall = time.perf_counter() - t0
                if rep >= 4:
                    rows.append((tm.t_coarse, tm.t_scan, tm.t_kernel, tm.t_2, wall))
            r = np.median(np.array(rows), axis=0) * 1e6
            print(json.dumps({"nc": nc, "L": L, "per": per, "mode": mode, "entry": entry,
                              "t_coarse_us": r[0], "t_scan_us": r[1], "t_kernel_us": r[2],
                              "t_2_us": r[3], "call_us": r[4]}), flush=True)
        dev.close()
    ix.close()
