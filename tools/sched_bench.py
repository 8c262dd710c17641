#!/usr/bin/env python
"""Routing cost per batch: host schedulers (group_microbatches on the CPU,
GPU probes, host overlap) vs laivg_schedule (all but the greedy on the GPU).
nc 4096, d 768, L 256, m 4, 8 workers with 10% of the lists resident."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_20969_b200 import laiv, shard  # noqa: E402

nc, d, L, m, nw = 4096, 768, 256, 4, 8
cen = laiv.synth_centroids(0, nc, d)
vecs, ids = laiv.synth_lists(0, cen, 2, 0.05)
ix = laiv.IvfIndex(cen, vecs, ids, np.arange(0, 2 * nc + 1, 2, dtype=np.uint64),
                   laiv.Metric.InnerProduct)
dev = laiv.Device(ix, 1 << 20)
rng = np.random.default_rng(0)
resident = (rng.random((nw, nc)) < 0.1).astype(np.uint8)
for n in (64, 256, 1024, 4096):
    qi, qo, _ = laiv.synth_queries(1, vecs, n, 0.01)

    def host():
        b = laiv.group_microbatches(qi, m)
        p = laiv.coarse_probe(dev, qi, L)
        return b, shard.route(b, p, resident)

    def gpu():
        b, a, _ = laiv.schedule(dev, qi, m, L, resident)
        return b, a

    hb, ha = host()
    gb, ga = gpu()
    assert [x.queries for x in hb] == [x.queries for x in gb] and ha == ga
    for name, fn in (("host", host), ("gpu", gpu)):
        fn()
        t0 = time.perf_counter()
        reps = 5
        for _ in range(reps):
            fn()
        print(json.dumps({"impl": name, "n": n, "ms": (time.perf_counter() - t0) / reps * 1e3}),
              flush=True)
