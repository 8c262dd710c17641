#!/usr/bin/env python
"""Batched coarse on the tensor cores at nq = 256 (nc 4096, d 768): a short
loop for ncu (`-k regex:coarse_tc`)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_20969_b200 import laiv  # noqa: E402

nc, d = 4096, 768
cen = laiv.synth_centroids(0, nc, d)
vecs, ids = laiv.synth_lists(0, cen, 2, 0.05)
ix = laiv.IvfIndex(cen, vecs, ids, np.arange(0, 2 * nc + 1, 2, dtype=np.uint64),
                   laiv.Metric.InnerProduct)
dev = laiv.Device(ix, 1 << 20, coarse_impl="tensor")
qi, qo, _ = laiv.synth_queries(1, vecs, 256, 0.01)
for _ in range(6):
    laiv.coarse_probe(dev, qo, 256)
