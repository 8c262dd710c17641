"""Batched exact selection (tensor-core coarse path) against the fp64 path:
equal probes, wall time per coarse_probe call; LAIVG_TC_PROBE=1 prints
the per-phase stamps of query 0."""
import sys, os, time, json
sys.path.insert(0, ".")
import numpy as np
from paper_2502_20969_b200 import laiv
nc, d = 4096, 768
cen = laiv.synth_centroids(0, nc, d); vecs, ids = laiv.synth_lists(0, cen, 2, 0.05)
off = np.arange(0, nc * 2 + 1, 2, dtype=np.uint64)
ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct)
qi, qo, _ = laiv.synth_queries(1, vecs, 256, 0.01)
dev = laiv.Device(ix, 1 << 20, coarse_impl="tensor")
ref = laiv.Device(ix, 1 << 20, coarse_impl="fp64")
for nq in (32, 256):
    for L in (128, 256):
        a = laiv.coarse_probe(dev, qo[:nq], L); b = laiv.coarse_probe(ref, qo[:nq], L)
        assert np.array_equal(a, b), (nq, L)
        for _ in range(5): laiv.coarse_probe(dev, qo[:nq], L)
        t0 = time.perf_counter(); n = 50
        for _ in range(n): laiv.coarse_probe(dev, qo[:nq], L)
        print(json.dumps({"nq": nq, "L": L, "ms": (time.perf_counter() - t0) / n * 1e3, "equal_fp64": True}), flush=True)
