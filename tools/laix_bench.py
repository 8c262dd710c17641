#!/usr/bin/env python
"""LAIX load/save throughput: the planted C1/C2 datastore
written with laivg_index_save, read back with laivg_index_load (parallel
pread into the final list-major block, then pinned in place), the
reference's load_index (oracle/_ref, one ifstream, row-by-row append) timed
on the same file, and a GPU search through the loaded index checked against
the index built from the arrays. One JSON line.

The file lives in /dev/shm by default (RAM-backed): the numbers are the
loader's memory-side cost, not a disk's.

    python tools/laix_bench.py --config c1 [--dir /dev/shm] [--no-ref]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--dir", default="/dev/shm")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    sys.path.insert(0, ROOT)
    import bench
    from paper_2502_20969_b200 import laiv

    cfg = bench.CONFIGS[a.config]
    cen, vecs, ids, off = bench.make_datastore(cfg, 1, 0)
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct, borrow=True, trust=True)
    path = os.path.join(a.dir, f"laivg_bench_{os.getpid()}.laix")
    out = {"config": a.config, "n": int(off[-1]), "d": cfg["d"], "lists": cfg["n_lists"]}
    try:
        t0 = time.perf_counter()
        ix.save(path, a.threads)
        out["save_s"] = time.perf_counter() - t0
        size = os.path.getsize(path)
        out["file_gb"] = size / 1e9
        out["save_gbs"] = size / out["save_s"] / 1e9
        loads = []
        for _ in range(3):
            t0 = time.perf_counter()
            lx = laiv.load_index(path, a.threads)
            loads.append(time.perf_counter() - t0)
            if _ < 2:
                lx.close()
        out["load_s"] = min(loads)
        out["load_gbs"] = size / out["load_s"] / 1e9
        out["threads"] = a.threads or os.cpu_count()
        v2, i2 = lx.store()
        out["store_identical"] = bool(np.array_equal(i2, ids) and np.array_equal(v2, vecs)
                                      and np.array_equal(lx.list_off, off))
        # the loaded (pinned-in-place) store serves the GPU path
        dev_a = laiv.Device(lx, 1 << 34)
        dev_b = laiv.Device(ix, 1 << 34)
        Q = vecs[np.random.default_rng(1).integers(0, len(vecs), 32)]
        L, k = cfg["nprobe"], cfg["k"]
        ra, _ = laiv.hybrid_search_batch(dev_a, Q, L, k)
        rb, _ = laiv.hybrid_search_batch(dev_b, Q, L, k)
        out["search_identical"] = bool(np.array_equal(ra.ids, rb.ids)
                                       and np.array_equal(ra.scores, rb.scores))
        if not a.no_ref:
            sys.path.insert(0, ROOT)
            import ctypes as C

            from oracle.oracle import RefLib

            if RefLib.available():
                ref = RefLib()
                h = C.c_void_p()
                t0 = time.perf_counter()
                kind = ref.L.ref_load_index(path.encode(), C.byref(h))
                out["ref_load_s"] = time.perf_counter() - t0
                out["ref_load_gbs"] = size / out["ref_load_s"] / 1e9
                out["ref_kind"] = int(kind)
                if kind == 0:
                    ref.L.ref_index_destroy(h)
    finally:
        if os.path.exists(path):
            os.unlink(path)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
