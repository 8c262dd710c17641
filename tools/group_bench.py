#!/usr/bin/env python
"""Micro-batch scan A/B: per-query scan (one fast table per query) vs the
list-major group scan (the union of the micro-batch's lists streamed once),
on the C4 datastore with every list resident. Micro-batches are formed by
group_microbatches over topical queries, as the C4 pipeline does. One JSON
line per (nprobe, mode) with the device times of the search call.

    python tools/group_bench.py --nprobe 128,256 --micro 2,4
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4s")
    ap.add_argument("--nprobe", default="128,256")
    ap.add_argument("--micro", default="4")
    ap.add_argument("--batches", type=int, default=48)
    a = ap.parse_args()
    sys.path.insert(0, ROOT)
    import bench
    from paper_2502_20969_b200 import laiv

    cfg = bench.CONFIGS[a.config]
    cen, vecs, ids, off = bench.make_datastore(cfg, 1, 0)
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct, borrow=True, trust=True)
    cap = int(off[-1]) * (4 * cfg["d"] + 8)
    devs = {}
    for mode in ("per_query", "group"):
        if mode == "per_query":
            os.environ["LAIVG_NO_GROUP_SCAN"] = "1"
        else:
            os.environ.pop("LAIVG_NO_GROUP_SCAN", None)
        dv = laiv.Device(ix, cap, max_batch=32)
        dv.store.clear()
        for c in range(cfg["n_lists"]):
            dv.store.insert(c)
        devs[mode] = dv
    n = 4 * a.batches * 4
    qi, qo, _, topic = laiv.synth_queries_topical(bench.QSEED, cen, vecs, off, n,
                                                 cfg.get("sigma", 0.008), cfg["topics"],
                                                 cfg["zipf"], cfg["neigh"])
    for L in [int(x) for x in a.nprobe.split(",")]:
        for m in [int(x) for x in a.micro.split(",")]:
            mbs = laiv.group_microbatches(qi[: m * a.batches], m)
            mbs = [np.asarray(b.queries, np.int64) for b in mbs if len(b.queries) == m]
            probes = laiv.coarse_probe(devs["group"], qo, L)
            out = {}
            for mode, dv in devs.items():
                for sel in mbs[:3]:
                    laiv.hybrid_search_batch(dv, qo[sel], L, cfg["k"])
                t2, ts, res = [], [], []
                for sel in mbs:
                    r, tm = laiv.hybrid_search_batch(dv, qo[sel], L, cfg["k"])
                    t2.append(tm.t_2)
                    ts.append(tm.t_scan)
                    res.append(r.ids.copy())
                out[mode] = res
                uni = np.mean([len(np.unique(probes[sel])) for sel in mbs])
                print(json.dumps({"nprobe": L, "micro": m, "mode": mode,
                                  "t2_ms_median": float(np.median(t2) * 1e3),
                                  "t_scan_ms_median": float(np.median(ts) * 1e3),
                                  "qps": m / float(np.median(t2)),
                                  "union_lists_mean": float(uni),
                                  "sum_lists": m * L}), flush=True)
            same = all(np.array_equal(x, y) for x, y in zip(out["group"], out["per_query"]))
            print(json.dumps({"nprobe": L, "micro": m, "results_identical": same}), flush=True)


if __name__ == "__main__":
    main()
