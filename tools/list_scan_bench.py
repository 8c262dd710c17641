#!/usr/bin/env python
"""Batched hit scan: per-query scan vs the list-major tensor-core scan
(listscan.cu) on one GPU, every probed list resident (hit rate 1).

One synthetic IVF-Flat store (nc lists x per vectors x 768, in HBM), batches
of nq topical queries (Zipf-skewed topics, so queries share lists). For each
nprobe: the device-timed scan phase (t_scan, events) and the whole batch call
of both paths, results compared bit for bit. One JSON line per nprobe.

    python tools/list_scan_bench.py --nc 4096 --per 1000 --nq 256 --nprobe 32,64,128
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nc", type=int, default=4096)
    ap.add_argument("--per", type=int, default=1000)
    ap.add_argument("--d", type=int, default=768)
    ap.add_argument("--nq", type=int, default=256)
    ap.add_argument("--nprobe", default="32,64,128")
    ap.add_argument("--topics", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--metric", default="ip", choices=["ip", "l2"])
    a = ap.parse_args()
    from paper_2502_20969_b200 import laiv

    t0 = time.time()
    cen = laiv.synth_centroids(7, a.nc, a.d)
    vecs, ids = laiv.synth_lists(7, cen, a.per, 0.05)
    off = np.arange(0, a.nc * a.per + 1, a.per, dtype=np.uint64)
    metric = laiv.Metric.InnerProduct if a.metric == "ip" else laiv.Metric.L2
    ix = laiv.IvfIndex(cen, vecs, ids, off, metric)
    bytes_all = a.nc * a.per * (4 * a.d + 8)
    maxL = max(int(x) for x in a.nprobe.split(","))
    dev = laiv.Device(ix, bytes_all + (1 << 20), miss_fetch="off", max_probe=maxL)
    for c in range(a.nc):
        dev.store.insert(c)
    _, qo, _, _ = laiv.synth_queries_topical(9, cen, vecs, off, a.nq, 0.02, n_topics=a.topics)
    print(json.dumps({"setup_s": round(time.time() - t0, 1), "vectors": a.nc * a.per}),
          flush=True)

    for L in [int(x) for x in a.nprobe.split(",")]:
        out = {"nprobe": L, "nq": a.nq, "k": 10, "metric": a.metric}
        res = {}
        for mode in ("0", "1"):
            os.environ["LAIVG_LIST_SCAN"] = mode
            laiv.hybrid_search_batch(dev, qo, L, 10)  # warm-up
            ts, tw = [], []
            for _ in range(a.reps):
                w0 = time.perf_counter()
                r, t = laiv.hybrid_search_batch(dev, qo, L, 10)
                tw.append(time.perf_counter() - w0)
                ts.append(t.t_scan)
            res[mode] = r
            key = "list" if mode == "1" else "query"
            out[key + "_scan_ms"] = round(1e3 * float(np.median(ts)), 3)
            out[key + "_call_ms"] = round(1e3 * float(np.median(tw)), 3)
            out[key + "_qps"] = round(a.nq / float(np.median(tw)), 1)
            if mode == "1":
                out["scanned_bytes"] = int(t.scanned_bytes)
        runs, fb, qpl = dev.list_scan_stats()
        out["queries_per_list"] = round(qpl, 2)
        out["list_runs"], out["list_fallbacks"] = runs, fb
        same = all(np.array_equal(res["0"].topk(q).ids, res["1"].topk(q).ids) and
                   np.array_equal(res["0"].topk(q).scores, res["1"].topk(q).scores)
                   for q in range(a.nq))
        out["identical"] = bool(same)
        # distinct list bytes the list scan must read at least once
        probes = laiv.coarse_probe(dev, qo, L)
        distinct = np.unique(np.asarray(probes).reshape(-1))
        out["distinct_lists"] = int(len(distinct))
        out["distinct_list_bytes"] = int(len(distinct) * a.per * a.d * 4)
        out["list_scan_gbps_distinct"] = round(
            out["distinct_list_bytes"] / (out["list_scan_ms"] * 1e-3) / 1e9, 1)
        out["query_scan_gbps_algorithmic"] = round(
            out["scanned_bytes"] / (out["query_scan_ms"] * 1e-3) / 1e9, 1)
        out["speedup_scan"] = round(out["query_scan_ms"] / out["list_scan_ms"], 2)
        print(json.dumps(out), flush=True)
    os.environ.pop("LAIVG_LIST_SCAN", None)


if __name__ == "__main__":
    main()
