"""Scan-kernel geometry sweep on one B200 (developer tool, not the bench).

Builds a planted datastore whose probe per query matches the C2 config
(nprobe 128 lists of 2442 x 768 fp32 = 962 MB scanned per query), makes every
list resident in the device cache, and times the scan kernel (CUDA events
around the launch, `t_scan`) for each (accumulation, tile, stages,
CTAs-per-SM) variant. Prints one JSON line per variant.

    python tools/sweep_scan.py [--lists 1024] [--queries 30]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_20969_b200 import laiv  # noqa: E402

VARIANTS = [
    # acc, impl, tile, stages, ctas_per_sm
    ("fp32", "tma", 0, 0, 0),
    ("fp64", "tma", 0, 0, 0),
    ("fp32", "tma", 8, 8, 1),
    ("fp32", "tma", 32, 2, 1),
    ("fp32", "tma", 8, 4, 2),
    ("fp32", "tma", 4, 8, 2),
    ("fp32", "tma", 16, 2, 2),
    ("fp32", "tma", 4, 16, 1),
    ("fp64", "tma", 8, 4, 2),
    ("fp32", "ldg", 0, 0, 0),
    ("fp32", "ldg", 0, 0, 3),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lists", type=int, default=1024)
    ap.add_argument("--per-list", type=int, default=2442)
    ap.add_argument("--nprobe", type=int, default=128)
    ap.add_argument("--queries", type=int, default=30)
    ap.add_argument("--metric", default="ip")
    ap.add_argument("--depth", action="store_true",
                    help="scan time vs nprobe for the default variants (fixed cost + slope)")
    args = ap.parse_args()
    global VARIANTS
    if args.depth:
        VARIANTS = [(a, "tma", 0, 0, 0, L) for a in ("fp32", "fp64") for L in (1, 8, 32, 128, 256)]
    else:
        VARIANTS = [v + (args.nprobe,) for v in VARIANTS]
    nc, per, d = args.lists, args.per_list, 768
    cen = laiv.synth_centroids(0, nc, d)
    vecs = laiv.pinned_empty((nc * per, d), np.float32)
    ids = np.empty(nc * per, np.uint64)
    laiv.synth_lists(0, cen, per, 0.05, vecs=vecs, ids=ids)
    off = np.arange(0, nc * per + 1, per, dtype=np.uint64)
    metric = laiv.Metric.InnerProduct if args.metric == "ip" else laiv.Metric.L2
    ix = laiv.IvfIndex(cen, vecs, ids, off, metric, borrow=True, trust=True)
    _, qo, _ = laiv.synth_queries(1, vecs, args.queries + 3, 0.008)
    member = 4 * d + 8
    for acc, impl, tile, stages, cps, nprobe in VARIANTS:
        try:
            dev = laiv.Device(ix, nc * per * member, acc_fp64=acc == "fp64", scan_impl=impl,
                              tma_tile=tile, tma_stages=stages, ctas_per_sm=cps)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"variant": [acc, impl, tile, stages, cps, nprobe], "error": str(e)}))
            continue
        plan = laiv.PrefetchPlan(list(range(nc)), 0, [])
        laiv.execute_prefetch(dev, plan, laiv.TransferChannel(1e9, laiv.ChannelMode.Device))
        dev.stage_queries(qo)
        ts, byts, ids0 = [], [], None
        for i in range(args.queries + 3):
            got_ids, _, _, t = dev.hybrid_search_staged(i, nprobe, 10)
            if i >= 3:
                ts.append(t.t_scan)
                byts.append(t.scanned_bytes)
            if i == 3:
                ids0 = got_ids
        ts = np.array(ts)
        gbs = np.array(byts) / ts / 1e9
        print(json.dumps({"variant": [acc, impl, tile, stages, cps, nprobe],
                          "t_scan_us_median": float(np.median(ts) * 1e6),
                          "t_scan_us_min": float(ts.min() * 1e6),
                          "gbs_median": float(np.median(gbs)), "gbs_max": float(gbs.max()),
                          "bytes": int(byts[0]), "first_ids": [int(x) for x in ids0[:3]]}),
              flush=True)
        dev.close()


if __name__ == "__main__":
    main()
