#!/usr/bin/env python
"""C5 (BASELINE.json configs[4]): nprobe sweep x cache-size sweep with the
routed pipeline of the C4 bench at W workers (emulated on one GPU unless run
under torchrun), reporting hit rate, exposed H2D and retrieval q/s per point.
One datastore for the whole sweep. One JSON line per (nprobe, cache %).

    python tools/sweep_c5.py --workers 8 --config c4s --steps 2 --warmup 1
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--config", default="c4s")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--window", type=float, default=0.15)
    ap.add_argument("--nprobe", default="32,64,128,256,512,1024")
    ap.add_argument("--cache", default="0.05,0.10,0.25,0.50")
    ap.add_argument("--peers", action="store_true")
    ap.add_argument("--acc", default="fp64", choices=["fp64", "fp32"])
    ap.add_argument("--micro", default="",
                    help="comma list of micro-batch sizes (default: the config's)")
    ap.add_argument("--list-scan", default="",
                    help="comma list of LAIVG_LIST_SCAN modes per point (0 off, 1 on, "
                         "auto = unset); default: the environment's")
    a = ap.parse_args()
    sys.path.insert(0, ROOT)
    import bench

    micros = [int(x) for x in a.micro.split(",")] if a.micro else [None]
    modes = a.list_scan.split(",") if a.list_scan else [None]
    points = [(m, mode, cf, L) for m in micros for mode in modes
              for cf in [float(x) for x in a.cache.split(",")]
              for L in [int(x) for x in a.nprobe.split(",")]]
    for micro, mode, cf, L in points:
        if mode is not None:
            if mode == "auto":
                os.environ.pop("LAIVG_LIST_SCAN", None)
            else:
                os.environ["LAIVG_LIST_SCAN"] = mode
        if True:
            cfg = dict(bench.CONFIGS[a.config], nprobe=L, cache_frac=cf)
            if micro:
                cfg["micro"] = micro
            bench.CONFIGS["_sweep"] = cfg
            args = argparse.Namespace(gpus=1, steps=a.steps, warmup=a.warmup, impl="ours",
                                      config="_sweep", metric="ip", window=a.window, sigma=None,
                                      cpu_sample=0, no_cpu_baseline=True, acc=a.acc, scan="tma",
                                      workers=a.workers, peers=a.peers, single="fused",
                                      window_load=0.0, window_buffer_gb=16.0, budget_scale=1.0)
            import io
            from contextlib import redirect_stdout

            buf = io.StringIO()
            with redirect_stdout(buf):
                bench.run_ours_routed(args, cfg)
            line = json.loads(buf.getvalue().strip().splitlines()[-1])
            r = line["routing"]
            print(json.dumps({"nprobe": L, "cache_fraction": cf, "workers": a.workers,
                              "emulated": line.get("emulated_workers"),
                              "value_qps": line["value"], "p50_step_ms": line["p50_latency_ms"],
                              "hit_rate": r["hit_rate"], "exposed_h2d_ms_mean": r["exposed_ms_mean"],
                              "fetched_lists_mean": r["fetched_lists_mean"],
                              "peer_lists_mean": r.get("peer_lists_mean", 0.0), "peers": a.peers,
                              "host_scan_ms_mean": r["host_scan_ms_max_mean"],
                              "schedule_ms_mean": r["schedule_ms_mean"],
                              "acc": a.acc, "micro": cfg.get("micro"),
                              "list_scan": mode or os.environ.get("LAIVG_LIST_SCAN", "auto"),
                              "gpu_scan_ms_per_step": line.get("roofline", {}).get("avg_launch_ms"),
                              "results_identical": line["value_e2e_results_identical"]}),
                  flush=True)


if __name__ == "__main__":
    main()
