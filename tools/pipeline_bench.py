#!/usr/bin/env python
"""Trace replay on measured times (pipeline.py, ChannelMode.Device) at C2
scale: HyDE-shaped traces (query arrival, a generation stage that emits the
hypothetical document's embedding q_out, a retrieval, an answer stage) over
the 10M x 768 planted store; lookahead prefetch from q_in under the real
generation window, hotness cache, similarity grouping, micro-batches of 4.
Prints one JSON line with the run's aggregates and the simulated-clock
aggregates of the same replay for comparison.

    python tools/pipeline_bench.py [--traces 64] [--window 0.15]
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
    ap.add_argument("--config", default="c2")
    ap.add_argument("--traces", type=int, default=64)
    ap.add_argument("--window", type=float, default=0.15)
    ap.add_argument("--micro", type=int, default=4)
    a = ap.parse_args()
    sys.path.insert(0, ROOT)
    import bench
    from paper_2502_20969_b200 import laiv
    from paper_2502_20969_b200 import pipeline as P

    cfg = bench.CONFIGS[a.config]
    cen, vecs, ids, off = bench.make_datastore(cfg, 1, 0)
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.InnerProduct, borrow=True, trust=True)
    qi, qo, _ = laiv.synth_queries(bench.QSEED, vecs, a.traces, cfg.get("sigma", 0.008))
    side = np.empty((2 * a.traces, cfg["d"]), np.float32)
    side[0::2], side[1::2] = qi, qo
    S, K = P.Stage, P.StageKind
    traces = [P.QueryTrace(t, P.PipelineKind.HyDE, [
        S(K.Generate, 2 * t, 0.0), S(K.Generate, 2 * t + 1, a.window),
        S(K.Retrieve, 2 * t + 1, 0.0), S(K.Generate, -1, a.window)]) for t in range(a.traces)]
    member = 4 * cfg["d"] + 8
    cap = int(cfg["cache_frac"] * cfg["n_lists"]) * cfg["per_list"] * member
    rc = P.RunConfig(n_probe=cfg["nprobe"], top_k=cfg["k"], capacity_bytes=2 * cap,
                     prefetch_budget_bytes=cap, cache_fraction=0.5, micro_batch=a.micro,
                     cost=laiv.CostModel(bandwidth_bytes_per_s=55e9),
                     flags=P.RunFlags(lookahead_on=True, prefetch_sched_on=True,
                                      cache_sched_on=True, cache_on=True),
                     validate_exactness=False)
    out = {"config": a.config, "traces": a.traces, "window_s": a.window, "micro_batch": a.micro,
           "capacity_gb": rc.capacity_bytes / 1e9, "budget_gb": rc.prefetch_budget_bytes / 1e9}
    for mode in (laiv.ChannelMode.SimulatedClock, laiv.ChannelMode.Device):
        rc.mode = mode
        t0 = time.perf_counter()
        rec = P.run_batch(traces, side, ix, rc)
        wall = time.perf_counter() - t0
        ag = P.aggregate(rec.rows, rec.makespan_s)
        out[mode.name] = {"makespan_s": rec.makespan_s, "wall_s": wall,
                          "mean_latency_s": ag.mean_latency_s,
                          "mean_retrieve_ms": ag.mean_retrieve_s * 1e3,
                          "mean_transfer_ms": ag.mean_transfer_s * 1e3,
                          "mean_hit_rate": ag.mean_hit_rate, "mean_coverage": ag.mean_coverage,
                          "throughput_traces_per_s": ag.throughput_qps,
                          "assertions_ok": rec.assertions_ok}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
