#!/usr/bin/env python
"""Summarise an ncu report (--set full) into a small JSON for profiles/.

    python tools/ncu_summary.py gpurun_out/x/prof.ncu-rep "<source command>" [config] \
        > profiles/rNN/x.json

`config` (the bench workload, e.g. c1 / c2) lets bench.py pick the summary for
its `roofline.traffic`.
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum",
]


def main():
    rep, src = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    config = sys.argv[3] if len(sys.argv) > 3 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    stall = [h for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled_")
             or h.startswith("smsp__pcsamp_warps_issue_stalled_")]
    out = {"source": src, "kernels": []}
    if config:
        out["config"] = config
    for r in rows[2:]:
        k = {"name": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                k[m] = f"{r[hdr.index(m)]} {units[hdr.index(m)]}".strip()
        st = []
        for h in stall:
            try:
                st.append((h.split("stalled_")[-1], float(r[hdr.index(h)])))
            except ValueError:
                pass
        k["top_stalls"] = sorted(st, key=lambda x: -x[1])[:6]
        out["kernels"].append(k)
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
