#!/usr/bin/env python
"""bench.py — lookahead IVF retrieval on B200 (BASELINE.json metric).

Workload (default `--config c2`, BASELINE.json configs[1]): synthetic
IVF-Flat 10M x 768 fp32 (4096 balanced lists of 2442 planted-cluster members,
SURVEY §8d generator), nprobe 128, k 10, inner product, single-query
lookahead prefetch on one B200.

One step = one query round of the TeleRAG pipeline (pipeline.cpp:357-441):
  1. the device cache (TieredStore, capacity 10% of the datastore) starts
     empty (cache off, pipeline.cpp:466-473);
  2. plan_prefetch from the pre-retrieval embedding q_in (GPU coarse ranking +
     host greedy walk) under budget = min(B_link * window, capacity)
     (calibrate_budget rule, budget.cpp:159-182);
  3. execute_prefetch: the planned IVF lists stream host->HBM on the copy
     stream while the generation-window kernel occupies the compute stream;
  4. hybrid_search for q_out: GPU coarse + list scan over the resident probed
     lists, host scan of the misses, merge.

Reported metric: retrieval queries/s and p50 retrieval latency, where the
retrieval latency of a query = exposed prefetch (copy end past window end)
+ the hybrid search. `value` uses queries staged in HBM; `e2e` the host-buffer
C-ABI call (query H2D and result D2H inside). The window itself is simulated
LLM time, reported separately (`pipeline_ms_per_step`).

`--impl reference` times the reference's own CPU search (laiv::ivf_search from
oracle/_ref/libref.so, built from the reference sources) on all host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1]
    "c2": dict(workload="synthetic IVF-Flat 10M x 768 fp32, 4096 lists, nprobe=128, k=10, "
                        "single-query lookahead prefetch on 1 x B200",
               n_lists=4096, per_list=2442, d=768, nprobe=128, k=10, window_s=0.15,
               cache_frac=0.10),
    # BASELINE.json configs[0] shape (1M x 768, 1024 lists, nprobe 32)
    "c1": dict(workload="synthetic IVF-Flat 1M x 768 fp32, 1024 lists, nprobe=32, k=10, batch=1",
               n_lists=1024, per_list=977, d=768, nprobe=32, k=10, window_s=0.02,
               cache_frac=0.10),
    # BASELINE.json configs[2]: micro-batch of 32 with lookahead prefetch
    "c3": dict(workload="synthetic IVF-Flat 20M x 768 fp32 (~61 GB host datastore), 4096 lists, "
                        "nprobe=256, batch=32, GPU cache sized to 10% of lists",
               n_lists=4096, per_list=4883, d=768, nprobe=256, k=10, window_s=0.15,
               cache_frac=0.10, batch=32),
    # C3's shape at half the datastore (fits a 1-GPU box next to the reference copy)
    "c3s": dict(workload="synthetic IVF-Flat 10M x 768 fp32, 4096 lists, nprobe=256, batch=32, "
                         "GPU cache sized to 10% of lists",
                n_lists=4096, per_list=2442, d=768, nprobe=256, k=10, window_s=0.15,
                cache_frac=0.10, batch=32),
    # batched retrieval with the whole index resident in HBM (30.8 GB of 180):
    # 256 queries per device batch share lists (8 per list at nprobe 128), so
    # the hits run on the list-major tensor-core scan (listscan.cu)
    "c2b": dict(workload="synthetic IVF-Flat 10M x 768 fp32, 4096 lists, nprobe=128, k=10, "
                         "batch=256 queries per device call, whole index resident in HBM",
                n_lists=4096, per_list=2442, d=768, nprobe=128, k=10, window_s=0.0,
                cache_frac=1.0, batch=256, resident_all=True),
    # BASELINE.json configs[3]: 256 topical queries per step, micro-batches of 4
    # grouped (group_microbatches) and routed cache-aware across the GPUs
    "c4": dict(workload="batched retrieval 256 queries/step, nprobe=256, cache-aware routing "
                        "across the GPUs (20M x 768 fp32, 4096 lists, per-GPU cache 10% of lists, "
                        "hotness-managed; Zipf-topical queries)",
               n_lists=4096, per_list=4883, d=768, nprobe=256, k=10, window_s=0.15,
               cache_frac=0.10, batch=256, routed=True, micro=4, topics=32, zipf=1.0,
               neigh=16, hot_fraction=0.5),
    "c4s": dict(workload="batched retrieval 256 queries/step, nprobe=256, cache-aware routing "
                         "(10M x 768 fp32, 4096 lists, per-GPU cache 10% of lists, "
                         "hotness-managed; Zipf-topical queries)",
                n_lists=4096, per_list=2442, d=768, nprobe=256, k=10, window_s=0.15,
                cache_frac=0.10, batch=256, routed=True, micro=4, topics=32, zipf=1.0,
                neigh=16, hot_fraction=0.5),
    # C2 where prefetch hiding can fail: a 50 ms window
    # (copy time ~ window at the calibrate_budget rule, budget uncapped by the
    # 25% cache) that streams a 16 GB "weights" buffer like a memory-bound
    # decode at ~5 TB/s, so the copies share HBM with it
    "c2h": dict(workload="synthetic IVF-Flat 10M x 768 fp32, 4096 lists, nprobe=128, k=10, "
                         "single-query lookahead prefetch, 50 ms decode-like window (16 GB "
                         "streamed at 5 TB/s), cache 25% of lists",
                n_lists=4096, per_list=2442, d=768, nprobe=128, k=10, window_s=0.05,
                cache_frac=0.25, window_load_gbps=5000.0, window_buffer_gb=16.0),
    "small": dict(workload="synthetic IVF-Flat 100K x 768 fp32, 256 lists, nprobe=16, k=10",
                  n_lists=256, per_list=400, d=768, nprobe=16, k=10, window_s=0.005,
                  cache_frac=0.25),
}
SEED, QSEED, SPREAD = 0, 1, 0.05


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def init_dist(world, local):
    """One process per GPU. torch.distributed carries only the control plane
    (barriers, the resident-set all-gather of the routed config, the max of
    the ranks' timings): gloo on the host. The retrieval data path has no
    collective. Returns (dist or None, this rank's CUDA ordinal)."""
    if world == 1:
        return None, 0
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo")
    n = max(1, torch.cuda.device_count())
    return dist, local % n


def host_threads(world):
    """Host miss-scan threads per rank: the node's cores split between the
    ranks (one process per GPU shares the host)."""
    return max(1, (os.cpu_count() or 1) // max(1, world))


def pin_rank_cores(rank, world):
    """One process per GPU: rank r runs (and spawns its miss-scan threads) on
    its own slice of the node's cores, so N ranks never share a core."""
    if world <= 1 or not hasattr(os, "sched_setaffinity"):
        return None
    cores = sorted(os.sched_getaffinity(0))
    per = max(1, len(cores) // world)
    mine = cores[rank * per:(rank + 1) * per] or cores[-per:]
    os.sched_setaffinity(0, mine)
    return mine


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# --------------------------------------------------------------------------
# datastore
# --------------------------------------------------------------------------
def make_datastore(cfg, world, rank, pinned=True, gen=None):
    """Planted-cluster list-major datastore. One process: pinned allocation.
    Several ranks: rank 0 fills a /dev/shm file that every rank maps and pins
    (one host copy shared by all GPUs). `gen` draws it: the product's
    laivg_synth_* (our arm) or oracle/libsynth.so, the same generator source
    built alone (the reference arm, which must not load liblaivg.so)."""
    if gen is None:
        from paper_2502_20969_b200 import laiv as gen
    laiv = gen

    nc, per, d = cfg["n_lists"], cfg["per_list"], cfg["d"]
    n = nc * per
    key = (nc, per, d, pinned, getattr(gen, "__name__", ""))
    if world == 1 and key in _DATASTORES:  # sweeps reuse one datastore
        return _DATASTORES[key]
    cen = laiv.synth_centroids(SEED, nc, d)
    t0 = time.time()
    if world == 1:
        vecs = gen.pinned_empty((n, d), np.float32) if pinned else np.empty((n, d), np.float32)
        ids = np.empty(n, np.uint64)
        laiv.synth_lists(SEED, cen, per, SPREAD, vecs=vecs, ids=ids)
    else:
        import torch.distributed as dist

        path = f"/dev/shm/laivg_{nc}x{per}x{d}_s{SEED}.bin"
        if rank == 0:
            mm = np.memmap(path, np.float32, "w+", shape=(n, d))
            ids = np.empty(n, np.uint64)
            laiv.synth_lists(SEED, cen, per, SPREAD, vecs=mm, ids=ids)
            mm.flush()
            del mm
        dist.barrier()
        vecs = np.memmap(path, np.float32, "r+", shape=(n, d))
        ids = np.arange(n, dtype=np.uint64)  # synth ids are j*per+i == row index
        dist.barrier()
        if rank == 0:  # every rank holds its mapping; the name can go now
            os.unlink(path)
        if pinned:
            from paper_2502_20969_b200._lib import check

            check(laiv.lib().laivg_host_register(vecs.ctypes.data, vecs.nbytes))
    off = np.arange(0, n + 1, per, dtype=np.uint64)
    log(f"[bench] datastore {n}x{d} ({n * (4 * d + 8) / 1e9:.1f} GB) in {time.time() - t0:.1f}s")
    if world == 1:
        _DATASTORES[key] = (cen, vecs, ids, off)
    return cen, vecs, ids, off


_DATASTORES = {}


def q_out_sigma(args, cfg, laiv, dev, vecs, L):
    """The q_out perturbation: --sigma, else the config's value (fixed so the
    reference arm draws the very same queries; it is what calibrate_sigma
    returns on these seeded datastores), with the measured mean coverage."""
    if args.sigma is not None and args.sigma < 0:  # --sigma -1: recalibrate
        return calibrate_sigma(laiv, dev, vecs, L)
    sigma = args.sigma or cfg.get("sigma", 0.008)
    qi, qo, _ = laiv.synth_queries(QSEED + 1000, vecs, 32, sigma)
    cov = float(np.mean([laiv.coverage(dev, a, b, L) for a, b in zip(qi, qo)]))
    return sigma, cov


def calibrate_sigma(laiv, dev, vecs, L, target=0.8, nq=32):
    """Largest q_out perturbation whose mean coverage at nprobe >= target
    (coverage in [0.6, 0.95]; acceptance.cpp:219-223)."""
    best = None
    for sigma in (0.002, 0.004, 0.006, 0.008, 0.010, 0.012, 0.015, 0.02, 0.03):
        qi, qo, _ = laiv.synth_queries(QSEED + 1000, vecs, nq, sigma)
        cov = float(np.mean([laiv.coverage(dev, a, b, L) for a, b in zip(qi, qo)]))
        if cov >= target:
            best = (sigma, cov)
        else:
            break
    return best if best else (0.002, None)


# --------------------------------------------------------------------------
# clocks (nvidia-smi during the timed region)
# --------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        self.lines = []
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                smax.append(float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def profiled_traffic(kernel_prefix: str, config: str = "c2"):
    """dram read+write bytes per launch of the dominant kernel from the newest
    committed `ncu --set full` summary of this workload (profiles/rNN/
    ncu_*full*_summary.json; a summary without a "config" key is C2), or None."""
    import glob

    paths = glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_*full*summary.json"))
    for path in sorted(paths, reverse=True):
        try:
            with open(path) as f:
                doc = json.load(f)
            if doc.get("config", "c2") != config:
                continue
            vals = []
            for k in doc["kernels"]:
                if kernel_prefix in k["name"]:
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

                    def nbytes(v):
                        x, unit = v.split()[:2]
                        return float(x.replace(",", "")) * scale[unit]

                    vals.append(nbytes(k["dram__bytes_read.sum"]) +
                                nbytes(k["dram__bytes_write.sum"]))
            if vals:
                return float(np.mean(vals)), os.path.relpath(path, ROOT)
        except (OSError, KeyError, ValueError, IndexError):
            continue
    return None, None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


# --------------------------------------------------------------------------
# reference CPU arm
# --------------------------------------------------------------------------
def reference_index(cen, vecs, ids, off, metric):
    from oracle.oracle import RefLib

    t0 = time.time()
    ri = RefLib().index(cen, vecs, ids, off, metric)
    log(f"[bench] reference index built in {time.time() - t0:.1f}s")
    return ri


def host_cpu_model():
    """lscpu-style model string of the host cores (state them)."""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(ri, q_out, L, k, threads, sample):
    """The reference laiv::ivf_search on `threads` host threads over `sample`
    queries; returns q/s, p50 latency and the results."""
    t0 = time.perf_counter()
    ids, sc, lat = ri.search_many(q_out[:sample], L, k, threads)
    wall = time.perf_counter() - t0
    return dict(qps=sample / wall, p50_ms=float(np.median(lat) * 1e3), wall_s=wall,
                ids=ids, scores=sc)


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0  # the reference arm is one host process on rank 0
    # workload from oracle/libsynth.so: the product library is never loaded here
    from oracle import synth

    cen, vecs, ids, off = make_datastore(cfg, 1, 0, pinned=False, gen=synth)
    metric = 0 if args.metric == "ip" else 1
    sigma = args.sigma or cfg.get("sigma", 0.008)  # the same queries as our arm
    qi, qo, _ = synth.synth_queries(QSEED, vecs, 4096, sigma)
    ri = reference_index(cen, vecs, ids, off, metric)
    threads = os.cpu_count() or 1
    per_step = threads
    L, k = cfg["nprobe"], cfg["k"]
    qpos = 0
    for _ in range(args.warmup):
        ri.search_many(qo[qpos:qpos + per_step], L, k, threads)
        qpos += per_step
    lats = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _, _, lat = ri.search_many(qo[qpos:qpos + per_step], L, k, threads)
        lats.extend(lat.tolist())
        qpos += per_step
    wall = time.perf_counter() - t0
    qps = args.steps * per_step / wall
    line = {
        "impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64-accumulate/f32", "data": "synthetic",
        "p50_latency_ms": float(np.median(lats) * 1e3),
        "config": config_block(cfg, args, sigma),
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads,
                         "kind": "reference", "cpu_model": host_cpu_model(),
                         "single_thread_latency_ms": float(np.median(lats) * 1e3),
                         "sample": f"{per_step} queries per step (one per host thread), "
                                   f"laiv::ivf_search from oracle/_ref/libref.so"},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


METRIC = "IVF retrieval queries/sec and p50 retrieval latency (prefetch-overlapped)"


def config_block(cfg, args, sigma):
    return {"workload": cfg["workload"], "n_vectors": cfg["n_lists"] * cfg["per_list"],
            "dim": cfg["d"], "n_lists": cfg["n_lists"], "nprobe": cfg["nprobe"], "k": cfg["k"],
            "metric": args.metric, "batch": cfg.get("batch", 1), "window_s": args.window,
            "cache_fraction_of_lists": cfg["cache_frac"], "q_out_sigma": sigma,
            "query_seed": QSEED,
            "budget_scale": args.budget_scale,
            "window_kind": (f"decode-like: {args.window_buffer_gb:g} GB streamed per token at "
                            f"{args.window_load:g} GB/s target" if args.window_load > 0
                            else "idle (%globaltimer spin)"),
            "l2_flush": "not needed: each query scans up to ~1 GB of lists > 126 MB L2, "
                        "and every step re-fetches its lists into a cleared cache"}


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def run_ours(args, cfg):
    from paper_2502_20969_b200 import laiv, shard

    rank, world, local = dist_env()
    dist = None
    dist, gpu = init_dist(world, local)
    pin_rank_cores(rank, world)
    cen, vecs, ids, off = make_datastore(cfg, world, rank)
    metric = laiv.Metric.InnerProduct if args.metric == "ip" else laiv.Metric.L2
    ix = laiv.IvfIndex(cen, vecs, ids, off, metric, borrow=True, trust=True)
    member = 4 * cfg["d"] + 8
    capacity = int(cfg["cache_frac"] * cfg["n_lists"]) * cfg["per_list"] * member
    dev = laiv.Device(ix, capacity, device=gpu, miss_threads=host_threads(world),
                      acc_fp64=args.acc == "fp64", scan_impl=args.scan,
                      single_query=args.single)
    L, k = cfg["nprobe"], cfg["k"]
    if args.window_load > 0:
        dev.window_load(int(args.window_buffer_gb * 1e9), args.window_load)
    # independent host-link peak: one large pinned copy per direction
    link_h2d, link_d2h = dev.link_peak(1 << 30)

    # link bandwidth for the calibrate_budget rule, measured on this box
    probe_plan = laiv.plan_prefetch(dev, cen[0], min(capacity, 64 * cfg["per_list"] * member))
    rep = laiv.execute_prefetch(dev, probe_plan, laiv.TransferChannel(1, laiv.ChannelMode.Device))
    dev.store.clear()
    b_link = rep.h2d_gbps * 1e9
    budget = int(min(b_link * args.window * args.budget_scale, capacity))
    sigma, cov = q_out_sigma(args, cfg, laiv, dev, vecs, L)
    # (one rank: extra queries of the same generator extend the CPU sample)
    nq_total = max((args.warmup + args.steps) * world + 8,
                   args.warmup + args.steps + (args.cpu_sample if world == 1 else 0))
    qi, qo, _ = laiv.synth_queries(QSEED, vecs, nq_total, sigma)
    mine = shard.shard_indices(nq_total, rank, world)[: args.warmup + args.steps]
    dev.stage_queries(qo[mine])
    chan = laiv.TransferChannel(b_link, laiv.ChannelMode.Device)
    log(f"[bench] rank {rank}: B_link {b_link / 1e9:.1f} GB/s, budget {budget / 1e9:.2f} GB, "
        f"sigma {sigma} (coverage {cov}), capacity {capacity / 1e9:.2f} GB")

    # e2e: the reference-facing C-ABI call (laivg_hybrid_search, the drop-in
    # for tiered.hpp:125-128) on host buffers, argument buffers bound once so
    # the timed region is the library call (query H2D and result D2H inside)
    import ctypes as C

    from paper_2502_20969_b200._lib import CostModelC, HybridTimingC, check

    e_ids = np.empty(k, np.uint64)
    e_sc = np.empty(k, np.float32)
    e_fast = np.empty(cfg["n_lists"], np.uint32)
    e_slow = np.empty(cfg["n_lists"], np.uint32)
    e_cnt, e_nf, e_ns, e_hr = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_double()
    e_tm = HybridTimingC()
    e_cm = CostModelC(32e9, 1e-3, 1e-5, 1)
    e_fn = laiv.lib().laivg_hybrid_search
    # the plain user call: no timing struct (the library then skips its
    # device-event queries); host-link bytes from the library's counters
    e_args = (dev.h, None, L, k, C.byref(e_cm), e_ids.ctypes.data, e_sc.ctypes.data,
              C.byref(e_cnt), e_fast.ctypes.data, C.byref(e_nf), e_slow.ctypes.data,
              C.byref(e_ns), C.byref(e_hr), None)
    qo_c = np.ascontiguousarray(qo, np.float32)
    lb_h, lb_d = C.c_uint64(), C.c_uint64()

    def link_bytes():
        check(laiv.lib().laivg_link_bytes(dev.h, C.byref(lb_h), C.byref(lb_d)))
        return lb_h.value, lb_d.value

    def e2e_call(qidx):
        a = list(e_args)
        a[1] = qo_c[qidx].ctypes.data
        h0, d0 = link_bytes()
        t = time.perf_counter()
        check(e_fn(*a))
        dt = time.perf_counter() - t
        h1, d1 = link_bytes()
        return (dt, e_ids[: e_cnt.value].copy(), e_sc[: e_cnt.value].copy(), h1 - h0, d1 - d0)

    def step(j, rec):
        qidx = mine[j]
        dev.store.clear()
        t0 = time.perf_counter()
        plan = laiv.plan_prefetch(dev, qi[qidx], budget)
        rp = laiv.execute_prefetch(dev, plan, chan, args.window)
        t1 = time.perf_counter()
        # the value path (query staged in HBM) and the e2e path (host buffers
        # through the C ABI) alternate which runs first, so neither always
        # sees the other's warm L2 / centroids
        if j % 2 == 0:
            got_ids, got_sc, nfast, tm = dev.hybrid_search_staged(j, L, k)
            t_e2e, e_got, _, e_h2d, e_d2h = e2e_call(qidx)
        else:
            t_e2e, e_got, _, e_h2d, e_d2h = e2e_call(qidx)
            got_ids, got_sc, nfast, tm = dev.hybrid_search_staged(j, L, k)
        if rec is not None:
            rec.append(dict(
                exposed=rp.overshoot_s, t_p=rp.t_p, window=rp.window_s, h2d_gbps=rp.h2d_gbps,
                window_read_gbps=rp.window_read_gbps,
                lat_value=rp.overshoot_s + tm.t_2, lat_e2e=rp.overshoot_s + t_e2e,
                t_scan=tm.t_scan, t_coarse=tm.t_coarse, t_g=tm.t_g, t_c=tm.t_c,
                t_kernel=tm.t_kernel,
                bytes=tm.scanned_bytes, hit=nfast / L, plan_s=t1 - t0,
                # inside the e2e call's timed region (counted by the library)
                h2d_bytes=e_h2d, d2h_bytes=e_d2h,
                # the lookahead copies run during the window; only the part
                # past its end (`exposed`) is in the retrieval latency
                prefetch_bytes=rp.bytes // member * 4 * cfg["d"],
                same=bool(np.array_equal(got_ids, e_got))))

    for j in range(args.warmup):
        step(j, None)
    if dist:
        dist.barrier()
    dev.sync()
    clocks = ClockSampler(gpu)
    launches0 = laiv.lib().laivg_kernel_launches()
    rec = []
    t0 = time.perf_counter()
    for j in range(args.warmup, args.warmup + args.steps):
        step(j, rec)
    dev.sync()
    wall = time.perf_counter() - t0
    launches = laiv.lib().laivg_kernel_launches() - launches0
    clk = clocks.stop()

    lat_v = np.array([r["lat_value"] for r in rec])
    lat_e = np.array([r["lat_e2e"] for r in rec])
    sum_v, sum_e = float(lat_v.sum()), float(lat_e.sum())
    if dist:  # the slowest rank defines the job
        sum_v, sum_e, wall = shard.max_over_ranks([sum_v, sum_e, wall])
    n_total = args.steps * world
    bytes_scan = sum(r["bytes"] for r in rec)
    t_scan = sum(r["t_scan"] for r in rec)
    t_kernel = sum(r["t_kernel"] for r in rec)
    peak, peak_kind = measured_peaks()
    fused = t_kernel > 0
    if fused:
        # one kernel per query: its algorithmic bytes are the probed resident
        # lists (reference accounting n*(4d+8)) plus the centroid matrix the
        # coarse phase reads, over its event-timed duration
        cen_bytes = cfg["n_lists"] * cfg["d"] * 4
        bytes_kernel = bytes_scan + cen_bytes * len(rec)
        kname, t_dom = "fused_query_kernel", t_kernel
    else:
        bytes_kernel, kname, t_dom = bytes_scan, f"scan_{args.scan}_kernel", t_scan
    achieved = bytes_kernel / t_dom / 1e9 if t_dom > 0 else 0.0
    exposed = np.array([r["exposed"] for r in rec])
    t_p = np.array([r["t_p"] for r in rec])
    traffic, traffic_src = (profiled_traffic(kname, args.config)
                            if args.scan == "tma" else (None, None))
    line = {
        "metric": METRIC, "value": n_total / sum_v, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sum_v / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": f"f32 data, {args.acc} accumulate" + (", fp64 re-score" if args.acc == "fp32" else ""), "data": "synthetic (planted clusters, SURVEY §8d)",
        "p50_latency_ms": float(np.median(lat_v) * 1e3),
        "p99_latency_ms": float(np.percentile(lat_v, 99) * 1e3),
        "pipeline_ms_per_step": wall / args.steps * 1e3,
        "config": config_block(cfg, args, sigma),
        "roofline": {"kernel": kname, "bound": "hbm", "achieved": achieved,
                     "peak": peak, "peak_kind": f"{peak_kind} copy (MEASURED_PEAKS.json hbm_gbs)",
                     "unit": "GB/s", "frac": achieved / peak,
                     "frac_vs_8tbps": achieved / 8000.0,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": bytes_kernel / max(len(rec), 1),
                     "avg_launch_ms": t_dom / max(len(rec), 1) * 1e3,
                     **({"bytes_note": "probed resident lists n*(4d+8) + centroids nc*d*4",
                         "scan_phase": {
                             "achieved": bytes_scan / t_scan / 1e9 if t_scan > 0 else 0.0,
                             "avg_ms": t_scan / max(len(rec), 1) * 1e3,
                             "note": "kernel time minus CTA 0's coarse + selection phase"}}
                        if fused else {})},
        "prefetch": {"h2d_gbps": float(np.mean([r["h2d_gbps"] for r in rec])),
                     "b_link_gbps": b_link / 1e9, "budget_gb": budget / 1e9,
                     "link_peak_h2d_gbps": link_h2d, "link_peak_d2h_gbps": link_d2h,
                     "h2d_frac_of_link_peak": float(np.mean([r["h2d_gbps"] for r in rec])) / link_h2d
                                              if link_h2d > 0 else None,
                     "copy_ms_mean": float(t_p.mean() * 1e3),
                     "window_ms_mean": float(np.mean([r["window"] for r in rec]) * 1e3),
                     "window_read_gbps": float(np.mean([r["window_read_gbps"] for r in rec])),
                     "hidden_frac": float(1.0 - exposed.sum() / t_p.sum()) if t_p.sum() else 1.0,
                     "exposed_ms_mean": float(exposed.mean() * 1e3),
                     "hit_rate": float(np.mean([r["hit"] for r in rec]))},
        "breakdown_ms": {k_: float(np.mean([r[k_] for r in rec]) * 1e3)
                         for k_ in ("t_coarse", "t_scan", "t_g", "t_c", "plan_s")},
        "e2e": {"value": n_total / sum_e, "unit": "queries/s",
                "p50_latency_ms": float(np.median(lat_e) * 1e3),
                "h2d_bytes_per_step": int(np.mean([r["h2d_bytes"] for r in rec])),
                "d2h_bytes_per_step": int(np.mean([r["d2h_bytes"] for r in rec])),
                "bytes_note": "host-link bytes inside the timed e2e call, counted by the "
                              "library (laivg_hybrid_timing.h2d_bytes/d2h_bytes): query row, "
                              "residency table, runtime-fetched missed lists; probe + result "
                              "lists read back",
                "prefetch_h2d_bytes_per_step": int(np.mean([r["prefetch_bytes"] for r in rec])),
                "prefetch_note": "lookahead copies during the generation window (outside the "
                                 "call); only the exposed part past the window end is in the "
                                 "latency",
                "order": "value and e2e calls alternate which runs first each step"},
        "value_e2e_results_identical": all(r["same"] for r in rec),
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        ri = reference_index(cen, np.asarray(vecs), ids, off, int(metric))
        threads = os.cpu_count() or 1
        sample = args.cpu_sample
        # the timed queries first, then more of the same generator
        cb = cpu_baseline(ri, qo[args.warmup:args.warmup + sample], L, k, threads, sample)
        # parity with the reference on the same inputs: every query of the
        # CPU sample (the timed ones first), through the C-ABI e2e call
        npar = sample
        eq = 0
        for j in range(npar):
            _, got_ids, got_sc, _, _ = e2e_call(args.warmup + j)
            eq += bool(np.array_equal(got_ids, cb["ids"][j]) and
                       np.array_equal(got_sc, cb["scores"][j]))
        line["cpu_baseline"] = {"value": cb["qps"], "unit": "queries/s", "cores": threads,
                                "kind": "reference", "cpu_model": host_cpu_model(),
                                "single_thread_latency_ms": cb["p50_ms"],
                                "p50_latency_ms": cb["p50_ms"], "wall_s": cb["wall_s"],
                                "cpu_seconds": cb["wall_s"] * threads,
                                "sample": f"{sample} q_out queries of the bench generator (the "
                                          f"{npar} timed ones first), laiv::ivf_search "
                                          f"(oracle/_ref) one query per host thread"}
        line["parity_vs_reference"] = {"queries": npar, "bit_identical": eq}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def run_ours_batch(args, cfg):
    """Micro-batch pipeline round (pipeline.cpp:346-441) on one GPU per rank:
    clear cache -> lookahead prefetch of the batch (one window, per-query
    budgets from split_budget) -> batched hybrid search of the batch's q_out.
    Retrieval latency of a batch = exposed H2D + the batched hybrid search."""
    from paper_2502_20969_b200 import laiv, shard

    rank, world, local = dist_env()
    dist = None
    dist, gpu = init_dist(world, local)
    pin_rank_cores(rank, world)
    B = cfg["batch"]
    cen, vecs, ids, off = make_datastore(cfg, world, rank)
    metric = laiv.Metric.InnerProduct if args.metric == "ip" else laiv.Metric.L2
    ix = laiv.IvfIndex(cen, vecs, ids, off, metric, borrow=True, trust=True)
    member = 4 * cfg["d"] + 8
    capacity = int(cfg["cache_frac"] * cfg["n_lists"]) * cfg["per_list"] * member
    dev = laiv.Device(ix, capacity, device=gpu, max_batch=B, miss_threads=host_threads(world),
                      acc_fp64=args.acc == "fp64", scan_impl=args.scan)
    L, k = cfg["nprobe"], cfg["k"]
    probe_plan = laiv.plan_prefetch(dev, cen[0], min(capacity, 64 * cfg["per_list"] * member))
    rep = laiv.execute_prefetch(dev, probe_plan, laiv.TransferChannel(1, laiv.ChannelMode.Device))
    dev.store.clear()
    b_link = rep.h2d_gbps * 1e9
    resident_all = bool(cfg.get("resident_all"))
    if resident_all:  # the whole index in HBM once; no per-step prefetch
        for c in range(cfg["n_lists"]):
            dev.store.insert(c)
        dev.sync()
    budget = int(min(b_link * args.window * args.budget_scale, capacity))
    budgets = laiv.split_budget(budget, laiv.MicroBatch(list(range(B))))
    sigma, cov = q_out_sigma(args, cfg, laiv, dev, vecs, L)
    nsteps = args.warmup + args.steps
    nq_total = nsteps * B * world
    qi, qo, _ = laiv.synth_queries(QSEED, vecs, nq_total, sigma)
    mine = np.concatenate([np.arange((j * world + rank) * B, (j * world + rank + 1) * B)
                           for j in range(nsteps)])
    dev.stage_queries(qo[mine])
    chan = laiv.TransferChannel(b_link, laiv.ChannelMode.Device)
    log(f"[bench] rank {rank}: batch {B}, B_link {b_link / 1e9:.1f} GB/s, budget "
        f"{budget / 1e9:.2f} GB ({budgets[0] / 1e6:.0f} MB/query), sigma {sigma} "
        f"(coverage {cov}), capacity {capacity / 1e9:.2f} GB")

    def step(j, rec):
        sel = mine[j * B:(j + 1) * B]
        t0 = time.perf_counter()
        if resident_all:
            rp = laiv.TransferReport(0.0, [], 0, 0.0, 0.0, 0.0, 0.0)
        else:
            dev.store.clear()
            rp, npl = laiv.prefetch_batch(dev, qi[sel], budgets, chan, args.window)
        t1 = time.perf_counter()
        got_ids, got_sc, cnt, nfast, tm = dev.hybrid_search_batch_staged(j * B, B, L, k)
        t2 = time.perf_counter()
        res, tm2 = laiv.hybrid_search_batch(dev, qo[sel], L, k)
        t3 = time.perf_counter()
        if rec is not None:
            nhit = int(nfast.sum())
            rec.append(dict(
                exposed=rp.overshoot_s, t_p=rp.t_p, window=rp.window_s, h2d_gbps=rp.h2d_gbps,
                window_read_gbps=rp.window_read_gbps,
                lat_value=rp.overshoot_s + tm.t_2, lat_e2e=rp.overshoot_s + (t3 - t2),
                t_scan=tm.t_scan, t_coarse=tm.t_coarse, t_g=tm.t_g, t_c=tm.t_c, t_2=tm.t_2,
                bytes=tm.scanned_bytes, hit=nhit / (B * L), plan_s=t1 - t0,
                fetched_lists=tm.fetched_lists, cpu_lists=tm.cpu_lists,
                fetched_bytes=tm.fetched_bytes, t_fetch=tm.t_fetch,
                miss_bytes=(B * L - nhit) * cfg["per_list"] * 4 * cfg["d"],
                prefetched=len(rp.transferred),
                h2d_bytes=B * 4 * cfg["d"] * 2 + rp.bytes // member * 4 * cfg["d"],
                d2h_bytes=B * (L * 4 + k * 12 + 8),
                list_scan=tm.list_scan, distinct=tm.distinct_bytes,
                same=bool(np.array_equal(got_ids, res.ids))))

    for j in range(args.warmup):
        step(j, None)
    if dist:
        dist.barrier()
    dev.sync()
    clocks = ClockSampler(gpu)
    launches0 = laiv.lib().laivg_kernel_launches()
    rec = []
    t0 = time.perf_counter()
    for j in range(args.warmup, nsteps):
        step(j, rec)
    dev.sync()
    wall = time.perf_counter() - t0
    launches = laiv.lib().laivg_kernel_launches() - launches0
    clk = clocks.stop()
    lat_v = np.array([r["lat_value"] for r in rec])
    lat_e = np.array([r["lat_e2e"] for r in rec])
    sum_v, sum_e = float(lat_v.sum()), float(lat_e.sum())
    if dist:
        sum_v, sum_e, wall = shard.max_over_ranks([sum_v, sum_e, wall])
    n_total = args.steps * B * world
    bytes_scan = sum(r["bytes"] for r in rec)
    t_scan = sum(r["t_scan"] for r in rec)
    peak, peak_kind = measured_peaks()
    list_scan = all(r["list_scan"] for r in rec)
    if list_scan:  # list-major scan: each distinct list is read (at least) once
        kname = "list_scan_tc_kernel"
        alg_bytes = sum(r["distinct"] for r in rec)
        alg_note = ("distinct resident probed lists, n*4d B each (the list-major scan reads "
                    "each once per 16 probing queries; the per-query scan would read the "
                    f"{bytes_scan / max(len(rec), 1) / 1e9:.1f} GB of (query, list) pairs)")
    else:
        kname = f"scan_{args.scan}_kernel"
        alg_bytes = bytes_scan
        alg_note = "every (query, resident probed list) pair, n*(4d+8) B (SURVEY §8d)"
    achieved = alg_bytes / t_scan / 1e9 if t_scan > 0 else 0.0
    traffic, traffic_src = profiled_traffic(kname, args.config)
    exposed = np.array([r["exposed"] for r in rec])
    t_p = np.array([r["t_p"] for r in rec])
    t_c = np.array([r["t_c"] for r in rec])
    miss_b = np.array([r["miss_bytes"] for r in rec])
    line = {
        "metric": METRIC, "value": n_total / sum_v, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sum_v / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": f"f32 data, {args.acc} accumulate", "data": "synthetic (planted clusters, SURVEY §8d)",
        "p50_latency_ms": float(np.median(lat_v) * 1e3),
        "p50_batch_note": "latency of one micro-batch of queries (all returned together)",
        "pipeline_ms_per_step": wall / args.steps * 1e3,
        "config": config_block(cfg, args, sigma),
        "roofline": {"kernel": kname, "bound": "hbm", "achieved": achieved,
                     "peak": peak, "peak_kind": f"{peak_kind} copy (MEASURED_PEAKS.json hbm_gbs)",
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": alg_bytes / max(len(rec), 1),
                     "algorithmic_bytes_are": alg_note,
                     "timed_as": "device events around the batch's whole scan phase "
                                 "(list scan: plan + scan + final kernels)",
                     "avg_launch_ms": t_scan / max(len(rec), 1) * 1e3},
        "miss_path": {"host_scan_ms_mean": float(t_c.mean() * 1e3),
                      "host_bytes_mean_gb": float(miss_b.mean() / 1e9),
                      "host_gbps_per_query_bytes": float(miss_b.sum() / t_c.sum() / 1e9)
                      if t_c.sum() else 0.0,
                      "host_threads": os.cpu_count(),
                      "runtime_fetch": {
                          "lists_mean": float(np.mean([r["fetched_lists"] for r in rec])),
                          "host_lists_mean": float(np.mean([r["cpu_lists"] for r in rec])),
                          "gb_mean": float(np.mean([r["fetched_bytes"] for r in rec]) / 1e9),
                          "copy_ms_mean": float(np.mean([r["t_fetch"] for r in rec]) * 1e3),
                          "h2d_gbps": float(sum(r["fetched_bytes"] for r in rec) /
                                            max(sum(r["t_fetch"] for r in rec), 1e-12) / 1e9)}},
        "prefetch": {"h2d_gbps": float(np.mean([r["h2d_gbps"] for r in rec])),
                     "b_link_gbps": b_link / 1e9, "budget_gb": budget / 1e9,
                     "hidden_frac": float(1.0 - exposed.sum() / t_p.sum()) if t_p.sum() else 1.0,
                     "exposed_ms_mean": float(exposed.mean() * 1e3),
                     "hit_rate": float(np.mean([r["hit"] for r in rec])),
                     "lists_prefetched_mean": float(np.mean([r["prefetched"] for r in rec]))},
        "breakdown_ms": {k_: float(np.mean([r[k_] for r in rec]) * 1e3)
                         for k_ in ("t_coarse", "t_scan", "t_g", "t_c", "t_2", "plan_s")},
        "e2e": {"value": n_total / sum_e, "unit": "queries/s",
                "p50_latency_ms": float(np.median(lat_e) * 1e3),
                "h2d_bytes_per_step": int(np.mean([r["h2d_bytes"] for r in rec])),
                "d2h_bytes_per_step": int(np.mean([r["d2h_bytes"] for r in rec]))},
        "value_e2e_results_identical": all(r["same"] for r in rec),
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        ri = reference_index(cen, np.asarray(vecs), ids, off, int(metric))
        threads = os.cpu_count() or 1
        sample = min(args.cpu_sample, args.steps * B)
        tq = mine[args.warmup * B: args.warmup * B + sample]
        cb = cpu_baseline(ri, qo[tq], L, k, threads, sample)
        eq = 0
        got_ids, got_sc, _, _, _ = dev.hybrid_search_batch_staged(args.warmup * B, B, L, k)
        for j in range(min(sample, B)):
            eq += bool(np.array_equal(got_ids[j], cb["ids"][j]) and
                       np.array_equal(got_sc[j], cb["scores"][j]))
        line["cpu_baseline"] = {"value": cb["qps"], "unit": "queries/s", "cores": threads,
                                "kind": "reference", "p50_latency_ms": cb["p50_ms"],
                                "sample": f"{sample} of the timed q_out queries, "
                                          f"laiv::ivf_search (oracle/_ref) one query per host "
                                          f"thread"}
        line["parity_vs_reference"] = {"queries": min(sample, B), "bit_identical": eq}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def run_ours_routed(args, cfg):
    """C4: per step, 256 topical queries are grouped into micro-batches of 4
    (group_microbatches on q_in, sched.cpp:39-70), routed to the workers by
    assign_cache_aware over every worker's resident set (sched.cpp:87-144;
    all-gathered across ranks), and each worker serves its micro-batches as
    ONE device batch: batched lookahead prefetch (one window, split_budget
    per query, budget clamped to capacity x (1 - cache fraction),
    pipeline.cpp:146-166) then batched hybrid search; its cache is kept
    across steps by the hotness policy (end_of_round + evict_to_fraction,
    pipeline.cpp:466-473). Step time = max over workers."""
    from paper_2502_20969_b200 import laiv, shard

    rank, world, local = dist_env()
    dist = None
    dist, gpu = init_dist(world, local)
    emulated = world == 1 and args.workers > 1
    W = world if world > 1 else max(1, args.workers)
    pin_rank_cores(rank, world)
    B, m = cfg["batch"], cfg["micro"]
    cen, vecs, ids, off = make_datastore(cfg, world, rank)
    metric = laiv.Metric.InnerProduct if args.metric == "ip" else laiv.Metric.L2
    ix = laiv.IvfIndex(cen, vecs, ids, off, metric, borrow=True, trust=True)
    member = 4 * cfg["d"] + 8
    capacity = int(cfg["cache_frac"] * cfg["n_lists"]) * cfg["per_list"] * member
    mine = list(range(W)) if emulated or world == 1 else [rank]
    # emulated workers get the host share a real W-GPU node would give each
    # rank (cores / W), not the whole host
    devs = {w: laiv.Device(ix, capacity, device=gpu,
                           max_batch=max(m, 32), miss_threads=host_threads(W),
                           acc_fp64=args.acc == "fp64", scan_impl=args.scan) for w in mine}
    params = laiv.CacheParams(cache_fraction=cfg["hot_fraction"])
    hot = {w: laiv.HotnessTable(params) for w in mine}
    # peer caches: every worker may copy another worker's cached lists
    # (in-process contexts, or CUDA IPC handles of the other ranks' slabs)
    peer_ids = {}  # (worker, peer worker) -> peer slot
    if args.peers:
        if world > 1:
            import torch.distributed as tdist

            handles = [None] * world
            tdist.all_gather_object(handles, devs[rank].slab_ipc_handle())
            others = [p for p in range(world) if p != rank]
            for i, p in enumerate(others):
                devs[rank].peer_attach(i, ipc_handle=handles[p])
                peer_ids[(rank, p)] = i
        else:
            for w in mine:
                others = [p for p in mine if p != w]
                for i, p in enumerate(others):
                    devs[w].peer_attach(i, other=devs[p])
                    peer_ids[(w, p)] = i
    d0 = devs[mine[0]]
    L, k = cfg["nprobe"], cfg["k"]
    probe_plan = laiv.plan_prefetch(d0, cen[0], min(capacity, 64 * cfg["per_list"] * member))
    rep = laiv.execute_prefetch(d0, probe_plan, laiv.TransferChannel(1, laiv.ChannelMode.Device))
    d0.store.clear()
    b_link = rep.h2d_gbps * 1e9
    budget = int(min(b_link * args.window, capacity * (1.0 - cfg["hot_fraction"])))
    sigma = args.sigma or cfg.get("sigma", 0.008)
    nsteps = args.warmup + args.steps
    qi, qo, _, topic = laiv.synth_queries_topical(QSEED, cen, vecs, off, nsteps * B, sigma,
                                                  cfg["topics"], cfg["zipf"], cfg["neigh"])
    chan = laiv.TransferChannel(b_link, laiv.ChannelMode.Device)
    log(f"[bench] rank {rank}: {W} worker(s){' emulated on cuda:0' if emulated else ''}, "
        f"B_link {b_link / 1e9:.1f} GB/s, prefetch budget {budget / 1e9:.2f} GB, capacity "
        f"{capacity / 1e9:.2f} GB, {cfg['topics']} topics zipf {cfg['zipf']}")

    def serve(w, mbs, rec_w):
        """Worker w serves its micro-batches in order (pipeline.cpp:574-589): per
        micro-batch, lookahead prefetch (budget split over its queries, one
        window), batched hybrid search, then cache maintenance."""
        dev, h = devs[w], hot[w]
        acc = dict(lat=0.0, lat_e2e=0.0, nq=0, hit=0, exposed=0.0, t_scan=0.0, bytes=0,
                   fetched=0, peer=0, t_c=0.0, same=True)
        if mbs:
            dev.stage_queries(qo[np.concatenate(mbs)])
        q0 = 0
        for sel in mbs:
            n = len(sel)
            budgets = laiv.split_budget(budget, laiv.MicroBatch(list(range(n))))
            rp, _ = laiv.prefetch_batch(dev, qi[sel], budgets, chan, args.window)
            for c in rp.transferred:
                h.on_fetch(c)
            got_ids, got_sc, cnt, nfast, tm = dev.hybrid_search_batch_staged(q0, n, L, k)
            t2 = time.perf_counter()
            res, _ = laiv.hybrid_search_batch(dev, qo[sel], L, k)
            t3 = time.perf_counter()
            q0 += n
            # cache maintenance between batches (pipeline.cpp:466-473)
            used = set(np.unique(laiv.coarse_probe(dev, qo[sel], L)).tolist())
            h.end_of_round(used)
            h.evict_to_fraction(dev)
            acc["lat"] += rp.overshoot_s + tm.t_2
            acc["lat_e2e"] += rp.overshoot_s + (t3 - t2)
            acc["nq"] += n
            acc["hit"] += int(nfast.sum())
            acc["exposed"] += rp.overshoot_s
            acc["t_scan"] += tm.t_scan
            acc["bytes"] += tm.scanned_bytes
            acc["fetched"] += tm.fetched_lists
            acc["peer"] += tm.peer_lists
            acc["t_c"] += tm.t_c
            acc["same"] = acc["same"] and bool(np.array_equal(got_ids, res.ids))
        rec_w.update(acc)

    def step(j, rec):
        g0 = j * B
        tr0 = time.perf_counter()
        # routing input: every worker's resident set (control plane)
        if world > 1:
            resident = shard.gather_resident(devs[rank].store.resident_mask(cfg["n_lists"]))
        else:
            resident = np.stack([devs[w].store.resident_mask(cfg["n_lists"]) for w in range(W)])
        # group_microbatches + probes + overlap popcounts on the GPU, greedy on
        # the host (identical on every rank: deterministic inputs)
        batches, assign, _ = laiv.schedule(d0, qi[g0:g0 + B], m, L, resident)
        t_route = time.perf_counter() - tr0
        if args.peers:  # epoch: every worker publishes its cache for this step
            for w in mine:
                devs[w].epoch_open()
            if world > 1:
                import torch.distributed as tdist

                offs = [None] * world
                tdist.all_gather_object(offs, devs[rank].store_offsets())
            else:
                offs = {w: devs[w].store_offsets() for w in mine}
            for (w, p), i in peer_ids.items():
                devs[w].peer_publish(i, offs[p])
        per = {}
        for w in mine:
            mbs = [np.asarray([g0 + q for q in mb.queries], dtype=np.int64)
                   for b, mb in enumerate(batches) if assign[b] == w and mb.queries]
            r = {}
            serve(w, mbs, r)
            per[w] = r
        if args.peers:
            if dist:
                dist.barrier()  # peers keep their lists until every rank is done
            for w in mine:
                devs[w].epoch_close()
        if rec is not None:
            rec.append(dict(
                lat=max(r["lat"] for r in per.values()),
                lat_e2e=max(r["lat_e2e"] for r in per.values()),
                nq={w: r["nq"] for w, r in per.items()},
                hit=sum(r["hit"] for r in per.values()) / (sum(r["nq"] for r in per.values()) * L
                                                           or 1),
                t_scan=sum(r["t_scan"] for r in per.values()),
                bytes=sum(r["bytes"] for r in per.values()),
                fetched=sum(r["fetched"] for r in per.values()),
                peer=sum(r["peer"] for r in per.values()),
                t_c=max(r["t_c"] for r in per.values()),
                exposed=max(r["exposed"] for r in per.values()),
                route=t_route,
                same=all(r["same"] for r in per.values())))

    for j in range(args.warmup):
        step(j, None)
    if dist:
        dist.barrier()
    for dv in devs.values():
        dv.sync()
    clocks = ClockSampler(gpu)
    launches0 = laiv.lib().laivg_kernel_launches()
    rec = []
    t0 = time.perf_counter()
    for j in range(args.warmup, nsteps):
        step(j, rec)
    for dv in devs.values():
        dv.sync()
    wall = time.perf_counter() - t0
    launches = laiv.lib().laivg_kernel_launches() - launches0
    clk = clocks.stop()
    lat = np.array([r["lat"] for r in rec])
    lat_e = np.array([r["lat_e2e"] for r in rec])
    if dist:  # per-step makespan: the slowest rank of each step
        lat = np.array(shard.max_over_ranks(lat.tolist()))
        lat_e = np.array(shard.max_over_ranks(lat_e.tolist()))
        wall = shard.max_over_ranks([wall])[0]
    n_total = args.steps * B
    t_scan = sum(r["t_scan"] for r in rec)
    bytes_scan = sum(r["bytes"] for r in rec)
    peak, peak_kind = measured_peaks()
    achieved = bytes_scan / t_scan / 1e9 if t_scan > 0 else 0.0
    line = {
        "metric": METRIC, "value": n_total / float(lat.sum()), "unit": "queries/s",
        "n_gpus": world, "workers": W, "emulated_workers": emulated,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(lat.mean() * 1e3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": f"f32 data, {args.acc} accumulate",
        "data": "synthetic (planted clusters, Zipf-topical queries, SURVEY §8d)",
        "p50_latency_ms": float(np.median(lat) * 1e3),
        "p50_batch_note": "makespan of one 256-query step over the workers",
        "pipeline_ms_per_step": wall / args.steps * 1e3,
        "config": dict(config_block(cfg, args, sigma), micro_batch=m, topics=cfg["topics"],
                       zipf=cfg["zipf"], hot_fraction=cfg["hot_fraction"],
                       routing="group_microbatches + assign_cache_aware"),
        "roofline": {"kernel": f"scan_{args.scan}_kernel", "bound": "hbm", "achieved": achieved,
                     "peak": peak, "peak_kind": f"{peak_kind} copy (MEASURED_PEAKS.json hbm_gbs)",
                     "unit": "GB/s", "frac": achieved / peak, "traffic": None},
        "routing": {"hit_rate": float(np.mean([r["hit"] for r in rec])),
                    "queries_per_worker_mean": {str(w): float(np.mean([r["nq"].get(w, 0)
                                                                       for r in rec]))
                                                for w in mine},
                    "fetched_lists_mean": float(np.mean([r["fetched"] for r in rec])),
                    "peer_lists_mean": float(np.mean([r["peer"] for r in rec])),
                    "peer_caches": bool(args.peers),
                    "host_scan_ms_max_mean": float(np.mean([r["t_c"] for r in rec]) * 1e3),
                    "exposed_ms_mean": float(np.mean([r["exposed"] for r in rec]) * 1e3),
                    "schedule_ms_mean": float(np.mean([r["route"] for r in rec]) * 1e3),
                    "schedule_note": "laivg_schedule: GPU grouping + GPU coarse probes + GPU "
                                     "overlap popcounts + host greedy, plus the resident-set "
                                     "all-gather, per 256-query step (not in the retrieval "
                                     "latency, as in pipeline.cpp:541-589)"},
        "e2e": {"value": n_total / float(lat_e.sum()), "unit": "queries/s",
                "p50_latency_ms": float(np.median(lat_e) * 1e3),
                "h2d_bytes_per_step": B * 4 * cfg["d"] * 2, "d2h_bytes_per_step": B * (k * 12 + 8)},
        "value_e2e_results_identical": all(r["same"] for r in rec),
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if emulated:
        line["emulation_note"] = ("workers share one GPU, its PCIe link and the host cores but "
                                  "run one after another; each worker's time is measured alone "
                                  "and the step takes the max (the reference's makespan rule, "
                                  "pipeline.cpp:604-605)")
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0



def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--metric", default="ip", choices=["ip", "l2"])
    ap.add_argument("--window", type=float, default=None)
    ap.add_argument("--sigma", type=float, default=None,
                    help="q_out noise; default the config's (0.008, coverage ~0.8); "
                         "negative: recalibrate for coverage >= 0.8")
    ap.add_argument("--cpu-sample", type=int, default=128,
                    help="queries in the reference CPU baseline sample (C2: ~20 s of CPU "
                         "work on 16 host threads)")
    ap.add_argument("--peers", action="store_true",
                    help="routed configs: misses cached by another worker are copied from "
                         "that worker's HBM cache (NVLink) instead of going to the host")
    ap.add_argument("--workers", type=int, default=0,
                    help="routed configs on one process: emulate this many GPU workers "
                         "(separate contexts and caches on cuda:0, run one after another; "
                         "the step time is the max over workers)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--acc", default="fp64", choices=["fp64", "fp32"],
                    help="scan accumulation: fp64 for every candidate as the reference "
                         "(default) or fp32 FMA + exact fp64 re-score of the survivors")
    ap.add_argument("--scan", default="tma", choices=["tma", "ldg"],
                    help="scan kernel: TMA bulk-copy staged (default) or direct LDG")
    ap.add_argument("--budget-scale", type=float, default=1.0,
                    help="lookahead budget = scale x B_link x window (capped by the cache); "
                         "above 1 the copies outlast the window (prefetch-hiding stress)")
    ap.add_argument("--window-load", type=float, default=None,
                    help="decode-like window: GB/s target read rate of the streamed "
                         "buffer (default: the config's, 0 = idle window)")
    ap.add_argument("--window-buffer-gb", type=float, default=None,
                    help="decode-like window: streamed buffer size in GB")
    ap.add_argument("--single", default="fused", choices=["fused", "chain"],
                    help="single-query search: one fused cooperative kernel (default) or "
                         "the multi-kernel chain")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.window is None:
        args.window = cfg["window_s"]
    if args.window_load is None:
        args.window_load = cfg.get("window_load_gbps", 0.0)
    if args.window_buffer_gb is None:
        args.window_buffer_gb = cfg.get("window_buffer_gb", 16.0)
    if args.impl == "reference":
        return run_reference(args, cfg)
    if cfg.get("routed"):
        return run_ours_routed(args, cfg)
    if cfg.get("batch", 1) > 1:
        return run_ours_batch(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
