"""The reference's pipeline caller (pipeline.hpp / pipeline.cpp, trace.hpp /
trace.cpp) driving the B200 hot path: trace replay with lookahead prefetch,
micro-batching, cache-aware routing and hotness-managed caches, one Device
(GPU cluster cache) per worker.

Two clocks, as the reference has:
  * ChannelMode.SimulatedClock (default): every retrieval, prefetch plan and
    cache decision runs on the GPU, and the phase times follow the
    reference's cost model (t_p = bytes / B, t_c = ceil(slow / P) * t_cc,
    t_g = fast * t_gc; pipeline.cpp:346-441). The RunRecord then equals the
    reference's run_batch record field for field (tests/test_gpu_pipeline.py,
    against records the unmodified reference wrote).
  * ChannelMode.Device: the same replay with MEASURED times: each round's
    prefetch streams on the copy engine under a generation-window kernel of
    the round's window length (times `time_scale`), t_p is the measured copy,
    and the retrieval times are the measured hybrid-search times.

Traces, sidecar and configs use the reference's file formats (load_traces /
save_traces JSONL, load_config key = value, save_records JSONL).
"""
from __future__ import annotations

import enum
import json
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import laiv


# ---------------------------------------------------------------------------
# traces (trace.hpp:16-97)
# ---------------------------------------------------------------------------
class StageKind(enum.IntEnum):                                      # trace.hpp:16
    Generate = 0
    Retrieve = 1
    Judge = 2


class PipelineKind(enum.IntEnum):                                   # trace.hpp:21-29
    HyDE = 0
    SubQ = 1
    Iter = 2
    IRG = 3
    FLARE = 4
    SRag = 5
    Custom = 6


_PIPE_NAMES = {PipelineKind.HyDE: "HyDE", PipelineKind.SubQ: "SubQ", PipelineKind.Iter: "Iter",
               PipelineKind.IRG: "IRG", PipelineKind.FLARE: "FLARE", PipelineKind.SRag: "S-RAG",
               PipelineKind.Custom: "custom"}


def pipeline_name(p: PipelineKind) -> str:                          # trace.cpp:72-83
    return _PIPE_NAMES[PipelineKind(p)]


def pipeline_from_name(name: str) -> PipelineKind:                  # trace.cpp:85-90
    for p, n in _PIPE_NAMES.items():
        if n == name:
            return p
    raise ValueError("unknown pipeline: " + name)


@dataclass
class Stage:                                                        # trace.hpp:41-48
    kind: StageKind = StageKind.Generate
    embedding_ref: int = -1
    duration_s: float = 0.0
    fanout: int = 1


@dataclass
class QueryTrace:                                                   # trace.hpp:53-59
    trace_id: int = 0
    pipeline: PipelineKind = PipelineKind.Custom
    stages: list[Stage] = field(default_factory=list)


def _stage_from_json(j) -> Stage:                                   # trace.cpp:30-43
    s = Stage(StageKind[j["kind"]] if j["kind"] in StageKind.__members__ else None,
              int(j["embedding_ref"]), float(j["duration_s"]), int(j["fanout"]))
    if s.kind is None:
        raise ValueError("unknown stage kind: " + str(j["kind"]))
    if s.duration_s < 0.0:
        raise ValueError("negative stage duration")
    if s.fanout < 1:
        raise ValueError("fanout must be >= 1")
    return s


def load_traces(path) -> list[QueryTrace]:                          # trace.cpp:117-154
    try:
        f = open(path)
    except OSError:
        raise RuntimeError(f"cannot open: {path}") from None
    out = []
    with f:
        for lineno, line in enumerate(f, 1):
            line = line.rstrip("\n")
            if not line:
                continue
            try:
                rec = json.loads(line)
                if int(rec["schema_version"]) != 1:
                    raise ValueError(f"schema_version {rec['schema_version']} does not match "
                                     "expected 1")
                out.append(QueryTrace(int(rec["trace_id"]), pipeline_from_name(rec["pipeline"]),
                                      [_stage_from_json(s) for s in rec["stages"]]))
            except Exception as e:  # noqa: BLE001 - the reference wraps every error
                raise RuntimeError(f"{path}:{lineno}: {e}") from None
    return out


def save_traces(path, traces: list[QueryTrace]) -> None:           # trace.cpp:97-115
    with open(path, "w") as f:
        for t in traces:
            f.write(json.dumps({"schema_version": 1, "trace_id": t.trace_id,
                                "pipeline": pipeline_name(t.pipeline),
                                "stages": [{"kind": s.kind.name, "embedding_ref": s.embedding_ref,
                                            "duration_s": s.duration_s, "fanout": s.fanout}
                                           for s in t.stages]}) + "\n")


def validate_traces(traces: list[QueryTrace], sidecar_count: int) -> None:  # trace.cpp:156-184
    for t in traces:
        where = f"trace {t.trace_id}"
        have_ref = False
        for s in t.stages:
            if s.embedding_ref >= 0 and s.embedding_ref + s.fanout > sidecar_count:
                raise RuntimeError(f"{where}: embedding_ref {s.embedding_ref} (+fanout "
                                   f"{s.fanout}) dangles past sidecar of {sidecar_count}")
            if s.kind == StageKind.Retrieve:
                if s.embedding_ref < 0:
                    raise RuntimeError(f"{where}: Retrieve stage has no query")
                if not have_ref:
                    raise RuntimeError(f"{where}: Retrieve has no preceding stage with an "
                                       "embedding")
            if s.embedding_ref >= 0:
                have_ref = True


@dataclass
class TracePhase:                                                   # pipeline.hpp:165-170
    plain_before_s: float = 0.0
    window_s: float = 0.0
    predictor_ref: int = -1
    query_refs: list[int] = field(default_factory=list)


@dataclass
class TraceWalk:                                                    # pipeline.hpp:172-175
    phases: list[TracePhase] = field(default_factory=list)
    tail_s: float = 0.0


def decompose_trace(trace: QueryTrace) -> TraceWalk:                # pipeline.cpp:231-290
    st = trace.stages
    # the stage right before a Retrieve opens its overlap window
    win = [False] * len(st)
    for i in range(1, len(st)):
        if st[i].kind == StageKind.Retrieve and st[i - 1].kind != StageKind.Retrieve:
            win[i - 1] = True
    walk, plain = TraceWalk(), 0.0
    for i, s in enumerate(st):
        if s.kind != StageKind.Retrieve:
            if not win[i]:
                plain += s.duration_s
            continue
        if s.embedding_ref < 0:
            raise RuntimeError(f"trace {trace.trace_id}: Retrieve stage without a query")
        has_win = i > 0 and win[i - 1]
        ph = TracePhase(plain_before_s=plain, window_s=st[i - 1].duration_s if has_win else 0.0)
        plain = 0.0
        # the latest embedding available when the window starts: a Judge's
        # ref is its input (counts for its own window), a Generate's its output
        pred = -1
        if has_win and st[i - 1].kind == StageKind.Judge and st[i - 1].embedding_ref >= 0:
            pred = st[i - 1].embedding_ref
        if pred < 0:
            for j in range((i - 1 if has_win else i) - 1, -1, -1):
                if st[j].embedding_ref >= 0:
                    pred = st[j].embedding_ref
                    break
        ph.predictor_ref = pred if pred >= 0 else s.embedding_ref
        ph.query_refs = [s.embedding_ref + f for f in range(s.fanout)]
        walk.phases.append(ph)
    walk.tail_s = plain
    return walk


# ---------------------------------------------------------------------------
# configuration (pipeline.hpp:18-60)
# ---------------------------------------------------------------------------
@dataclass
class RunFlags:                                                     # pipeline.hpp:18-23
    lookahead_on: bool = True
    prefetch_sched_on: bool = False
    cache_sched_on: bool = False
    cache_on: bool = False


@dataclass
class RunConfig:                                                    # pipeline.hpp:25-57
    n_probe: int = 16
    top_k: int = 3
    prefetch_budget_bytes: int = 0
    capacity_bytes: int = 0
    cache_fraction: float = 0.5
    cost: laiv.CostModel = field(default_factory=laiv.CostModel)
    workers: int = 1
    micro_batch: int = 1
    mode: laiv.ChannelMode = laiv.ChannelMode.SimulatedClock
    flags: RunFlags = field(default_factory=RunFlags)
    h_init: float = 1.0
    h_inc: float = 1.0
    decay: float = 2.0
    warmup_traces: int = 0
    validate_exactness: bool = True
    seed: int = 0
    time_scale: float = 1.0  # Device mode: window kernel length = window_s * time_scale

    def cache_params(self) -> laiv.CacheParams:
        return laiv.CacheParams(self.h_init, self.h_inc, self.decay, self.cache_fraction)

    def validate_and_clamp(self) -> str:                            # pipeline.cpp:146-168
        self.cost.validate()
        if self.n_probe < 1 or self.top_k < 1:
            raise ValueError("n_probe and top_k must be >= 1")
        if self.workers < 1 or self.micro_batch < 1:
            raise ValueError("workers and micro_batch must be >= 1")
        if self.flags.cache_on:
            _validate_cache(self.cache_params())
        reserved = self.cache_fraction if self.flags.cache_on else 0.0
        cap = int(float(self.capacity_bytes) * (1.0 - reserved))
        if self.flags.lookahead_on and self.prefetch_budget_bytes > cap:
            w = (f"prefetch_budget_bytes {self.prefetch_budget_bytes} exceeds the usable "
                 f"capacity {cap}, clamping")
            self.prefetch_budget_bytes = cap
            return w
        return ""


def _validate_cache(p: laiv.CacheParams) -> None:                   # cache.cpp:11-21
    if p.h_init <= 0.0 or p.h_inc <= 0.0:
        raise ValueError("h_init and h_inc must be positive")
    if p.decay <= 1.0:
        raise ValueError("decay factor must exceed 1")
    if p.cache_fraction <= 0.0 or p.cache_fraction > 1.0:
        raise ValueError("cache_fraction must be in (0, 1]")


def _bool(v: str) -> bool:
    if v in ("true", "1", "on"):
        return True
    if v in ("false", "0", "off"):
        return False
    raise ValueError(f"expected a boolean, got '{v}'")


def _u64(v: str) -> int:
    d = float(v)
    if d < 0.0 or d != math.floor(d) or d > 9.007199254740992e15:
        raise ValueError(f"expected a non-negative integer, got '{v}'")
    return int(d)


def _set_cost(c: RunConfig, **kw):
    c.cost = laiv.CostModel(**{**c.cost.__dict__, **kw})


_FIELDS = {  # key -> setter (pipeline.cpp:57-127)
    "n_probe": lambda c, v: setattr(c, "n_probe", int(v)),
    "top_k": lambda c, v: setattr(c, "top_k", int(v)),
    "prefetch_budget_bytes": lambda c, v: setattr(c, "prefetch_budget_bytes", _u64(v)),
    "capacity_bytes": lambda c, v: setattr(c, "capacity_bytes", _u64(v)),
    "cache_fraction": lambda c, v: setattr(c, "cache_fraction", float(v)),
    "bandwidth_bytes_per_s": lambda c, v: _set_cost(c, bandwidth_bytes_per_s=float(v)),
    "t_cc": lambda c, v: _set_cost(c, t_cc=float(v)),
    "t_gc": lambda c, v: _set_cost(c, t_gc=float(v)),
    "parallel_slots": lambda c, v: _set_cost(c, parallel_slots=int(v)),
    "workers": lambda c, v: setattr(c, "workers", int(v)),
    "micro_batch": lambda c, v: setattr(c, "micro_batch", int(v)),
    "mode": lambda c, v: setattr(c, "mode", {"simulated": laiv.ChannelMode.SimulatedClock,
                                             "measured": laiv.ChannelMode.Measured,
                                             "device": laiv.ChannelMode.Device}[v]),
    "lookahead_on": lambda c, v: setattr(c.flags, "lookahead_on", _bool(v)),
    "prefetch_sched_on": lambda c, v: setattr(c.flags, "prefetch_sched_on", _bool(v)),
    "cache_sched_on": lambda c, v: setattr(c.flags, "cache_sched_on", _bool(v)),
    "cache_on": lambda c, v: setattr(c.flags, "cache_on", _bool(v)),
    "h_init": lambda c, v: setattr(c, "h_init", float(np.float32(v))),
    "h_inc": lambda c, v: setattr(c, "h_inc", float(np.float32(v))),
    "decay": lambda c, v: setattr(c, "decay", float(np.float32(v))),
    "warmup_traces": lambda c, v: setattr(c, "warmup_traces", int(v)),
    "validate_exactness": lambda c, v: setattr(c, "validate_exactness", _bool(v)),
    "seed": lambda c, v: setattr(c, "seed", _u64(v)),
    "time_scale": lambda c, v: setattr(c, "time_scale", float(v)),
}


def load_config(path) -> RunConfig:                                 # pipeline.cpp:170-212
    try:
        f = open(path)
    except OSError:
        raise RuntimeError(f"cannot open config: {path}") from None
    cfg = RunConfig()
    with f:
        for lineno, line in enumerate(f, 1):
            s = line.strip(" \t\r\n")
            if not s or s.startswith("#"):
                continue
            if "=" not in s:
                raise RuntimeError(f"{path}:{lineno}: expected key = value")
            key, value = (x.strip(" \t\r") for x in s.split("=", 1))
            if key not in _FIELDS:
                raise RuntimeError(f"{path}:{lineno}: unknown config key '{key}'")
            try:
                _FIELDS[key](cfg, value)
            except Exception as e:  # noqa: BLE001
                raise RuntimeError(f"{path}:{lineno}: {key}: {e}") from None
    for key, setter in _FIELDS.items():  # LAIV_<KEY> overrides
        env = os.environ.get("LAIV_" + key.upper())
        if env is not None:
            setter(cfg, env)
    return cfg


# ---------------------------------------------------------------------------
# records (pipeline.hpp:62-130)
# ---------------------------------------------------------------------------
@dataclass
class RetrievalRow:                                                 # pipeline.hpp:63-74
    round: int = 0
    t2: float = 0.0
    t_c: float = 0.0
    t_g: float = 0.0
    hit_rate: float = 0.0
    coverage: float = 0.0
    probed: int = 0
    fast: int = 0
    slow: int = 0
    result_ids: list[int] = field(default_factory=list)


@dataclass
class TransferRow:                                                  # pipeline.hpp:76-81
    round: int = 0
    bytes: int = 0
    t_p: float = 0.0
    clusters: int = 0


@dataclass
class TraceRow:                                                     # pipeline.hpp:85-99
    trace_id: int = 0
    pipeline: PipelineKind = PipelineKind.Custom
    worker: int = 0
    batch: int = 0
    total_s: float = 0.0
    gen_plain_s: float = 0.0
    overlap_s: float = 0.0
    retrieve_s: float = 0.0
    tail_s: float = 0.0
    transfer_s: float = 0.0
    transfer_bytes: int = 0
    retrievals: list[RetrievalRow] = field(default_factory=list)
    transfers: list[TransferRow] = field(default_factory=list)


@dataclass
class BatchDecision:                                                # pipeline.hpp:101-105
    batch: int = 0
    worker: int = 0
    overlap: int = 0


@dataclass
class RunRecord:                                                    # pipeline.hpp:113-121
    rows: list[TraceRow] = field(default_factory=list)
    decisions: list[BatchDecision] = field(default_factory=list)
    hotness: list[tuple[int, dict[int, float]]] = field(default_factory=list)
    makespan_s: float = 0.0
    workers: int = 1
    assertions_ok: bool = True
    assertion_failures: list[str] = field(default_factory=list)


@dataclass
class Aggregates:                                                   # pipeline.hpp:123-134
    traces: int = 0
    retrievals: int = 0
    mean_latency_s: float = 0.0
    mean_hit_rate: float = 0.0
    mean_coverage: float = 0.0
    mean_gen_s: float = 0.0
    mean_retrieve_s: float = 0.0
    mean_transfer_s: float = 0.0
    total_transfer_bytes: float = 0.0
    throughput_qps: float = 0.0


def aggregate(rows: list[TraceRow], makespan_s: float) -> Aggregates:  # pipeline.cpp:625-655
    a = Aggregates(traces=len(rows))
    if not rows:
        return a
    hit = cov = 0.0
    for r in rows:
        a.mean_latency_s += r.total_s
        a.mean_gen_s += r.gen_plain_s + r.overlap_s + r.tail_s
        a.mean_retrieve_s += r.retrieve_s
        a.mean_transfer_s += r.transfer_s
        a.total_transfer_bytes += float(r.transfer_bytes)
        for rr in r.retrievals:
            hit += rr.hit_rate
            cov += rr.coverage
            a.retrievals += 1
    n = float(len(rows))
    a.mean_latency_s /= n
    a.mean_gen_s /= n
    a.mean_retrieve_s /= n
    a.mean_transfer_s /= n
    if a.retrievals:
        a.mean_hit_rate = hit / a.retrievals
        a.mean_coverage = cov / a.retrievals
    if makespan_s > 0.0:
        a.throughput_qps = len(rows) / makespan_s
    return a


def save_records(path, rec: RunRecord) -> None:                     # pipeline.cpp:765-822
    with open(path, "w") as f:
        f.write(json.dumps({"type": "meta", "schema_version": 1, "makespan_s": rec.makespan_s,
                            "workers": rec.workers, "assertions_ok": rec.assertions_ok,
                            "assertion_failures": rec.assertion_failures}) + "\n")
        for r in rec.rows:
            f.write(json.dumps({
                "type": "trace", "trace_id": r.trace_id, "pipeline": pipeline_name(r.pipeline),
                "worker": r.worker, "batch": r.batch, "total_s": r.total_s,
                "gen_plain_s": r.gen_plain_s, "overlap_s": r.overlap_s,
                "retrieve_s": r.retrieve_s, "tail_s": r.tail_s, "transfer_s": r.transfer_s,
                "transfer_bytes": r.transfer_bytes,
                "retrievals": [rr.__dict__ for rr in r.retrievals],
                "transfers": [t.__dict__ for t in r.transfers]}) + "\n")
        for d in rec.decisions:
            f.write(json.dumps({"type": "decision", "batch": d.batch, "worker": d.worker,
                                "overlap": d.overlap}) + "\n")
        for w, h in rec.hotness:
            f.write(json.dumps({"type": "hotness", "worker": w,
                                "entries": [[c, v] for c, v in sorted(h.items())]}) + "\n")


# ---------------------------------------------------------------------------
# serving (pipeline.cpp:293-617)
# ---------------------------------------------------------------------------
class Worker:
    """One serving worker: a Device (its GPU cluster cache = the TieredStore)
    and its HotnessTable; `clock` is its busy time (pipeline.cpp:296-303)."""

    def __init__(self, ix: laiv.IvfIndex, cfg: RunConfig, device: int = 0):
        self.dev = laiv.Device(ix, cfg.capacity_bytes, device=device,
                               max_batch=max(32, cfg.micro_batch))
        self.dev.store.clear()
        self.hot = laiv.HotnessTable(cfg.cache_params())
        self.clock = 0.0

    def hotness_snapshot(self) -> dict[int, float]:
        return {c: self.hot.hotness(c) for c in range(self.dev.ix.nc) if self.hot.tracked(c)}


def _modeled_t2(slow: int, fast: int, cost: laiv.CostModel) -> float:  # tiered.cpp:186-195
    return max(math.ceil(slow / cost.parallel_slots) * cost.t_cc, fast * cost.t_gc)


def _device_retrievals(dev, walks, act, r, sidecar, cfg, rows, used, traces, failures) -> float:
    """Device mode: the round's retrievals of every active trace as batched
    hybrid searches (laivg_hybrid_search_batch: one coarse + one scan launch
    per max_batch queries, the misses list-major on the host or fetched
    through the HBM ring); results per query equal hybrid_search's. Returns
    the measured phase time."""
    refs = [(i, walks[i].phases[r].predictor_ref, ref)
            for i in act for ref in walks[i].phases[r].query_refs]
    if not refs:
        return 0.0
    Q = np.stack([sidecar[ref] for _, _, ref in refs])
    probes = laiv.coarse_probe(dev, Q, cfg.n_probe).reshape(len(refs), -1)
    probed = probes.shape[1]
    t2 = 0.0
    step = 256
    for q0 in range(0, len(refs), step):
        res, tm = laiv.hybrid_search_batch(dev, Q[q0:q0 + step], cfg.n_probe, cfg.top_k, cfg.cost)
        t2 += tm.t_2
        for j in range(res.counts.shape[0]):
            i, pred, ref = refs[q0 + j]
            rr = RetrievalRow(round=r, coverage=laiv.coverage(dev, sidecar[pred], Q[q0 + j],
                                                              cfg.n_probe))
            rr.t_c, rr.t_g = tm.t_c, tm.t_g  # the batch's phase times
            rr.fast = int(res.nfast[j])
            rr.probed = probed
            rr.slow = probed - rr.fast
            rr.hit_rate = rr.fast / probed if probed else 0.0
            top = res.topk(j)
            rr.result_ids = [e.id for e in top.entries]
            used.update(int(c) for c in probes[q0 + j])
            if cfg.validate_exactness and failures is not None:
                want = laiv.ivf_search(dev, Q[q0 + j], cfg.n_probe, cfg.top_k)
                if [(e.id, e.score) for e in want.entries] != \
                        [(e.id, e.score) for e in top.entries]:
                    failures.append(f"trace {traces[i].trace_id}: hybrid top-k differs "
                                    "from the monolithic search")
            rows[i].retrievals.append(rr)
    return t2


def serve_microbatch(traces: list[QueryTrace], budgets: list[int], sidecar: np.ndarray,
                     cfg: RunConfig, worker: Worker, failures: list[str] | None):
    """One micro-batch of traces on one worker, round by round: the rounds'
    prefetches share one window, the retrievals of a round run as one phase
    (pipeline.cpp:305-473). Returns (batch_time, rows)."""
    dev = worker.dev
    walks = [decompose_trace(t) for t in traces]
    rows = [TraceRow(trace_id=t.trace_id, pipeline=t.pipeline) for t in traces]
    measured = cfg.mode == laiv.ChannelMode.Device
    chan = laiv.TransferChannel(cfg.cost.bandwidth_bytes_per_s,
                                laiv.ChannelMode.Device if measured
                                else laiv.ChannelMode.SimulatedClock)
    used: set[int] = set()
    batch_time = 0.0
    # Device mode runs on one clock: every trace-second (plain generation,
    # windows, tail) is scaled by time_scale next to the measured copy and
    # retrieval times
    scale = cfg.time_scale if measured else 1.0
    for r in range(max((len(w.phases) for w in walks), default=0)):
        act = [i for i, w in enumerate(walks) if r < len(w.phases)]
        plain_r = max(walks[i].phases[r].plain_before_s for i in act) * scale
        window_r = max(walks[i].phases[r].window_s for i in act)
        t_p_total = 0.0
        if measured and cfg.flags.lookahead_on:
            # the round's prefetches as one batch: one coarse pass, the
            # sequential plans against the filling store, ONE generation
            # window for all their copies (laivg_prefetch_batch)
            q_in = np.stack([sidecar[walks[i].phases[r].predictor_ref] for i in act])
            bud = np.array([budgets[i] for i in act], np.uint64)
            rep, nplan = laiv.prefetch_batch(dev, q_in, bud, chan, window_r * scale)
            t_p_total = rep.t_p
            k0 = 0
            for j, i in enumerate(act):
                mine = rep.transferred[k0:k0 + int(nplan[j])]
                k0 += int(nplan[j])
                b = sum(dev.ix.cluster_bytes(c) for c in mine)
                tp = rep.t_p * b / rep.bytes if rep.bytes else 0.0
                if cfg.flags.cache_on:
                    for c in mine:
                        worker.hot.on_fetch(c)
                if b > 0 or mine:
                    rows[i].transfers.append(TransferRow(r, b, tp, len(mine)))
                rows[i].transfer_s += tp
                rows[i].transfer_bytes += b
        elif cfg.flags.lookahead_on:
            for i in act:
                ph = walks[i].phases[r]
                budget = min(budgets[i], dev.store.free_bytes())
                plan = laiv.plan_prefetch(dev, sidecar[ph.predictor_ref], budget)
                rep = laiv.execute_prefetch(dev, plan, chan,
                                            window_r * (cfg.time_scale if measured else 1.0))
                t_p_total += rep.t_p
                if cfg.flags.cache_on:
                    for c in rep.transferred:
                        worker.hot.on_fetch(c)
                if rep.bytes > 0 or rep.transferred:
                    rows[i].transfers.append(TransferRow(r, rep.bytes, rep.t_p,
                                                         len(rep.transferred)))
                rows[i].transfer_s += rep.t_p
                rows[i].transfer_bytes += rep.bytes
        t1_r = max(window_r * scale, t_p_total)
        tot_fast = tot_slow = tot_probed = 0
        t2_meas = 0.0
        if measured and cfg.flags.lookahead_on:
            t2_meas = _device_retrievals(dev, walks, act, r, sidecar, cfg, rows, used,
                                         traces, failures)
        for i in act if not (measured and cfg.flags.lookahead_on) else ():
            ph = walks[i].phases[r]
            pred = sidecar[ph.predictor_ref]
            for ref in ph.query_refs:
                q = sidecar[ref]
                rr = RetrievalRow(round=r, coverage=laiv.coverage(dev, pred, q, cfg.n_probe))
                if cfg.flags.lookahead_on:
                    res, tm = laiv.hybrid_search(dev, q, cfg.n_probe, cfg.top_k, cfg.cost)
                    rr.t_c, rr.t_g = (tm.t_c, tm.t_g) if measured else (tm.model_t_c,
                                                                         tm.model_t_g)
                    t2_meas += tm.t_2
                    rr.hit_rate = res.hit_rate
                    rr.fast, rr.slow = len(res.fast_clusters), len(res.slow_clusters)
                    rr.probed = rr.fast + rr.slow
                    rr.result_ids = [e.id for e in res.topk.entries]
                    used.update(res.fast_clusters)
                    used.update(res.slow_clusters)
                    if cfg.validate_exactness and failures is not None:
                        want = laiv.ivf_search(dev, q, cfg.n_probe, cfg.top_k)
                        if [(e.id, e.score) for e in want.entries] != \
                                [(e.id, e.score) for e in res.topk.entries]:
                            failures.append(f"trace {traces[i].trace_id}: hybrid top-k differs "
                                            "from the monolithic search")
                else:
                    probe = laiv.coarse_probe(dev, q, cfg.n_probe).reshape(-1)
                    tk = laiv.ivf_search(dev, q, cfg.n_probe, cfg.top_k)
                    rr.probed = rr.slow = len(probe)
                    rr.t_c = math.ceil(rr.slow / cfg.cost.parallel_slots) * cfg.cost.t_cc
                    rr.result_ids = [e.id for e in tk.entries]
                    used.update(int(c) for c in probe)
                tot_fast += rr.fast
                tot_slow += rr.slow
                tot_probed += rr.probed
                rows[i].retrievals.append(rr)
        if measured:
            t2_r = t2_meas
        elif cfg.flags.lookahead_on:
            t2_r = _modeled_t2(tot_slow, tot_fast, cfg.cost)
        else:
            t2_r = math.ceil(tot_probed / cfg.cost.parallel_slots) * cfg.cost.t_cc
        for i in act:
            rows[i].gen_plain_s += plain_r
            rows[i].overlap_s += t1_r
            rows[i].retrieve_s += t2_r
            for rr in rows[i].retrievals:
                if rr.round == r:
                    rr.t2 = t2_r
        batch_time += plain_r + t1_r + t2_r
    tail_r = 0.0
    for w, row in zip(walks, rows):
        row.tail_s = w.tail_s * scale
        row.total_s = row.gen_plain_s + row.overlap_s + row.retrieve_s + row.tail_s
        tail_r = max(tail_r, row.tail_s)
    batch_time += tail_r
    # cache maintenance between batches (pipeline.cpp:462-472)
    if cfg.flags.cache_on:
        worker.hot.end_of_round(used)
        worker.hot.evict_to_fraction(dev)
    else:
        dev.store.clear()
        worker.hot.clear()
    return batch_time, rows


def run_batch(traces: list[QueryTrace], sidecar, ix: laiv.IvfIndex, cfg: RunConfig,
              devices: list[int] | None = None) -> RunRecord:       # pipeline.cpp:498-617
    """Full replay: optional similarity grouping, optional cache-aware
    assignment, per-worker clocks, cache update and eviction after every
    micro-batch; warm-up traces first, excluded from the record. Worker w
    runs on GPU devices[w % len(devices)]."""
    if not traces:
        raise ValueError("run_batch needs at least one trace")
    import copy

    cfg = copy.deepcopy(cfg)
    cfg.validate_and_clamp()
    sidecar = np.ascontiguousarray(sidecar, np.float32)
    validate_traces(traces, sidecar.shape[0])
    devices = devices or [0]
    workers = [Worker(ix, cfg, devices[w % len(devices)]) for w in range(cfg.workers)]
    rec = RunRecord(workers=cfg.workers)
    warm = min(cfg.warmup_traces, len(traces) - 1) if cfg.flags.cache_on else 0

    def sched_ref(t: QueryTrace) -> int:
        for s in t.stages:
            if s.embedding_ref >= 0:
                return s.embedding_ref
        raise RuntimeError(f"trace {t.trace_id} carries no embedding")

    def serve_split(begin: int, end: int, measured: bool):
        n = end - begin
        if n == 0:
            return
        queries = np.stack([sidecar[sched_ref(traces[i])] for i in range(begin, end)])
        batches = (laiv.group_microbatches(queries, cfg.micro_batch) if cfg.flags.prefetch_sched_on
                   else laiv.chunk_microbatches(n, cfg.micro_batch))
        snaps = [laiv.WorkerState(w, set(wk.dev.store.resident().keys()), cfg.capacity_bytes)
                 for w, wk in enumerate(workers)]
        d0 = workers[0].dev
        assign = (laiv.assign_cache_aware(d0, batches, snaps, queries, cfg.n_probe)
                  if cfg.flags.cache_sched_on
                  else laiv.assign_round_robin(len(batches), len(workers)))
        if measured:
            for b, mb in enumerate(batches):
                rec.decisions.append(BatchDecision(b, assign[b], laiv.assignment_overlap(
                    d0, [mb], snaps, [assign[b]], queries, cfg.n_probe)))
        for w, wk in enumerate(workers):
            for b, mb in enumerate(batches):
                if assign[b] != w:
                    continue
                bt = [traces[begin + q] for q in mb.queries]
                budgets = laiv.split_budget(cfg.prefetch_budget_bytes, mb)
                t, rows = serve_microbatch(bt, budgets, sidecar, cfg, wk,
                                           rec.assertion_failures if measured else None)
                wk.clock += t
                if measured:
                    for row in rows:
                        row.worker, row.batch = w, b
                        rec.rows.append(row)

    if warm > 0:
        serve_split(0, warm, False)
        for wk in workers:
            wk.clock = 0.0
    serve_split(warm, len(traces), True)
    for w, wk in enumerate(workers):
        rec.makespan_s = max(rec.makespan_s, wk.clock)
        if wk.dev.store.recompute_used_bytes() != wk.dev.store.used_bytes():
            rec.assertion_failures.append("fast-tier byte accounting drifted from the resident set")
        if cfg.flags.cache_on:
            rec.hotness.append((w, wk.hotness_snapshot()))
    rec.assertions_ok = not rec.assertion_failures
    return rec


def aggregate_by_pipeline(rows: list[TraceRow]) -> dict[str, Aggregates]:  # pipeline.cpp:654-666
    grouped: dict[str, list[TraceRow]] = {}
    for r in rows:
        grouped.setdefault(pipeline_name(r.pipeline), []).append(r)
    return {k: aggregate(v, 0.0) for k, v in sorted(grouped.items())}


def _fmt_full(v: float) -> str:                                     # pipeline.cpp:29-33
    return "%.17g" % v


_GETTERS = {  # key -> value text (pipeline.cpp:57-127, same order as _FIELDS)
    "n_probe": lambda c: str(c.n_probe),
    "top_k": lambda c: str(c.top_k),
    "prefetch_budget_bytes": lambda c: str(c.prefetch_budget_bytes),
    "capacity_bytes": lambda c: str(c.capacity_bytes),
    "cache_fraction": lambda c: _fmt_full(c.cache_fraction),
    "bandwidth_bytes_per_s": lambda c: _fmt_full(c.cost.bandwidth_bytes_per_s),
    "t_cc": lambda c: _fmt_full(c.cost.t_cc),
    "t_gc": lambda c: _fmt_full(c.cost.t_gc),
    "parallel_slots": lambda c: str(c.cost.parallel_slots),
    "workers": lambda c: str(c.workers),
    "micro_batch": lambda c: str(c.micro_batch),
    "mode": lambda c: {laiv.ChannelMode.SimulatedClock: "simulated",
                       laiv.ChannelMode.Measured: "measured",
                       laiv.ChannelMode.Device: "device"}[laiv.ChannelMode(c.mode)],
    "lookahead_on": lambda c: "true" if c.flags.lookahead_on else "false",
    "prefetch_sched_on": lambda c: "true" if c.flags.prefetch_sched_on else "false",
    "cache_sched_on": lambda c: "true" if c.flags.cache_sched_on else "false",
    "cache_on": lambda c: "true" if c.flags.cache_on else "false",
    "h_init": lambda c: _fmt_full(c.h_init),
    "h_inc": lambda c: _fmt_full(c.h_inc),
    "decay": lambda c: _fmt_full(c.decay),
    "warmup_traces": lambda c: str(c.warmup_traces),
    "validate_exactness": lambda c: "true" if c.validate_exactness else "false",
    "seed": lambda c: str(c.seed),
    "time_scale": lambda c: _fmt_full(c.time_scale),
}


# keys only this port writes; each is written only when it differs from the
# reference's behaviour, so a config saved here for a reference-expressible
# run loads in the reference's load_config (which rejects unknown keys,
# pipeline.cpp:170-212)
_EXTENSION_KEYS = {"time_scale": lambda c: c.time_scale != 1.0}


def save_config(path, cfg: RunConfig) -> None:                     # pipeline.cpp:215-226
    try:
        f = open(path, "w")
    except OSError:
        raise RuntimeError(f"cannot open for writing: {path}") from None
    with f:
        for key, get in _GETTERS.items():
            if key in _EXTENSION_KEYS and not _EXTENSION_KEYS[key](cfg):
                continue
            f.write(f"{key} = {get(cfg)}\n")


def load_records(path) -> RunRecord:                                # pipeline.cpp:824-901
    try:
        f = open(path)
    except OSError:
        raise RuntimeError(f"cannot open: {path}") from None
    rec, have_meta = RunRecord(), False
    with f:
        for lineno, line in enumerate(f, 1):
            line = line.rstrip("\n")
            if not line:
                continue
            try:
                j = json.loads(line)
                t = j["type"]
                if t == "meta":
                    if int(j["schema_version"]) != 1:
                        raise ValueError(f"unsupported record schema version {j['schema_version']}")
                    rec.makespan_s = float(j["makespan_s"])
                    rec.workers = int(j["workers"])
                    rec.assertions_ok = bool(j["assertions_ok"])
                    rec.assertion_failures = list(j["assertion_failures"])
                    have_meta = True
                elif t == "trace":
                    row = TraceRow(int(j["trace_id"]), pipeline_from_name(j["pipeline"]),
                                   int(j["worker"]), int(j["batch"]), float(j["total_s"]),
                                   float(j["gen_plain_s"]), float(j["overlap_s"]),
                                   float(j["retrieve_s"]), float(j["tail_s"]),
                                   float(j["transfer_s"]), int(j["transfer_bytes"]))
                    row.retrievals = [RetrievalRow(**r) for r in j["retrievals"]]
                    row.transfers = [TransferRow(**x) for x in j["transfers"]]
                    rec.rows.append(row)
                elif t == "decision":
                    rec.decisions.append(BatchDecision(int(j["batch"]), int(j["worker"]),
                                                       int(j["overlap"])))
                elif t == "hotness":
                    rec.hotness.append((int(j["worker"]),
                                        {int(c): float(np.float32(v)) for c, v in j["entries"]}))
                else:
                    raise ValueError(f"unknown record type '{t}'")
            except Exception as e:  # noqa: BLE001 - the reference wraps every error
                raise RuntimeError(f"{path}:{lineno}: {e}") from None
    if not have_meta:
        raise RuntimeError(f"{path}: missing meta record")
    return rec


def run_single(trace: QueryTrace, sidecar, worker: Worker, cfg: RunConfig,
               failures: list[str] | None = None) -> TraceRow:      # pipeline.cpp:478-496
    """Replays one trace against a worker's cache (and hotness table) and
    advances them; run_batch with one worker and micro-batch 1."""
    import copy

    local = copy.deepcopy(cfg)
    local.capacity_bytes = worker.dev.store.capacity_bytes()
    local.validate_and_clamp()
    sidecar = np.ascontiguousarray(sidecar, np.float32)
    _, rows = serve_microbatch([trace], [local.prefetch_budget_bytes], sidecar, local, worker,
                               failures)
    return rows[0]


def calibrate_budget(traces: list[QueryTrace], pipeline: PipelineKind | None,
                     bandwidth_bytes_per_s: float) -> float:        # budget.cpp:159-182
    """Prefetch budget = mean duration of the stage right before each
    Retrieve x link bandwidth (the paper's B_link * t_LLM rule)."""
    if bandwidth_bytes_per_s <= 0.0:
        raise ValueError("bandwidth must be positive")
    total, count = 0.0, 0
    for t in traces:
        if pipeline is not None and t.pipeline != pipeline:
            continue
        for i in range(1, len(t.stages)):
            if t.stages[i].kind == StageKind.Retrieve and \
                    t.stages[i - 1].kind != StageKind.Retrieve:
                total += t.stages[i - 1].duration_s
                count += 1
    if count == 0:
        raise RuntimeError("no pre-retrieval stage found in the calibration traces")
    return (total / count) * bandwidth_bytes_per_s
