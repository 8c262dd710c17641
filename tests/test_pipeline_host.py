"""Host side of the pipeline caller (pipeline.py): trace / config / record
file formats and the trace decomposition, against the reference's files
(tests/golden/pipeline/) and the rules of trace.cpp / pipeline.cpp."""
import json
import os

import pytest

from paper_2502_20969_b200 import laiv
from paper_2502_20969_b200 import pipeline as P

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "pipeline")


@pytest.mark.parametrize("shape", ["HyDE", "SubQ", "Iter", "IRG", "FLARE", "SRAG"])
def test_trace_files_round_trip(tmp_path, shape):
    src = os.path.join(G, f"traces_{shape}.jsonl")
    traces = P.load_traces(src)
    assert len(traces) == 16
    out = tmp_path / "t.jsonl"
    P.save_traces(out, traces)
    a = [json.loads(x) for x in open(src)]
    b = [json.loads(x) for x in open(out)]
    assert a == b
    for t in traces:
        walk = P.decompose_trace(t)
        assert walk.phases, t
        for ph in walk.phases:
            assert ph.predictor_ref >= 0 and ph.query_refs


def test_decompose_rules():
    S, K = P.Stage, P.StageKind
    t = P.QueryTrace(1, P.PipelineKind.Custom, [
        S(K.Generate, 0, 0.0), S(K.Generate, 1, 0.4), S(K.Retrieve, 1, 0.0, 2),
        S(K.Generate, -1, 0.3), S(K.Judge, 5, 0.2), S(K.Retrieve, 6, 0.0), S(K.Generate, -1, 0.7)])
    w = P.decompose_trace(t)
    assert len(w.phases) == 2
    # phase 0: window = the Generate right before (0.4 s); predictor = the
    # latest ref BEFORE the window stage (a Generate's ref is its output)
    assert w.phases[0].window_s == 0.4 and w.phases[0].plain_before_s == 0.0
    assert w.phases[0].predictor_ref == 0 and w.phases[0].query_refs == [1, 2]
    # phase 1: a Judge window counts its own (input) ref
    assert w.phases[1].plain_before_s == 0.3 and w.phases[1].window_s == 0.2
    assert w.phases[1].predictor_ref == 5 and w.phases[1].query_refs == [6]
    assert w.tail_s == 0.7


def test_validate_traces_errors():
    S, K = P.Stage, P.StageKind
    with pytest.raises(RuntimeError, match="dangles past sidecar"):
        P.validate_traces([P.QueryTrace(3, stages=[S(K.Generate, 9, 0.0, 2)])], 10)
    with pytest.raises(RuntimeError, match="Retrieve stage has no query"):
        P.validate_traces([P.QueryTrace(3, stages=[S(K.Generate, 0), S(K.Retrieve, -1)])], 10)
    with pytest.raises(RuntimeError, match="no preceding stage"):
        P.validate_traces([P.QueryTrace(3, stages=[S(K.Retrieve, 0)])], 10)


def test_load_config_and_clamp(tmp_path, monkeypatch):
    c = P.load_config(os.path.join(G, "cfg_d.conf"))
    assert (c.n_probe, c.top_k, c.workers, c.micro_batch) == (16, 10, 3, 2)
    assert c.flags.cache_on and c.flags.prefetch_sched_on and not c.flags.cache_sched_on
    assert c.cost.parallel_slots == 4 and c.h_inc == 0.5 and c.decay == 3.0
    w = c.validate_and_clamp()
    assert "clamping" in w and c.prefetch_budget_bytes == 100000
    monkeypatch.setenv("LAIV_TOP_K", "7")
    assert P.load_config(os.path.join(G, "cfg_d.conf")).top_k == 7
    bad = tmp_path / "bad.conf"
    bad.write_text("n_probe = 4\nnope = 1\n")
    with pytest.raises(RuntimeError, match="bad.conf:2: unknown config key 'nope'"):
        P.load_config(bad)
    bad.write_text("cache_on = maybe\n")
    with pytest.raises(RuntimeError, match="expected a boolean"):
        P.load_config(bad)
    c = P.RunConfig(workers=0)
    with pytest.raises(ValueError):
        c.validate_and_clamp()


def test_load_traces_errors(tmp_path):
    p = tmp_path / "t.jsonl"
    p.write_text('{"schema_version": 2, "trace_id": 0, "pipeline": "HyDE", "stages": []}\n')
    with pytest.raises(RuntimeError, match="t.jsonl:1: schema_version 2 does not match"):
        P.load_traces(p)
    p.write_text('{"schema_version": 1, "trace_id": 0, "pipeline": "Nope", "stages": []}\n')
    with pytest.raises(RuntimeError, match="unknown pipeline: Nope"):
        P.load_traces(p)
    with pytest.raises(RuntimeError, match="cannot open"):
        P.load_traces(tmp_path / "missing.jsonl")


def test_aggregate():
    rows = [P.TraceRow(total_s=2.0, gen_plain_s=1.0, overlap_s=0.5, retrieve_s=0.5,
                       retrievals=[P.RetrievalRow(hit_rate=0.5, coverage=1.0)]),
            P.TraceRow(total_s=4.0, retrieve_s=1.0,
                       retrievals=[P.RetrievalRow(hit_rate=1.0, coverage=0.5)])]
    a = P.aggregate(rows, 2.0)
    assert a.mean_latency_s == 3.0 and a.mean_hit_rate == 0.75 and a.throughput_qps == 1.0
    assert laiv.ChannelMode.Device == 2


def test_records_and_config_round_trip(tmp_path):
    # load_records of the reference's own record files, save_records back:
    # the same JSON objects (pipeline.cpp:765-901)
    for name in ("rec_HyDE_b.jsonl", "rec_SubQ_d.jsonl"):
        src = os.path.join(G, name)
        rec = P.load_records(src)
        out = tmp_path / name
        P.save_records(out, rec)
        assert [json.loads(x) for x in open(src)] == [json.loads(x) for x in open(out)]
    c = P.load_config(os.path.join(G, "cfg_b.conf"))
    P.save_config(tmp_path / "c.conf", c)
    c2 = P.load_config(tmp_path / "c.conf")
    assert c2 == c
    # exactly the reference's keys, in its order (pipeline.cpp:57-127), when
    # no extension is in use: the file loads in the reference's load_config
    keys = [ln.split(" = ")[0] for ln in open(tmp_path / "c.conf")]
    assert keys == ["n_probe", "top_k", "prefetch_budget_bytes", "capacity_bytes",
                    "cache_fraction", "bandwidth_bytes_per_s", "t_cc", "t_gc", "parallel_slots",
                    "workers", "micro_batch", "mode", "lookahead_on", "prefetch_sched_on",
                    "cache_sched_on", "cache_on", "h_init", "h_inc", "decay", "warmup_traces",
                    "validate_exactness", "seed"]
    c.time_scale = 0.5
    P.save_config(tmp_path / "c2.conf", c)
    assert P.load_config(tmp_path / "c2.conf").time_scale == 0.5
    bad = tmp_path / "r.jsonl"
    bad.write_text('{"type": "trace"}\n')
    with pytest.raises(RuntimeError, match="r.jsonl:1"):
        P.load_records(bad)
    bad.write_text("")
    with pytest.raises(RuntimeError, match="missing meta record"):
        P.load_records(bad)


def test_calibrate_budget():
    # budget.cpp:159-182: mean duration of the stage before each Retrieve x B
    traces = P.load_traces(os.path.join(G, "traces_Iter.jsonl"))
    durs = [t.stages[i - 1].duration_s for t in traces for i in range(1, len(t.stages))
            if t.stages[i].kind == P.StageKind.Retrieve
            and t.stages[i - 1].kind != P.StageKind.Retrieve]
    acc = 0.0
    for x in durs:  # sequential, as the reference adds (Python's sum() compensates)
        acc += x
    want = (acc / len(durs)) * 64e9
    assert P.calibrate_budget(traces, None, 64e9) == want
    assert P.calibrate_budget(traces, P.PipelineKind.Iter, 64e9) == want
    with pytest.raises(RuntimeError, match="no pre-retrieval stage"):
        P.calibrate_budget(traces, P.PipelineKind.HyDE, 64e9)
    with pytest.raises(ValueError):
        P.calibrate_budget(traces, None, 0.0)
