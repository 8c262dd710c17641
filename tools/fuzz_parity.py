#!/usr/bin/env python
"""Randomised parity sweep of the GPU path against the C oracle (test
infrastructure: the oracle is the checker). Each trial draws an index shape
(lists of ragged sizes incl. empty ones, odd dimensions, duplicated rows for
exact ties), a metric, a residency, a miss mode, nprobe and k (incl. k above
the candidate count), and checks single-query hybrid_search, the batch path
and the scan-only search_clusters against the oracle with the §8c rule,
batch == single == staged single bit for bit, and the prefetch planner and
coverage exactly.

    python tools/fuzz_parity.py --trials 200 --seed 1
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=100)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    from common import assert_topk_parity
    from oracle.oracle import Oracle
    from paper_2502_20969_b200 import laiv

    orc = Oracle()
    rng = np.random.default_rng(a.seed)
    fails = []
    for t in range(a.trials):
        nc = int(rng.choice([1, 2, 3, 7, 33, 64, 300]))
        d = int(rng.choice([1, 3, 4, 8, 17, 64, 128, 256, 768]))
        metric = int(rng.integers(0, 2))
        sizes = rng.integers(0, 60, nc)
        sizes[rng.random(nc) < 0.2] = 0
        n = int(sizes.sum())
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint64)
        vecs = rng.standard_normal((n, d)).astype(np.float32)
        if n > 4:  # exact duplicates -> score ties broken by id
            dup = rng.integers(0, n, max(1, n // 10))
            vecs[dup] = vecs[rng.integers(0, n)]
        ids = rng.choice(np.arange(1, 10 * n + 2, dtype=np.uint64), n, replace=False) \
            if n else np.zeros(0, np.uint64)
        cen = rng.standard_normal((nc, d)).astype(np.float32)
        L = int(rng.integers(0, nc + 3))
        k = int(rng.choice([1, 2, 5, 10, 33, 100]))
        nq = int(rng.integers(1, 20))
        Q = rng.standard_normal((nq, d)).astype(np.float32)
        fetch = str(rng.choice(["off", "auto", "all"]))
        frac = float(rng.choice([0.0, 0.3, 1.0]))
        cfg = dict(trial=t, nc=nc, d=d, metric=metric, n=n, L=L, k=k, nq=nq, fetch=fetch,
                   frac=frac)
        try:
            ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
            dev = laiv.Device(ix, 1 << 26, max_batch=32, miss_fetch=fetch, fetch_chunk_mb=1)
            dev.store.clear()
            for c in range(nc):
                if rng.random() < frac and sizes[c] > 0:
                    dev.store.insert(c)
            os.environ["LAIVG_LIST_SCAN"] = "1"  # list-major tensor-core scan
            res_ls, _ = laiv.hybrid_search_batch(dev, Q, L, k)
            os.environ["LAIVG_LIST_SCAN"] = "0"  # per-query scan
            res, _ = laiv.hybrid_search_batch(dev, Q, L, k)
            os.environ.pop("LAIVG_LIST_SCAN", None)
            for q in range(nq):
                assert np.array_equal(res_ls.topk(q).ids, res.topk(q).ids), "list != query ids"
                assert np.array_equal(res_ls.topk(q).scores, res.topk(q).scores), \
                    "list != query scores"
            dev.stage_queries(Q)
            for q in range(nq):
                single, _ = laiv.hybrid_search(dev, Q[q], L, k)
                got = res.topk(q)
                assert np.array_equal(got.ids, single.topk.ids), "batch != single ids"
                assert np.array_equal(got.scores, single.topk.scores), "batch != single scores"
                # the staged-row entry (single-query kernel reading HBM rows)
                si, ss, _, _ = dev.hybrid_search_staged(q, L, k)
                assert np.array_equal(si, single.topk.ids), "staged != host ids"
                assert np.array_equal(ss, single.topk.scores), "staged != host scores"
                want = orc.ivf_search(cen, vecs, ids, off, metric, Q[q], L, k)
                assert_topk_parity(metric, got.ids, got.scores, *want)
                probe = laiv.coarse_probe(dev, Q[q], L).reshape(-1)
                sc = laiv.search_clusters(dev, Q[q], probe, k)
                want2 = orc.search_clusters(vecs, ids, off, metric, Q[q], probe, k)
                assert_topk_parity(metric, sc.ids, sc.scores, *want2)
            # planner + coverage (tiered.cpp:67-84, 200-211), exact
            member = 4 * d + 8
            cb = sizes.astype(np.uint64) * np.uint64(member)
            resident = dev.store.resident_mask(nc).astype(np.uint8)
            budget = int(rng.integers(0, int(cb.sum()) + 2))
            plan = laiv.plan_prefetch(dev, Q[0], budget)
            order = orc.rank_clusters(cen, metric, Q[0])
            wp, wpb, wsk = orc.plan_prefetch(order, cb, resident, budget)
            assert list(plan.clusters) == list(wp) and plan.planned_bytes == wpb, "plan"
            assert list(plan.skipped) == list(wsk), "plan skipped"
            if L > 0 and nq > 1:
                assert laiv.coverage(dev, Q[0], Q[1], L) == \
                    orc.coverage(cen, metric, Q[0], Q[1], L), "coverage"
            del dev, ix
        except Exception as e:  # noqa: BLE001 - report and continue
            fails.append(dict(cfg, error=repr(e)[:300]))
    print(json.dumps({"trials": a.trials, "seed": a.seed, "failures": len(fails),
                      "first": fails[:5]}), flush=True)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
