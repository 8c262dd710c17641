"""Pins the C restatement (oracle/oracle.c) to the reference's own outputs.

Golden fixtures come from the unmodified reference (tests/golden/make_golden.py);
every check here is bit-exact, as the reference's tests are (both sides run
fp64 CPU code with the same per-term arithmetic).
"""
import numpy as np
import pytest

from common import (IP, L2, accept1_case, expected_row, golden, hybrid_d8_case,
                    planted_data)


@pytest.mark.parametrize("name", ["l2", "ip"])
def test_hybrid_d8_ivf_search(orc, name):
    # test_tiered.cpp:206-236: hybrid == monolithic for 200 random residencies
    case, queries, g = hybrid_d8_case(orc, name)
    p = f"{name}_"
    for t in range(200):
        L, k = int(g[p + "L"][t]), int(g[p + "k"][t])
        ids, sc = orc.ivf_search(case.centroids, case.vecs, case.ids, case.list_off,
                                 case.metric, queries[t], L, k)
        want_ids, want_sc = expected_row(g, p, t)
        assert np.array_equal(ids, want_ids) and np.array_equal(sc, want_sc), t
        # the fast/slow split the reference reports
        probe = orc.coarse_probe(case.centroids, case.metric, queries[t], L)
        mask = g[p + "masks"][t]
        fast = [c for c in probe if mask[c]]
        slow = [c for c in probe if not mask[c]]
        ef, es = g[p + "exp_fast"][t], g[p + "exp_slow"][t]
        assert fast == [int(c) for c in ef[ef >= 0]]
        assert slow == [int(c) for c in es[es >= 0]]


@pytest.mark.parametrize("name", ["l2", "ip"])
def test_hybrid_d8_rank_clusters(orc, name):
    case, queries, g = hybrid_d8_case(orc, name)
    for t in range(50):
        order = orc.rank_clusters(case.centroids, case.metric, queries[t])
        assert np.array_equal(order, g[f"{name}_rank"][t])


def test_acceptance1_exactness(orc):
    # acceptance.cpp:61-98 criterion #1
    case, queries, masks, full_q, g = accept1_case(orc)
    for t in range(0, 1000, 3):
        ids, sc = orc.ivf_search(case.centroids, case.vecs, case.ids, case.list_off, L2,
                                 queries[t], int(g["L"][t]), int(g["k"][t]))
        want_ids, want_sc = expected_row(g, "", t)
        assert np.array_equal(ids, want_ids) and np.array_equal(sc, want_sc)
    for t in range(200):
        k = int(g["full_k"][t])
        ids, sc = orc.exact_search(case.vecs, case.ids, L2, full_q[t], k)
        assert np.array_equal(ids, g["full_ids"][t, :k]) and np.array_equal(sc, g["full_scores"][t, :k])


@pytest.mark.parametrize("name,metric", [("l2", L2), ("ip", IP)])
def test_planted_d768(orc, name, metric):
    cen, vecs, ids, off, qi, qo, g = planted_data()
    for t in range(0, 40, 4):
        got = orc.ivf_search(cen, vecs, ids, off, metric, qo[t], 8, 10)
        assert np.array_equal(got[0], g[f"{name}_ids"][t])
        assert np.array_equal(got[1], g[f"{name}_scores"][t])
        assert np.array_equal(orc.rank_clusters(cen, metric, qi[t]), g[f"{name}_rank"][t])
        assert orc.coverage(cen, metric, qi[t], qo[t], 8) == g[f"{name}_coverage"][t]
    cb = np.full(64, 300 * (4 * 768 + 8), np.uint64)
    nores = np.zeros(64, np.uint8)
    for t in range(0, 40, 5):
        order = orc.rank_clusters(cen, metric, qi[t])
        for b, bud in enumerate(g[f"{name}_budgets"]):
            plan, _, _ = orc.plan_prefetch(order, cb, nores, int(bud))
            want = g[f"{name}_plans"][t, b]
            assert list(plan) == [int(x) for x in want[want >= 0]]


def test_plan_prefetch_known_answers(orc):
    # test_tiered.cpp:21-79: 1-D clusters of 5, 3, 4 members at 0, 1, 2;
    # query -1 ranks them 0, 1, 2; one member costs 12 bytes.
    cen = np.array([[0.0], [1.0], [2.0]], np.float32)
    order = orc.rank_clusters(cen, L2, np.array([-1.0], np.float32))
    assert list(order) == [0, 1, 2]
    cb = np.array([60, 36, 48], np.uint64)
    none = np.zeros(3, np.uint8)
    assert [list(x) if not isinstance(x, int) else x
            for x in orc.plan_prefetch(order, cb, none, 8 * 12)] == [[0, 1], 96, [2]]
    assert [list(x) if not isinstance(x, int) else x
            for x in orc.plan_prefetch(order, cb, none, 7 * 12)] == [[0], 60, [1, 2]]
    assert [list(x) if not isinstance(x, int) else x
            for x in orc.plan_prefetch(order, cb, none, 4 * 12)] == [[1], 36, [0, 2]]
    assert [list(x) if not isinstance(x, int) else x
            for x in orc.plan_prefetch(order, cb, none, 0)] == [[], 0, [0, 1, 2]]
    res = np.array([1, 0, 0], np.uint8)
    assert list(orc.plan_prefetch(order, cb, res, 100 * 12)[0]) == [1, 2]


def test_sched_golden(orc):
    g = golden("sched.npz")
    from common import sha
    q = orc.random_matrix(256, 768, 717)
    assert sha(q) == str(g["group_sha"])
    batches = orc.group_microbatches(q, 4)
    assert len(batches) == 64
    order = [x for b in batches for x in b]
    assert order == [int(x) for x in g["group_order"]]
    for i in range(len(g["split_total"])):
        n = int(g["split_n"][i])
        got = orc.split_budget(int(g["split_total"][i]), g["split_batch"][i, :n])
        assert list(got) == [int(x) for x in g["split_out"][i, :n]]


def test_assign_cache_aware_golden(orc):
    case, _, _ = hybrid_d8_case(orc, "l2")
    g = golden("sched.npz")
    batches = [[0, 1], [2, 3], [4, 5], [6, 7], [8, 9], [10, 11]]
    for t in range(20):
        qs = orc.random_matrix(12, 8, 7000 + t)
        got = orc.assign_cache_aware(batches, g["assign_resident"][t], case.centroids, L2, qs, 4)
        assert list(got) == [int(x) for x in g["assign_out"][t]]


def test_hotness_law(orc):
    # acceptance.cpp:382-403: h' = h/d (+ inc) exactly in float32
    rng = np.random.default_rng(515)
    h = (rng.random(100000) * 32.0).astype(np.float32) + np.float32(1e-3)
    d = (1.0 + rng.random(100000) * 9.0).astype(np.float32)
    inc = (rng.random(100000) * 8.0).astype(np.float32) + np.float32(1e-3)
    used = (rng.random(100000) < 0.5).astype(np.uint8)
    want = h / d
    want = np.where(used == 1, want + inc, want).astype(np.float32)
    for i in range(0, 100000, 997):
        got = orc.hotness_end_of_round(h[i:i + 1], used[i:i + 1], float(d[i]), float(inc[i]))
        assert got[0] == want[i]


def hotness_replay(script, cb):
    """cache.cpp:27-66 restated in Python (small, pure loops)."""
    h_init, h_inc, decay, frac = script["params"]
    h_init, h_inc, decay = np.float32(h_init), np.float32(h_inc), np.float32(decay)
    cap = script["cap"]
    hot, resident = {}, {}
    out = []
    for ins, used in script["ops"]:
        for c in ins:
            resident[c] = int(cb[c])
            hot[c] = h_init
        for c in list(hot):
            v = np.float32(hot[c] / decay)
            if c in used:
                v = np.float32(v + h_inc)
            hot[c] = v
        budget = int(frac * float(cap))
        order = sorted(resident, key=lambda c: (hot.get(c, np.float32(0)), c))
        ev = []
        for c in order:
            if sum(resident.values()) <= budget:
                break
            del resident[c]
            hot.pop(c, None)
            ev.append(c)
        out.append(ev)
    return out, {c: float(hot[c]) for c in resident}


def test_hotness_scripts(orc):
    case, _, _ = hybrid_d8_case(orc, "l2")
    cb = case.cluster_bytes()
    for s in golden("hotness.json"):
        ev, final = hotness_replay(s, cb)
        assert ev == s["evicted"]
        assert final == {int(k): v for k, v in s["final"].items()}
