"""The host (slow) tier on the CPU (no GPU needed): laivg_slow_tier_scan is the
miss path of hybrid_search (tiered.cpp:169) — list-major, AVX2 / AVX-512 fp64
scoring — checked against the reference goldens (bit-exact at D = 8) and the
C oracle (§8c rule at D = 768), one query at a time and batched."""
import numpy as np
import pytest

from common import IP, L2, assert_topk_parity, expected_row, hybrid_d8_case, planted_data


@pytest.mark.parametrize("name", ["l2", "ip"])
def test_slow_tier_d8_golden(orc, laiv, name):
    case, queries, g = hybrid_d8_case(orc, name)
    ix = laiv.IvfIndex(case.centroids, case.vecs, case.ids, case.list_off,
                       laiv.Metric(case.metric))
    p = f"{name}_"
    sel = list(range(0, 200, 3))
    lists = [orc.coarse_probe(case.centroids, case.metric, queries[t], int(g[p + "L"][t]))
             for t in sel]
    # one batched call with per-query k would differ; group by k
    for k in sorted(set(int(g[p + "k"][t]) for t in sel)):
        ts = [t for t in sel if int(g[p + "k"][t]) == k]
        got = laiv.slow_tier_scan(ix, queries[ts], [lists[sel.index(t)] for t in ts], k,
                                  threads=4)
        for t, tk in zip(ts, got):
            want_ids, want_sc = expected_row(g, p, t)
            assert_topk_parity(case.metric, tk.ids, tk.scores, want_ids, want_sc, exact=True)


@pytest.mark.parametrize("metric", [IP, L2])
def test_slow_tier_d768_batched(orc, laiv, metric):
    cen, vecs, ids, off, qi, qo, g = planted_data()
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric(metric))
    rng = np.random.default_rng(metric)
    lists = []
    for t in range(12):
        ls = [int(c) for c in rng.choice(64, size=int(rng.integers(0, 9)), replace=False)]
        if t % 4 == 1 and ls:
            ls.append(ls[0])  # a cluster named twice counts twice (ivf.cpp:301-323)
        lists.append(ls)
    batched = laiv.slow_tier_scan(ix, qo[:12], lists, 10, threads=3)
    for t in range(12):
        single = laiv.slow_tier_scan(ix, qo[t:t + 1], [lists[t]], 10, threads=1)[0]
        assert np.array_equal(single.ids, batched[t].ids)
        assert np.array_equal(single.scores, batched[t].scores)
        want = orc.search_clusters(vecs, ids, off, metric, qo[t], lists[t], 10)
        assert_topk_parity(metric, batched[t].ids, batched[t].scores, *want)
    with pytest.raises(ValueError):
        laiv.slow_tier_scan(ix, qo[:1], [[64]], 5)
    with pytest.raises(ValueError):
        laiv.slow_tier_scan(ix, qo[:1], [[1]], 0)
