"""Shared test helpers: golden fixtures, regenerated inputs, the parity rule."""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

IP, L2 = 0, 1
U64MAX = np.iinfo(np.uint64).max


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def golden(name: str):
    path = os.path.join(GOLDEN, name)
    if name.endswith(".json"):
        with open(path) as f:
            return json.load(f)
    return np.load(path)


def list_major(db, members):
    rows = np.asarray(members).astype(np.int64)
    return np.ascontiguousarray(db[rows]), np.asarray(members).astype(np.uint64)


class Case:
    """One golden index: centroids + list-major store + metric."""

    def __init__(self, centroids, list_off, members, db, metric):
        self.centroids = np.ascontiguousarray(centroids, np.float32)
        self.list_off = np.asarray(list_off, np.uint64)
        self.vecs, self.ids = list_major(db, members)
        self.metric = metric
        self.nc, self.d = self.centroids.shape

    def cluster_bytes(self):
        return np.diff(self.list_off).astype(np.uint64) * np.uint64(4 * self.d + 8)


def hybrid_d8_case(orc, name: str):
    g = golden("hybrid_d8.npz")
    db = orc.random_matrix(2048, 8, 101)
    assert sha(db) == str(g["db_sha"])
    metric = L2 if name == "l2" else IP
    case = Case(g[f"{name}_centroids"], g[f"{name}_list_off"], g[f"{name}_members"], db, metric)
    queries = np.array([orc.random_matrix(1, 8, 9000 + t)[0] for t in range(200)])
    assert sha(queries) == str(g[f"{name}_queries_sha"])
    return case, queries, g


def accept1_case(orc):
    g = golden("accept1_d16.npz")
    db = orc.random_matrix(4096, 16, 2026)
    assert sha(db) == str(g["db_sha"])
    case = Case(g["centroids"], g["list_off"], g["members"], db, L2)
    queries = np.array([orc.random_matrix(1, 16, 50000 + t)[0] for t in range(1000)])
    assert sha(queries) == str(g["queries_sha"])
    masks = np.unpackbits(g["masks"], axis=1)[:, :64]
    full_q = np.array([orc.random_matrix(1, 16, 90000 + t)[0] for t in range(200)])
    return case, queries, masks, full_q, g


PLANTED = dict(seed=7, nc=64, per_list=300, d=768, spread=0.05, nq=40, sigma=0.015, qseed=11)


def planted_data():
    """The planted D=768 datastore of planted_d768.npz (product generator)."""
    from paper_2502_20969_b200 import laiv

    p = PLANTED
    cen = laiv.synth_centroids(p["seed"], p["nc"], p["d"])
    vecs, ids = laiv.synth_lists(p["seed"], cen, p["per_list"], p["spread"])
    off = np.arange(0, p["nc"] * p["per_list"] + 1, p["per_list"], dtype=np.uint64)
    qi, qo, _ = laiv.synth_queries(p["qseed"], vecs, p["nq"], p["sigma"])
    g = golden("planted_d768.npz")
    assert sha(vecs) == str(g["sha_vecs"]) and sha(cen) == str(g["sha_cen"])
    assert sha(qi) == str(g["sha_qin"]) and sha(qo) == str(g["sha_qout"])
    return cen, vecs, ids, off, qi, qo, g


def expected_row(g, prefix, t):
    n = int(g[f"{prefix}exp_count"][t])
    return g[f"{prefix}exp_ids"][t, :n], g[f"{prefix}exp_scores"][t, :n]


def assert_topk_parity(metric, got_ids, got_sc, ref_ids, ref_sc, rel=1e-5, exact=False):
    """The north-star parity rule.

    Top-k ids equal except across adjacent entries whose reference scores are
    within `rel` relative of each other (near-ties may swap); ids absent from
    one side must sit within `rel` of the k-th (boundary) score; scores of
    matched ids within `rel` relative. `exact=True` demands bit equality.
    """
    got_ids, ref_ids = np.asarray(got_ids, np.uint64), np.asarray(ref_ids, np.uint64)
    got_sc, ref_sc = np.asarray(got_sc, np.float32), np.asarray(ref_sc, np.float32)
    assert got_ids.size == ref_ids.size, (got_ids, ref_ids)
    if exact:
        assert np.array_equal(got_ids, ref_ids), (got_ids, ref_ids)
        assert np.array_equal(got_sc, ref_sc), (got_sc, ref_sc)
        return
    if got_ids.size == 0:
        return

    def close(a, b):
        return abs(float(a) - float(b)) <= rel * max(abs(float(b)), 1e-30)

    ref_map = {int(i): float(s) for i, s in zip(ref_ids, ref_sc)}
    for i, s in zip(got_ids, got_sc):
        if int(i) in ref_map:
            assert close(s, ref_map[int(i)]), (int(i), s, ref_map[int(i)])
    boundary = float(ref_sc[-1])
    for i in set(map(int, got_ids)) ^ set(map(int, ref_ids)):
        s = ref_map.get(i)
        if s is None:
            s = float(got_sc[list(map(int, got_ids)).index(i)])
        assert close(s, boundary), ("id outside the near-tie band", i, s, boundary)
    for p in range(got_ids.size):
        if got_ids[p] != ref_ids[p]:
            assert close(got_sc[p], ref_sc[p]), ("swap across a real gap", p)


def probe_parity(got, ref_order, ref_scores, L, rel=1e-5):
    """Cluster selection equal except for boundary near-ties."""
    got = list(map(int, got))
    want = list(map(int, ref_order[:L]))
    if got == want:
        return True
    if set(got) != set(want):
        sL = ref_scores[ref_order[L - 1]]
        for c in set(got) ^ set(want):
            assert abs(ref_scores[c] - sL) <= rel * max(abs(sL), 1e-30), (c, ref_scores[c], sL)
    return False
