"""ctypes bindings for the test-only checkers.

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` leg import this module. The product package
(paper_2502_20969_b200) never does.

* ``Oracle``  — the C restatement in oracle.c (liboracle.so), each function
  citing the reference file:line it restates.
* ``RefLib``  — the unmodified reference core (oracle/_ref/libref.so) built
  from /root/reference sources by oracle/Makefile; ``None`` when not built.

Store layout everywhere: list-major ``vecs[N, D] f32``, ``ids[N] u64``,
``list_off[nc + 1] u64`` (the LAIX order, ivf.cpp:373-388).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
IP, L2 = 0, 1

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _build_if_missing(path: str) -> None:
    if not os.path.exists(path):
        import subprocess

        subprocess.check_call(["make", "-s", "-C", HERE])


class Oracle:
    """C restatement of the reference hot path (oracle.c)."""

    def __init__(self) -> None:
        path = os.path.join(HERE, "liboracle.so")
        _build_if_missing(path)
        L = C.CDLL(path)
        self.L = L
        u32, u64, i32, f32 = C.c_uint32, C.c_uint64, C.c_int, C.c_float
        L.orc_derive_seed.restype = u64
        L.orc_derive_seed.argtypes = [u64, C.c_char_p]
        L.orc_random_matrix.argtypes = [u64, u32, u64, C.c_double, _f32p]
        L.orc_score_rounded.restype = f32
        L.orc_score_rounded.argtypes = [i32, _f32p, _f32p, u32]
        L.orc_rank_clusters.argtypes = [_f32p, u32, u32, i32, _f32p, _u32p, C.c_void_p]
        L.orc_coarse_probe.restype = u32
        L.orc_coarse_probe.argtypes = [_f32p, u32, u32, i32, _f32p, i32, _u32p]
        L.orc_search_clusters.restype = i32
        L.orc_search_clusters.argtypes = [_f32p, _u64p, _u64p, u32, u32, i32, _f32p,
                                          _u32p, u32, i32, _u64p, _f32p]
        L.orc_ivf_search.restype = i32
        L.orc_ivf_search.argtypes = [_f32p, _f32p, _u64p, _u64p, u32, u32, i32, _f32p,
                                     i32, i32, _u64p, _f32p]
        L.orc_exact_search.restype = i32
        L.orc_exact_search.argtypes = [_f32p, _u64p, u64, u32, i32, _f32p, i32, _u64p, _f32p]
        L.orc_plan_prefetch.restype = u32
        L.orc_plan_prefetch.argtypes = [_u32p, u32, _u64p, _u8p, u64, _u32p,
                                        C.POINTER(u64), _u32p, C.POINTER(u32)]
        L.orc_coverage.restype = C.c_double
        L.orc_coverage.argtypes = [_f32p, u32, u32, i32, _f32p, _f32p, i32]
        L.orc_group_microbatches.restype = u32
        L.orc_group_microbatches.argtypes = [_f32p, u64, u32, u64, _u64p, _u64p]
        L.orc_assign_cache_aware.restype = i32
        L.orc_assign_cache_aware.argtypes = [_u64p, _u64p, u32, _u8p, u32, _f32p, u32,
                                             u32, i32, _f32p, i32, _u32p]
        L.orc_assignment_overlap.restype = u64
        L.orc_assignment_overlap.argtypes = [_u64p, _u64p, u32, _u8p, u32, _u32p, _f32p,
                                             u32, u32, i32, _f32p, i32]
        L.orc_split_budget.restype = i32
        L.orc_split_budget.argtypes = [u64, _u64p, u64, _u64p]
        L.orc_hotness_end_of_round.argtypes = [_f32p, _u8p, u32, f32, f32]

    # rng.hpp / test_util.hpp
    def derive_seed(self, seed: int, label: str) -> int:
        return int(self.L.orc_derive_seed(seed, label.encode()))

    def random_matrix(self, n: int, dim: int, seed: int, scale: float = 1.0) -> np.ndarray:
        out = np.empty((n, dim), np.float32)
        self.L.orc_random_matrix(n, dim, seed, scale, out.reshape(-1))
        return out

    def score_rounded(self, metric, q, row) -> float:
        q, row = _c(q, np.float32), _c(row, np.float32)
        return float(self.L.orc_score_rounded(metric, q, row, q.size))

    # ivf.cpp:269-299
    def rank_clusters(self, centroids, metric, q, with_scores=False):
        centroids = _c(centroids, np.float32)
        nc, d = centroids.shape
        order = np.empty(nc, np.uint32)
        scores = np.empty(nc, np.float64)
        self.L.orc_rank_clusters(centroids.reshape(-1), nc, d, metric, _c(q, np.float32),
                                 order, scores.ctypes.data)
        return (order, scores) if with_scores else order

    def coarse_probe(self, centroids, metric, q, L):
        centroids = _c(centroids, np.float32)
        nc, d = centroids.shape
        out = np.empty(max(nc, 1), np.uint32)
        n = self.L.orc_coarse_probe(centroids.reshape(-1), nc, d, metric,
                                    _c(q, np.float32), int(L), out)
        return out[:n].copy()

    # ivf.cpp:301-349
    def search_clusters(self, vecs, ids, list_off, metric, q, clusters, k):
        vecs = _c(vecs, np.float32)
        d = vecs.shape[1]
        nc = len(list_off) - 1
        cl = _c(clusters, np.uint32)
        oid = np.empty(max(k, 1), np.uint64)
        osc = np.empty(max(k, 1), np.float32)
        n = self.L.orc_search_clusters(vecs.reshape(-1), _c(ids, np.uint64),
                                       _c(list_off, np.uint64), nc, d, metric,
                                       _c(q, np.float32), cl, cl.size, int(k), oid, osc)
        if n == -1:
            raise ValueError("k must be >= 1")
        if n == -2:
            raise ValueError("unknown cluster id")
        return oid[:n].copy(), osc[:n].copy()

    def ivf_search(self, centroids, vecs, ids, list_off, metric, q, L, k):
        centroids = _c(centroids, np.float32)
        vecs = _c(vecs, np.float32)
        nc, d = centroids.shape
        oid = np.empty(max(k, 1), np.uint64)
        osc = np.empty(max(k, 1), np.float32)
        n = self.L.orc_ivf_search(centroids.reshape(-1), vecs.reshape(-1),
                                  _c(ids, np.uint64), _c(list_off, np.uint64), nc, d,
                                  metric, _c(q, np.float32), int(L), int(k), oid, osc)
        if n < 0:
            raise ValueError("k must be >= 1")
        return oid[:n].copy(), osc[:n].copy()

    def exact_search(self, db, ids, metric, q, k):
        db = _c(db, np.float32)
        n, d = db.shape
        oid = np.empty(max(k, 1), np.uint64)
        osc = np.empty(max(k, 1), np.float32)
        got = self.L.orc_exact_search(db.reshape(-1), _c(ids, np.uint64), n, d, metric,
                                      _c(q, np.float32), int(k), oid, osc)
        if got < 0:
            raise ValueError("k must be >= 1")
        return oid[:got].copy(), osc[:got].copy()

    # tiered.cpp:67-84
    def plan_prefetch(self, order, cluster_bytes, resident, budget):
        order = _c(order, np.uint32)
        nc = order.size
        plan = np.empty(max(nc, 1), np.uint32)
        skipped = np.empty(max(nc, 1), np.uint32)
        pb = C.c_uint64(0)
        ns = C.c_uint32(0)
        n = self.L.orc_plan_prefetch(order, nc, _c(cluster_bytes, np.uint64),
                                     _c(resident, np.uint8), int(budget), plan,
                                     C.byref(pb), skipped, C.byref(ns))
        return plan[:n].copy(), int(pb.value), skipped[: ns.value].copy()

    def coverage(self, centroids, metric, q_in, q_out, L):
        centroids = _c(centroids, np.float32)
        nc, d = centroids.shape
        return float(self.L.orc_coverage(centroids.reshape(-1), nc, d, metric,
                                          _c(q_in, np.float32), _c(q_out, np.float32),
                                          int(L)))

    # sched.cpp
    def group_microbatches(self, queries, m):
        queries = _c(queries, np.float32)
        n, d = queries.shape
        order = np.empty(max(n, 1), np.uint64)
        off = np.empty(n + 1, np.uint64)
        nb = self.L.orc_group_microbatches(queries.reshape(-1), n, d, int(m), order, off)
        return [order[off[b]:off[b + 1]].tolist() for b in range(nb)]

    @staticmethod
    def _csr(batches):
        off = np.zeros(len(batches) + 1, np.uint64)
        for i, b in enumerate(batches):
            off[i + 1] = off[i] + len(b)
        mem = np.array([x for b in batches for x in b] or [0], np.uint64)
        return off, mem

    def assign_cache_aware(self, batches, resident, centroids, metric, queries, L):
        off, mem = self._csr(batches)
        resident = _c(resident, np.uint8)
        nw, nc = resident.shape
        centroids = _c(centroids, np.float32)
        out = np.empty(max(len(batches), 1), np.uint32)
        rc = self.L.orc_assign_cache_aware(off, mem, len(batches), resident.reshape(-1), nw,
                                           centroids.reshape(-1), nc, centroids.shape[1],
                                           metric, _c(queries, np.float32).reshape(-1),
                                           int(L), out)
        if rc < 0:
            raise ValueError("need at least one worker")
        return out[: len(batches)].copy()

    def assignment_overlap(self, batches, resident, assignment, centroids, metric, queries, L):
        off, mem = self._csr(batches)
        resident = _c(resident, np.uint8)
        nw, nc = resident.shape
        centroids = _c(centroids, np.float32)
        return int(self.L.orc_assignment_overlap(
            off, mem, len(batches), resident.reshape(-1), nw, _c(assignment, np.uint32),
            centroids.reshape(-1), nc, centroids.shape[1], metric,
            _c(queries, np.float32).reshape(-1), int(L)))

    def split_budget(self, total, batch):
        b = _c(batch, np.uint64)
        out = np.empty(max(b.size, 1), np.uint64)
        if self.L.orc_split_budget(int(total), b, b.size, out) < 0:
            raise ValueError("cannot split a budget over an empty batch")
        return out[: b.size].copy()

    def hotness_end_of_round(self, h, used, decay, h_inc):
        h = _c(h, np.float32).copy()
        self.L.orc_hotness_end_of_round(h, _c(used, np.uint8), h.size, decay, h_inc)
        return h


class RefLib:
    """The unmodified reference core (oracle/_ref/libref.so)."""

    def __init__(self, path: str | None = None) -> None:
        path = path or os.path.join(HERE, "_ref", "libref.so")
        L = C.CDLL(path)
        self.L = L
        u32, u64, i32, f32, vp = C.c_uint32, C.c_uint64, C.c_int, C.c_float, C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_gaussians.argtypes = [u64, u64, _f64p]
        L.ref_derive_seed.restype = u64
        L.ref_derive_seed.argtypes = [u64, C.c_char_p]
        L.ref_index_create.restype = vp
        L.ref_index_create.argtypes = [_f32p, u32, u32, i32, C.c_void_p, C.c_void_p, _u64p]
        L.ref_index_destroy.argtypes = [vp]
        L.ref_cluster_bytes.restype = u64
        L.ref_cluster_bytes.argtypes = [vp, u32]
        L.ref_rank_clusters.argtypes = [vp, _f32p, _u32p]
        L.ref_coarse_probe.argtypes = [vp, _f32p, i32, _u32p]
        L.ref_search_clusters.argtypes = [vp, _f32p, _u32p, u32, i32, _u64p, _f32p]
        L.ref_ivf_search.argtypes = [vp, _f32p, i32, i32, _u64p, _f32p]
        L.ref_exact_search.argtypes = [vp, _f32p, i32, _u64p, _f32p]
        L.ref_score_clusters.restype = C.c_int64
        L.ref_score_clusters.argtypes = [vp, _f32p, _u32p, u32, u64, _u64p, _f32p]
        L.ref_pairwise_l2.argtypes = [_f32p, u64, _f32p, u64, u32, _f32p]
        L.ref_hybrid_search.argtypes = [vp, _u8p, _f32p, i32, i32, _u64p, _f32p, _u32p,
                                        C.POINTER(u32), _u32p, C.POINTER(u32),
                                        C.POINTER(C.c_double)]
        L.ref_plan_prefetch.argtypes = [vp, _f32p, u64, _u8p, _u32p, C.POINTER(u32),
                                        C.POINTER(u64), _u32p, C.POINTER(u32)]
        L.ref_coverage.restype = C.c_double
        L.ref_coverage.argtypes = [vp, _f32p, _f32p, i32]
        L.ref_build_index.argtypes = [_f32p, u64, u32, u32, u64, i32, i32, i32, _f32p,
                                      _u64p, _u64p]
        L.ref_group_microbatches.argtypes = [_f32p, u64, u32, u64, _u64p, _u64p]
        L.ref_assign_cache_aware.argtypes = [vp, _u64p, _u64p, u32, _u8p, u32, _f32p, u64,
                                             i32, _u32p]
        L.ref_assignment_overlap.restype = C.c_int64
        L.ref_assignment_overlap.argtypes = [vp, _u64p, _u64p, u32, _u8p, u32, _u32p, _f32p,
                                             u64, i32]
        L.ref_split_budget.argtypes = [u64, _u64p, u64, _u64p]
        L.ref_cache_create.restype = vp
        L.ref_cache_create.argtypes = [u64, f32, f32, f32, C.c_double]
        L.ref_cache_destroy.argtypes = [vp]
        L.ref_cache_insert.argtypes = [vp, u32, u64, i32]
        L.ref_cache_on_fetch.argtypes = [vp, u32]
        L.ref_cache_end_of_round.argtypes = [vp, _u32p, u32]
        L.ref_cache_evict_to_fraction.argtypes = [vp, _u32p]
        L.ref_cache_hotness.restype = f32
        L.ref_cache_hotness.argtypes = [vp, u32]
        L.ref_cache_used.restype = u64
        L.ref_cache_used.argtypes = [vp]
        L.ref_cache_contains.argtypes = [vp, u32]
        L.ref_save_index.argtypes = [vp, C.c_char_p]
        L.ref_load_index.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.ref_index_lists.argtypes = [vp, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_search_many.argtypes = [vp, i32, C.c_void_p, u64, i32, i32, i32, _u64p, _f32p,
                                      C.c_void_p]

    @staticmethod
    def available(path: str | None = None) -> bool:
        return os.path.exists(path or os.path.join(HERE, "_ref", "libref.so"))

    def err(self) -> str:
        return self.L.ref_last_error().decode()

    def check(self, rc):
        if rc < 0:
            raise RuntimeError(self.err())
        return rc

    def pairwise_l2(self, a, b):
        A, B = _c(a, np.float32), _c(b, np.float32)
        out = np.empty(A.shape[0] * B.shape[0], np.float32)
        self.check(self.L.ref_pairwise_l2(A.reshape(-1), A.shape[0], B.reshape(-1), B.shape[0],
                                          A.shape[1], out))
        return out

    def rng_gaussians(self, seed, n):
        out = np.empty(n, np.float64)
        self.L.ref_rng_gaussians(seed, n, out)
        return out

    def build_index(self, db, nc, seed=0, max_iters=25, spherical=False, metric=L2):
        db = _c(db, np.float32)
        n, d = db.shape
        cen = np.empty((nc, d), np.float32)
        off = np.empty(nc + 1, np.uint64)
        mem = np.empty(n, np.uint64)
        self.check(self.L.ref_build_index(db.reshape(-1), n, d, nc, seed, max_iters,
                                          int(spherical), metric, cen.reshape(-1), off, mem))
        return cen, off, mem

    def index(self, centroids, vecs, ids, list_off, metric):
        return RefIndex(self, centroids, vecs, ids, list_off, metric)

    def group_microbatches(self, queries, m):
        queries = _c(queries, np.float32)
        n, d = queries.shape
        order = np.empty(max(n, 1), np.uint64)
        off = np.empty(n + 1, np.uint64)
        nb = self.check(self.L.ref_group_microbatches(queries.reshape(-1), n, d, int(m),
                                                      order, off))
        return [order[off[b]:off[b + 1]].tolist() for b in range(nb)]

    def split_budget(self, total, batch):
        b = _c(batch, np.uint64)
        out = np.empty(max(b.size, 1), np.uint64)
        self.check(self.L.ref_split_budget(int(total), b, b.size, out))
        return out[: b.size].copy()


class RefIndex:
    """laiv::IvfIndex + laiv::EmbeddingMatrix held by the reference library."""

    def __init__(self, lib: RefLib, centroids, vecs, ids, list_off, metric):
        self.lib = lib
        self.centroids = _c(centroids, np.float32)
        self.nc, self.d = self.centroids.shape
        self._vecs = _c(vecs, np.float32)
        self._ids = _c(ids, np.uint64)
        self._off = _c(list_off, np.uint64)
        h = lib.L.ref_index_create(self.centroids.reshape(-1), self.nc, self.d, metric,
                                   self._vecs.ctypes.data, self._ids.ctypes.data, self._off)
        if not h:
            raise RuntimeError(lib.err())
        self.h = h
        self.metric = metric

    def close(self):
        if self.h:
            self.lib.L.ref_index_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def cluster_bytes(self):
        return np.array([self.lib.L.ref_cluster_bytes(self.h, c) for c in range(self.nc)],
                        np.uint64)

    def rank_clusters(self, q):
        out = np.empty(self.nc, np.uint32)
        self.lib.check(self.lib.L.ref_rank_clusters(self.h, _c(q, np.float32), out))
        return out

    def coarse_probe(self, q, L):
        out = np.empty(max(self.nc, 1), np.uint32)
        n = self.lib.check(self.lib.L.ref_coarse_probe(self.h, _c(q, np.float32), int(L), out))
        return out[:n].copy()

    def search_clusters(self, q, clusters, k):
        cl = _c(clusters, np.uint32)
        oid = np.empty(max(k, 1), np.uint64)
        osc = np.empty(max(k, 1), np.float32)
        n = self.lib.check(self.lib.L.ref_search_clusters(self.h, _c(q, np.float32), cl,
                                                          cl.size, int(k), oid, osc))
        return oid[:n].copy(), osc[:n].copy()

    def ivf_search(self, q, L, k):
        oid = np.empty(max(k, 1), np.uint64)
        osc = np.empty(max(k, 1), np.float32)
        n = self.lib.check(self.lib.L.ref_ivf_search(self.h, _c(q, np.float32), int(L),
                                                     int(k), oid, osc))
        return oid[:n].copy(), osc[:n].copy()

    def score_clusters(self, q, clusters):
        cl = _c(clusters, np.uint32)
        cap = int(sum(int(self._off[c + 1] - self._off[c]) for c in cl if c < self.nc))
        oid = np.empty(max(cap, 1), np.uint64)
        osc = np.empty(max(cap, 1), np.float32)
        n = self.lib.L.ref_score_clusters(self.h, _c(q, np.float32), cl, cl.size, cap, oid, osc)
        if n < 0:
            raise ValueError(self.lib.err())
        return oid[:n].copy(), osc[:n].copy()

    def exact_search(self, q, k):
        oid = np.empty(max(k, 1), np.uint64)
        osc = np.empty(max(k, 1), np.float32)
        n = self.lib.check(self.lib.L.ref_exact_search(self.h, _c(q, np.float32), int(k),
                                                       oid, osc))
        return oid[:n].copy(), osc[:n].copy()

    def hybrid_search(self, resident, q, L, k):
        oid = np.empty(max(k, 1), np.uint64)
        osc = np.empty(max(k, 1), np.float32)
        fast = np.empty(max(self.nc, 1), np.uint32)
        slow = np.empty(max(self.nc, 1), np.uint32)
        nf, ns, hr = C.c_uint32(), C.c_uint32(), C.c_double()
        n = self.lib.check(self.lib.L.ref_hybrid_search(
            self.h, _c(resident, np.uint8), _c(q, np.float32), int(L), int(k), oid, osc,
            fast, C.byref(nf), slow, C.byref(ns), C.byref(hr)))
        return dict(ids=oid[:n].copy(), scores=osc[:n].copy(), fast=fast[: nf.value].copy(),
                    slow=slow[: ns.value].copy(), hit_rate=hr.value)

    def plan_prefetch(self, q, budget, resident):
        plan = np.empty(max(self.nc, 1), np.uint32)
        skipped = np.empty(max(self.nc, 1), np.uint32)
        npl, ns, pb = C.c_uint32(), C.c_uint32(), C.c_uint64()
        self.lib.check(self.lib.L.ref_plan_prefetch(
            self.h, _c(q, np.float32), int(budget), _c(resident, np.uint8), plan,
            C.byref(npl), C.byref(pb), skipped, C.byref(ns)))
        return plan[: npl.value].copy(), int(pb.value), skipped[: ns.value].copy()

    def coverage(self, q_in, q_out, L):
        return float(self.lib.L.ref_coverage(self.h, _c(q_in, np.float32),
                                             _c(q_out, np.float32), int(L)))

    def assign_cache_aware(self, batches, resident, queries, L):
        off, mem = Oracle._csr(batches)
        resident = _c(resident, np.uint8)
        q = _c(queries, np.float32)
        out = np.empty(max(len(batches), 1), np.uint32)
        self.lib.check(self.lib.L.ref_assign_cache_aware(
            self.h, off, mem, len(batches), resident.reshape(-1), resident.shape[0],
            q.reshape(-1), q.shape[0], int(L), out))
        return out[: len(batches)].copy()

    def search_many(self, Q, L, k, threads, mode=0):
        """Reference ivf_search (mode 0) / hybrid_search with an empty store
        (mode 1) over nq queries on `threads` host threads; returns ids,
        scores and per-query latency (s)."""
        Q = _c(Q, np.float32)
        nq = Q.shape[0]
        ids = np.zeros((nq, k), np.uint64)
        sc = np.zeros((nq, k), np.float32)
        lat = np.zeros(nq, np.float64)
        self.lib.check(self.lib.L.ref_search_many(self.h, mode, Q.ctypes.data, nq, int(L),
                                                  int(k), int(threads), ids.reshape(-1),
                                                  sc.reshape(-1), lat.ctypes.data))
        return ids, sc, lat
