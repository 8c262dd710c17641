"""Python mirror of the reference `laiv` hot-path interface, backed by liblaivg.

Names, argument meaning and error behaviour follow
/root/reference/proj/core/include/laiv/{vectorstore,ivf,tiered,sched,cache,
budget}.hpp so tests read like the reference's own. The one structural
difference: the reference threads ``(IvfIndex, EmbeddingMatrix, TieredStore)``
through every call, while here a :class:`Device` binds the index, one GPU and
that GPU's cluster cache (the TieredStore), so calls take the device first.

Exception mapping: std::invalid_argument -> ValueError, std::runtime_error ->
RuntimeError, std::logic_error -> LogicError, CUDA failures -> CudaError.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
import enum
from dataclasses import dataclass, field

import numpy as np

from ._lib import (Channel, CostModelC, CudaError, HybridTimingC, LogicError, Opts,
                   TransferReportC, check, lib)

__all__ = [
    "Metric", "ScoredId", "TopK", "IvfIndex", "Device", "TieredStore", "Residency",
    "ChannelMode", "TransferChannel", "PrefetchPlan", "TransferReport", "CostModel",
    "HybridResult", "HybridTiming", "MicroBatch", "WorkerState", "HotnessTable",
    "CacheParams", "rank_clusters", "coarse_probe", "search_clusters", "ivf_search",
    "plan_prefetch", "execute_prefetch", "incremental_prefetch", "hybrid_search",
    "coverage", "hybrid_search_batch", "prefetch_batch", "slow_tier_scan", "BatchResult", "ivf_search_batch",
    "group_microbatches", "chunk_microbatches", "assign_cache_aware",
    "assign_round_robin", "assignment_overlap", "split_budget", "default_nprobe",
    "LogicError", "CudaError", "synth_centroids", "synth_lists", "synth_queries",
    "synth_queries_topical", "group_microbatches_gpu", "schedule",
]


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class Metric(enum.IntEnum):          # vectorstore.hpp:18
    InnerProduct = 0
    L2 = 1


class Residency(enum.IntEnum):       # tiered.hpp:17
    Prefetched = 0
    Cached = 1


class ChannelMode(enum.IntEnum):     # tiered.hpp:65 (+ Device)
    SimulatedClock = 0
    Measured = 1
    Device = 2


@dataclass(frozen=True)
class ScoredId:                      # vectorstore.hpp:23-28
    id: int
    score: float


@dataclass
class TopK:                          # vectorstore.hpp:42-47
    k: int
    entries: list[ScoredId] = field(default_factory=list)

    @property
    def ids(self) -> np.ndarray:
        return np.array([e.id for e in self.entries], np.uint64)

    @property
    def scores(self) -> np.ndarray:
        return np.array([e.score for e in self.entries], np.float32)


def default_nprobe(n_clusters: int) -> int:  # ivf.cpp:264-267
    return max(1, int(np.floor(4.0 * np.sqrt(float(n_clusters)) + 0.5)))


def _view(addr, n, dtype):
    """numpy view of n elements of library memory at addr (no copy)."""
    if n == 0 or not addr:
        return np.zeros(0, dtype)
    buf = (C.c_char * (n * np.dtype(dtype).itemsize)).from_address(addr)
    return np.frombuffer(buf, dtype, n)


def load_index(path, threads: int = 0) -> "IvfIndex":   # ivf.hpp:98
    return IvfIndex.load(path, threads)


def save_index(path, ix: "IvfIndex", threads: int = 0) -> None:   # ivf.hpp:96
    ix.save(path, threads)


class IvfIndex:
    """IvfIndex + EmbeddingMatrix over a list-major store (ivf.hpp:26-50).

    ``vecs[N, D]`` rows are ordered list by list (the LAIX layout,
    ivf.cpp:373-388), ``ids[N]`` their ids and ``list_off[nc + 1]`` the list
    boundaries. ``borrow=True`` keeps the caller's arrays (they must outlive
    the index; pinned via :func:`pinned_empty` for full copy bandwidth).
    """

    def __init__(self, centroids, vecs, ids, list_off, metric: Metric,
                 borrow: bool = False, trust: bool = False):
        L = lib()
        self.centroids = _c(centroids, np.float32)
        if self.centroids.ndim != 2:
            raise ValueError("centroids must be [nc, d]")
        self.nc, self.d = self.centroids.shape
        self.list_off = _c(list_off, np.uint64)
        if self.list_off.size != self.nc + 1:
            raise ValueError("centroid/list count mismatch")
        self.metric = Metric(metric)
        self._vecs = _c(vecs, np.float32).reshape(-1, self.d) if self.d else None
        self._ids = _c(ids, np.uint64)
        flags = (1 if borrow else 0) | (2 if trust else 0)
        h = C.c_void_p()
        check(L.laivg_index_create(self.centroids.ctypes.data, self.nc, self.d, int(metric),
                                   self._vecs.ctypes.data, self._ids.ctypes.data,
                                   self.list_off.ctypes.data, flags, C.byref(h)))
        self.h = h
        if not borrow:  # the library holds its own pinned copy
            self._vecs = None
            self._ids = None

    @classmethod
    def from_lists(cls, centroids, lists, db_ids, db_vecs, metric: Metric):
        """Build the list-major store from reference-style lists of ids over a
        row store (ids -> rows), as load_index does (ivf.cpp:437-455)."""
        db_ids = np.asarray(db_ids, np.uint64)
        row_of = {int(i): r for r, i in enumerate(db_ids)}
        off = [0]
        rows = []
        for lst in lists:
            for i in lst:
                if int(i) not in row_of:
                    raise RuntimeError(f"index references id {int(i)} missing from the datastore")
                rows.append(row_of[int(i)])
            off.append(len(rows))
        rows = np.array(rows, np.int64)
        d = np.asarray(centroids).shape[1]
        vecs = np.asarray(db_vecs, np.float32)[rows] if len(rows) else np.zeros((0, d), np.float32)
        return cls(centroids, vecs, db_ids[rows] if len(rows) else np.zeros(0, np.uint64),
                   np.array(off, np.uint64), metric)

    @classmethod
    def load(cls, path, threads: int = 0) -> "IvfIndex":
        """load_index (ivf.hpp:98): a LAIX file read straight into the
        library's pinned list-major store (laivg_index_load)."""
        h = C.c_void_p()
        check(lib().laivg_index_load(os.fsencode(path), threads, C.byref(h)))
        self = cls.__new__(cls)
        self.h = h
        self.nc = int(lib().laivg_index_num_clusters(h))
        self.d = int(lib().laivg_index_dim(h))
        self.metric = Metric(lib().laivg_index_metric(h))
        v, i, o, c = (C.c_void_p() for _ in range(4))
        check(lib().laivg_index_store(h, C.byref(v), C.byref(i), C.byref(o), C.byref(c)))
        self.list_off = _view(o.value, self.nc + 1, np.uint64).copy()
        self.centroids = _view(c.value, self.nc * self.d, np.float32).reshape(self.nc, self.d).copy()
        self._vecs = None
        self._ids = None
        return self

    def save(self, path, threads: int = 0) -> None:
        """save_index (ivf.hpp:96): the LAIX bytes of this index."""
        check(lib().laivg_index_save(self.h, os.fsencode(path), threads))

    def store(self):
        """Zero-copy (vecs[N, d], ids[N]) views of the library's store; valid
        while this index lives."""
        v, i = C.c_void_p(), C.c_void_p()
        check(lib().laivg_index_store(self.h, C.byref(v), C.byref(i), None, None))
        n = int(self.list_off[-1])
        return (_view(v.value, n * self.d, np.float32).reshape(n, self.d),
                _view(i.value, n, np.uint64))

    def close(self):
        if getattr(self, "h", None):
            live = [d for d in getattr(self, "_devices", ()) if getattr(d, "h", None)]
            if live:
                raise LogicError(f"IvfIndex.close() while {len(live)} Device(s) still use it: "
                                 "close them first (their contexts copy lists from this store)")
            lib().laivg_index_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def num_clusters(self) -> int:
        return self.nc

    def dim(self) -> int:
        return self.d

    def cluster_bytes(self, c: int) -> int:          # ivf.hpp:40
        if not 0 <= c < self.nc:
            raise IndexError("cluster out of range")
        return int(lib().laivg_index_cluster_bytes(self.h, c))

    def total_payload_bytes(self) -> int:            # ivf.hpp:41
        return int(lib().laivg_index_total_payload_bytes(self.h))

    def total_vectors(self) -> int:
        return int(lib().laivg_index_total_vectors(self.h))

    def list_len(self, c: int) -> int:
        return int(self.list_off[c + 1] - self.list_off[c])


class TieredStore:
    """The GPU cluster cache of a Device (tiered.hpp:22-56)."""

    def __init__(self, dev: "Device"):
        # weak: a Device must be freed by refcount as soon as the caller drops
        # it (its cluster cache can hold most of HBM)
        self._dev = weakref.ref(dev)

    @property
    def _h(self):
        dev = self._dev()
        if dev is None or not dev.h:
            raise LogicError("TieredStore used after its Device was closed")
        return dev.h

    def capacity_bytes(self) -> int:
        return int(lib().laivg_store_capacity_bytes(self._h))

    def used_bytes(self) -> int:
        return int(lib().laivg_store_used_bytes(self._h))

    def free_bytes(self) -> int:
        return int(lib().laivg_store_free_bytes(self._h))

    def contains(self, c: int) -> bool:
        return bool(lib().laivg_store_contains(self._h, c))

    def resident_count(self) -> int:
        return int(lib().laivg_store_resident_count(self._h))

    def resident(self) -> dict[int, tuple[Residency, int]]:
        n = self.resident_count()
        cl = np.zeros(max(n, 1), np.uint32)
        tg = np.zeros(max(n, 1), np.uint8)
        by = np.zeros(max(n, 1), np.uint64)
        got = C.c_uint32()
        check(lib().laivg_store_resident(self._h, cl.ctypes.data, tg.ctypes.data,
                                         by.ctypes.data, C.byref(got)))
        return {int(cl[i]): (Residency(int(tg[i])), int(by[i])) for i in range(got.value)}

    def insert(self, c: int, tag: Residency = Residency.Prefetched) -> None:
        check(lib().laivg_store_insert(self._h, c, int(tag)))

    def evict(self, c: int) -> int:
        b = C.c_uint64()
        check(lib().laivg_store_evict(self._h, c, C.byref(b)))
        return int(b.value)

    def retag_all(self, tag: Residency) -> None:
        check(lib().laivg_store_retag_all(self._h, int(tag)))

    def clear(self) -> None:
        check(lib().laivg_store_clear(self._h))

    def bytes_with_tag(self, tag: Residency) -> int:
        return int(lib().laivg_store_bytes_with_tag(self._h, int(tag)))

    def recompute_used_bytes(self) -> int:
        return int(lib().laivg_store_recompute_used_bytes(self._h))

    def compact(self) -> None:
        check(lib().laivg_store_compact(self._h))

    def resident_mask(self, nc: int) -> np.ndarray:
        m = np.zeros(nc, np.uint8)
        for c in self.resident():
            m[c] = 1
        return m


class Device:
    """One GPU bound to an index, with its cluster cache and streams."""

    def __init__(self, ix: IvfIndex, capacity_bytes: int, device: int = 0,
                 miss_threads: int = 0, max_batch: int = 0, max_probe: int = 0,
                 acc_fp64: bool = True, scan_impl: str = "tma", tma_tile: int = 0,
                 tma_stages: int = 0, ctas_per_sm: int = 0, coarse_impl: str = "auto",
                 miss_fetch: str = "auto", fetch_chunk_mb: int = 0,
                 single_query: str = "fused"):
        L = lib()
        o = Opts()
        L.laivg_opts_default(C.byref(o))
        o.device = device
        o.capacity_bytes = int(capacity_bytes)
        o.miss_threads = miss_threads
        o.max_batch = max_batch
        o.max_probe = max_probe
        o.acc_fp64 = 1 if acc_fp64 else 0
        if scan_impl not in ("tma", "ldg"):
            raise ValueError("scan_impl must be 'tma' or 'ldg'")
        o.scan_impl = 0 if scan_impl == "tma" else 1
        o.tma_tile, o.tma_stages, o.ctas_per_sm = tma_tile, tma_stages, ctas_per_sm
        impls = {"auto": 0, "fp64": 1, "tensor": 2}
        if coarse_impl not in impls:
            raise ValueError("coarse_impl must be 'auto', 'fp64' or 'tensor'")
        o.coarse_impl = impls[coarse_impl]
        fetches = {"off": 0, "auto": 1, "all": 2}
        if miss_fetch not in fetches:
            raise ValueError("miss_fetch must be 'off', 'auto' or 'all'")
        o.miss_fetch = fetches[miss_fetch]
        o.fetch_chunk_mb = fetch_chunk_mb
        if single_query not in ("fused", "chain"):
            raise ValueError("single_query must be 'fused' or 'chain'")
        o.single_chain = 0 if single_query == "fused" else 1
        h = C.c_void_p()
        check(L.laivg_ctx_create(ix.h, C.byref(o), C.byref(h)))
        self.h = h
        self.ix = ix
        if not hasattr(ix, "_devices"):
            ix._devices = weakref.WeakSet()
        ix._devices.add(self)
        self.store = TieredStore(self)

    def close(self):
        if getattr(self, "h", None):
            lib().laivg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        check(lib().laivg_ctx_sync(self.h))

    def window(self, seconds: float) -> float:
        out = C.c_double()
        check(lib().laivg_window(self.h, seconds, C.byref(out)))
        return out.value

    def window_load(self, buffer_bytes: int, read_gbps: float) -> None:
        """Decode-like generation windows: stream `buffer_bytes` of HBM once per
        token period (buffer_bytes / read_gbps); 0 restores the idle window."""
        check(lib().laivg_window_load(self.h, int(buffer_bytes), float(read_gbps)))

    def link_peak(self, nbytes: int = 1 << 30) -> tuple[float, float]:
        """Pinned H2D / D2H GB/s of this GPU's host link (one large copy each)."""
        a, b = C.c_double(), C.c_double()
        check(lib().laivg_link_peak(self.h, int(nbytes), C.byref(a), C.byref(b)))
        return a.value, b.value

    def list_scan_stats(self) -> tuple[int, int, float]:
        """(batches on the list-major tensor-core scan, of which fell back to
        the per-query scan, EMA of queries per resident probed list)."""
        r, f, q = C.c_uint64(), C.c_uint64(), C.c_double()
        check(lib().laivg_list_scan_stats(self.h, C.byref(r), C.byref(f), C.byref(q)))
        return r.value, f.value, q.value

    def stage_queries(self, Q) -> None:
        Q = _c(Q, np.float32).reshape(-1, self.ix.d)
        self._staged = Q
        check(lib().laivg_stage_queries(self.h, Q.ctypes.data, Q.shape[0]))

    def hybrid_search_staged(self, qi: int, L: int, k: int):
        ids = np.empty(k, np.uint64)
        sc = np.empty(k, np.float32)
        cnt, nf = C.c_uint32(), C.c_uint32()
        t = HybridTimingC()
        check(lib().laivg_hybrid_search_staged(self.h, qi, L, k, ids.ctypes.data,
                                               sc.ctypes.data, C.byref(cnt), C.byref(nf),
                                               C.byref(t)))
        return ids[: cnt.value], sc[: cnt.value], nf.value, _timing(t)

    def hybrid_search_batch_staged(self, q0: int, nq: int, L: int, k: int):
        """Batched hybrid search over staged queries [q0, q0 + nq): returns
        ids[nq][k], scores[nq][k], counts[nq], nfast[nq] and the batch timing."""
        ids = np.empty((nq, k), np.uint64)
        sc = np.empty((nq, k), np.float32)
        cnt = np.empty(nq, np.uint32)
        nf = np.empty(nq, np.uint32)
        t = HybridTimingC()
        check(lib().laivg_hybrid_search_batch_staged(self.h, q0, nq, L, k, ids.ctypes.data,
                                                     sc.ctypes.data, cnt.ctypes.data,
                                                     nf.ctypes.data, C.byref(t)))
        return ids, sc, cnt, nf, _timing(t)

    # ---- peer caches (laivg.h, "peer caches") ----
    def epoch_open(self) -> None:
        check(lib().laivg_epoch_open(self.h))

    def epoch_close(self) -> None:
        check(lib().laivg_epoch_close(self.h))

    def store_offsets(self) -> np.ndarray:
        out = np.empty(self.ix.nc, np.int64)
        check(lib().laivg_store_offsets(self.h, out.ctypes.data))
        return out

    def slab_ipc_handle(self) -> bytes:
        buf = (C.c_char * 64)()
        check(lib().laivg_slab_ipc_handle(self.h, buf))
        return bytes(buf)

    def peer_attach(self, peer: int, other: "Device | None" = None,
                    ipc_handle: bytes | None = None) -> None:
        if other is not None:
            check(lib().laivg_peer_attach_local(self.h, peer, other.h))
        else:
            buf = (C.c_char * 64).from_buffer_copy(ipc_handle)
            check(lib().laivg_peer_attach_ipc(self.h, peer, buf))

    def peer_publish(self, peer: int, offsets) -> None:
        if offsets is None:
            check(lib().laivg_peer_publish(self.h, peer, None))
        else:
            o = _c(offsets, np.int64)
            check(lib().laivg_peer_publish(self.h, peer, o.ctypes.data))

    def coarse_approx(self, Q) -> np.ndarray:
        """Diagnostics: raw tf32 tensor-core coarse scores [nq][nc]."""
        Q = _c(Q, np.float32).reshape(-1, self.ix.d)
        out = np.empty((Q.shape[0], self.ix.nc), np.float32)
        check(lib().laivg_debug_coarse_approx(self.h, Q.ctypes.data, Q.shape[0],
                                              out.ctypes.data))
        return out


# --------------------------------------------------------------------------
# ivf.hpp
# --------------------------------------------------------------------------
def rank_clusters(dev: Device, q, with_scores: bool = False):     # ivf.hpp:68-69
    Q = _c(q, np.float32).reshape(-1, dev.ix.d)
    nq, nc = Q.shape[0], dev.ix.nc
    order = np.empty((nq, nc), np.uint32)
    scores = np.empty((nq, nc), np.float64) if with_scores else None
    check(lib().laivg_rank_clusters(dev.h, Q.ctypes.data, nq, order.ctypes.data, _ptr(scores)))
    if np.ndim(q) == 1:
        order = order[0]
        scores = None if scores is None else scores[0]
    return (order, scores) if with_scores else order


def coarse_probe(dev: Device, q, L: int):                         # ivf.hpp:72-73
    Q = _c(q, np.float32).reshape(-1, dev.ix.d)
    nq = Q.shape[0]
    lp = min(max(int(L), 0), dev.ix.nc)
    out = np.empty((nq, max(lp, 1)), np.uint32)
    got = C.c_uint32()
    check(lib().laivg_coarse_probe(dev.h, Q.ctypes.data, nq, int(L), out.ctypes.data,
                                   C.byref(got)))
    out = out[:, : got.value]
    return out[0] if np.ndim(q) == 1 else out


def _check_q(dev: Device, q) -> np.ndarray:
    q = _c(q, np.float32).reshape(-1)
    if q.size != dev.ix.d:
        raise ValueError("query dim mismatch")
    return q


def search_clusters(dev: Device, q, clusters, k: int) -> TopK:    # ivf.hpp:85-87
    q = _check_q(dev, q)
    cl = _c(clusters, np.uint32)
    ids = np.empty(max(k, 1), np.uint64)
    sc = np.empty(max(k, 1), np.float32)
    cnt = C.c_uint32()
    check(lib().laivg_search_clusters(dev.h, q.ctypes.data, cl.ctypes.data, cl.size, int(k),
                                      ids.ctypes.data, sc.ctypes.data, C.byref(cnt)))
    return TopK(k, [ScoredId(int(ids[i]), float(sc[i])) for i in range(cnt.value)])


def score_clusters(dev: Device, q, clusters) -> list[ScoredId]:   # ivf.hpp:75-81
    """Every member of ``clusters`` (in order, duplicates included) scored
    against q, unranked (ivf.cpp:301-324); resident lists on the GPU."""
    q = _check_q(dev, q)
    cl = _c(clusters, np.uint32).reshape(-1)
    if cl.size and int(cl.max()) >= dev.ix.nc:
        bad = int(cl[np.argmax(cl >= dev.ix.nc)])
        raise ValueError(f"unknown cluster id {bad}")
    n = int(sum(dev.ix.list_len(int(c)) for c in cl))
    ids = np.empty(max(n, 1), np.uint64)
    sc = np.empty(max(n, 1), np.float32)
    got = C.c_uint64()
    check(lib().laivg_score_clusters(dev.h, q.ctypes.data, _ptr(cl if cl.size else None), cl.size,
                                     n, ids.ctypes.data, sc.ctypes.data, C.byref(got)))
    return [ScoredId(int(ids[i]), float(sc[i])) for i in range(got.value)]


def score_clusters_arrays(dev: Device, q, clusters):
    """score_clusters as (ids[n], scores[n]) arrays."""
    q = _check_q(dev, q)
    cl = _c(clusters, np.uint32).reshape(-1)
    n = int(sum(dev.ix.list_len(int(c)) for c in cl if 0 <= int(c) < dev.ix.nc))
    ids = np.empty(max(n, 1), np.uint64)
    sc = np.empty(max(n, 1), np.float32)
    got = C.c_uint64()
    check(lib().laivg_score_clusters(dev.h, q.ctypes.data, _ptr(cl if cl.size else None), cl.size,
                                     n, ids.ctypes.data, sc.ctypes.data, C.byref(got)))
    return ids[: got.value], sc[: got.value]


def exact_search(dev: Device, q, k: int) -> TopK:                 # vectorstore.hpp:94-98
    """Brute force over every row of the index's datastore (the union of its
    lists), any k >= 1; ties by ascending id (vectorstore.cpp:117-139)."""
    q = _check_q(dev, q)
    ids = np.empty(max(k, 1), np.uint64)
    sc = np.empty(max(k, 1), np.float32)
    cnt = np.zeros(1, np.uint32)
    check(lib().laivg_exact_search(dev.h, q.ctypes.data, 1, int(k), ids.ctypes.data,
                                   sc.ctypes.data, cnt.ctypes.data))
    return TopK(k, [ScoredId(int(ids[i]), float(sc[i])) for i in range(int(cnt[0]))])


def pairwise_l2(dev: Device, a, b) -> np.ndarray:                 # vectorstore.hpp:100-102
    """Dense a.count() x b.count() Euclidean distances (row-major f32), the
    reference's serial fp64 arithmetic on the device's GPU (bit-identical)."""
    A = np.ascontiguousarray(np.asarray(a, np.float32))
    B = np.ascontiguousarray(np.asarray(b, np.float32))
    if A.ndim != 2 or B.ndim != 2:
        raise ValueError("pairwise_l2: matrices must be 2-D")
    if A.shape[1] != B.shape[1]:
        raise ValueError("pairwise_l2: dim mismatch")
    out = np.empty((A.shape[0], B.shape[0]), np.float32)
    if out.size == 0:
        return out.reshape(-1)
    check(lib().laivg_pairwise_l2(dev.h, A.ctypes.data, A.shape[0], B.ctypes.data, B.shape[0],
                                  A.shape[1], out.ctypes.data))
    return out.reshape(-1)


def ivf_search(dev: Device, q, L: int, k: int) -> TopK:           # ivf.hpp:90-91
    q = _check_q(dev, q)
    ids = np.empty(max(k, 1), np.uint64)
    sc = np.empty(max(k, 1), np.float32)
    cnt = np.zeros(1, np.uint32)
    check(lib().laivg_ivf_search(dev.h, q.ctypes.data, 1, int(L), int(k), ids.ctypes.data,
                                 sc.ctypes.data, cnt.ctypes.data))
    return TopK(k, [ScoredId(int(ids[i]), float(sc[i])) for i in range(int(cnt[0]))])


def slow_tier_scan(ix: IvfIndex, Q, lists_per_query, k: int, threads: int = 0) -> list[TopK]:
    """The host (slow) tier of hybrid_search on its own: per query, the best-k
    over the members of the given clusters, scored on the host with the
    reference's fp64 arithmetic (tiered.cpp:169)."""
    Q = _c(Q, np.float32).reshape(-1, ix.d)
    nq = Q.shape[0]
    if len(lists_per_query) != nq:
        raise ValueError("one cluster list per query")
    off = np.zeros(nq + 1, np.uint32)
    for q, ls in enumerate(lists_per_query):
        off[q + 1] = off[q] + len(ls)
    flat = _c([c for ls in lists_per_query for c in ls] or [0], np.uint32)
    ids = np.empty((max(nq, 1), max(k, 1)), np.uint64)
    sc = np.empty((max(nq, 1), max(k, 1)), np.float32)
    cnt = np.zeros(max(nq, 1), np.uint32)
    check(lib().laivg_slow_tier_scan(ix.h, Q.ctypes.data, nq, flat.ctypes.data, off.ctypes.data,
                                     int(k), threads, ids.ctypes.data, sc.ctypes.data,
                                     cnt.ctypes.data))
    return [TopK(k, [ScoredId(int(ids[q, i]), float(sc[q, i])) for i in range(int(cnt[q]))])
            for q in range(nq)]


def ivf_search_batch(dev: Device, Q, L: int, k: int) -> list[TopK]:
    """ivf_search for a batch (one device pass per max_batch queries)."""
    Q = _c(Q, np.float32).reshape(-1, dev.ix.d)
    nq = Q.shape[0]
    ids = np.empty((nq, max(k, 1)), np.uint64)
    sc = np.empty((nq, max(k, 1)), np.float32)
    cnt = np.zeros(nq, np.uint32)
    check(lib().laivg_ivf_search(dev.h, Q.ctypes.data, nq, int(L), int(k), ids.ctypes.data,
                                 sc.ctypes.data, cnt.ctypes.data))
    return [TopK(k, [ScoredId(int(ids[q, i]), float(sc[q, i])) for i in range(int(cnt[q]))])
            for q in range(nq)]


# --------------------------------------------------------------------------
# tiered.hpp / budget.hpp
# --------------------------------------------------------------------------
@dataclass
class TransferChannel:                                            # tiered.hpp:68-74
    bandwidth_bytes_per_s: float = 32e9
    mode: ChannelMode = ChannelMode.SimulatedClock

    def transfer_time_s(self, nbytes: int) -> float:
        return float(nbytes) / self.bandwidth_bytes_per_s


@dataclass
class PrefetchPlan:                                               # tiered.hpp:59-63
    clusters: list[int] = field(default_factory=list)
    planned_bytes: int = 0
    skipped: list[int] = field(default_factory=list)


@dataclass
class TransferReport:                                             # tiered.hpp:76-82
    t_p: float = 0.0
    transferred: list[int] = field(default_factory=list)
    bytes: int = 0
    overshoot_s: float = 0.0
    window_s: float = 0.0
    h2d_gbps: float = 0.0
    window_read_gbps: float = 0.0  # HBM read rate of a decode-like window (0: idle window)


@dataclass
class CostModel:                                                  # budget.hpp:13-24
    bandwidth_bytes_per_s: float = 32e9
    t_cc: float = 1e-3
    t_gc: float = 1e-5
    parallel_slots: int = 1

    def validate(self):
        if not (self.bandwidth_bytes_per_s > 0 and self.t_cc > 0 and self.t_gc > 0
                and self.parallel_slots > 0):
            raise ValueError("cost model fields must be positive")


@dataclass
class HybridTiming:                                               # tiered.hpp:84-88
    t_g: float = 0.0
    t_c: float = 0.0
    t_2: float = 0.0
    model_t_g: float = 0.0
    model_t_c: float = 0.0
    model_t_2: float = 0.0
    t_coarse: float = 0.0
    t_scan: float = 0.0
    scanned_vectors: int = 0
    scanned_bytes: int = 0
    fetched_lists: int = 0     # misses fetched H2D on demand and scanned on the GPU
    cpu_lists: int = 0         # distinct misses scanned by the host
    fetched_bytes: int = 0
    t_fetch: float = 0.0
    peer_lists: int = 0        # misses copied from a peer GPU's cache (NVLink)
    peer_bytes: int = 0
    h2d_bytes: int = 0         # host-link bytes the call moved (counted by the library)
    d2h_bytes: int = 0
    t_kernel: float = 0.0      # fused single-query kernel duration (0: multi-kernel chain)
    list_scan: int = 0         # batch hits scanned by the list-major tensor-core scan
    distinct_bytes: int = 0    # batch: vector bytes of the distinct resident probed lists


@dataclass
class HybridResult:                                               # tiered.hpp:90-95
    topk: TopK
    fast_clusters: list[int]
    slow_clusters: list[int]
    hit_rate: float


def _timing(t: HybridTimingC) -> HybridTiming:
    return HybridTiming(t.t_g, t.t_c, t.t_2, t.model_t_g, t.model_t_c, t.model_t_2,
                        t.t_coarse, t.t_scan, int(t.scanned_vectors), int(t.scanned_bytes),
                        int(t.fetched_lists), int(t.cpu_lists), int(t.fetched_bytes), t.t_fetch,
                        int(t.peer_lists), int(t.peer_bytes), int(t.h2d_bytes),
                        int(t.d2h_bytes), t.t_kernel, int(t.list_scan), int(t.distinct_bytes))


def plan_prefetch(dev: Device, q_in, budget_bytes: int) -> PrefetchPlan:  # tiered.hpp:100-101
    q = _check_q(dev, q_in)
    nc = dev.ix.nc
    plan = np.empty(max(nc, 1), np.uint32)
    skipped = np.empty(max(nc, 1), np.uint32)
    npl, ns, pb = C.c_uint32(), C.c_uint32(), C.c_uint64()
    check(lib().laivg_plan_prefetch(dev.h, q.ctypes.data, int(budget_bytes), plan.ctypes.data,
                                    C.byref(npl), C.byref(pb), skipped.ctypes.data, C.byref(ns)))
    return PrefetchPlan(plan[: npl.value].tolist(), int(pb.value), skipped[: ns.value].tolist())


def _report(r: TransferReportC, transferred) -> TransferReport:
    return TransferReport(r.t_p, list(transferred), int(r.bytes), r.overshoot_s, r.window_s,
                          r.h2d_gbps, r.window_read_gbps)


def execute_prefetch(dev: Device, plan: PrefetchPlan, chan: TransferChannel,
                     overlap_window_s: float = 0.0) -> TransferReport:  # tiered.hpp:107-110
    cl = _c(plan.clusters, np.uint32)
    out = np.empty(max(cl.size, 1), np.uint32)
    ch = Channel(chan.bandwidth_bytes_per_s, int(chan.mode))
    r = TransferReportC()
    check(lib().laivg_execute_prefetch(dev.h, cl.ctypes.data, cl.size, C.byref(ch),
                                       overlap_window_s, out.ctypes.data, C.byref(r)))
    return _report(r, out[: r.n_transferred].tolist())


def prefetch_batch(dev: Device, Q_in, budgets, chan: TransferChannel,
                   overlap_window_s: float = 0.0):
    """Lookahead prefetch of a micro-batch: one coarse pass, sequential plans
    against the filling store (pipeline.cpp:357-371), one window. Returns the
    TransferReport and each query's planned count."""
    Q = _c(Q_in, np.float32).reshape(-1, dev.ix.d)
    nq = Q.shape[0]
    b = _c(budgets, np.uint64)
    if b.size != nq:
        raise ValueError("one budget per query")
    out = np.empty(max(dev.ix.nc, 1), np.uint32)
    npl = np.empty(max(nq, 1), np.uint32)
    ch = Channel(chan.bandwidth_bytes_per_s, int(chan.mode))
    r = TransferReportC()
    check(lib().laivg_prefetch_batch(dev.h, Q.ctypes.data, nq, b.ctypes.data, C.byref(ch),
                                     overlap_window_s, out.ctypes.data, npl.ctypes.data,
                                     C.byref(r)))
    return _report(r, out[: r.n_transferred].tolist()), npl[:nq].copy()


def incremental_prefetch(dev: Device, q_round, budget_bytes: int, chan: TransferChannel,
                         overlap_window_s: float = 0.0) -> TransferReport:  # tiered.hpp:114-117
    q = _check_q(dev, q_round)
    out = np.empty(max(dev.ix.nc, 1), np.uint32)
    ch = Channel(chan.bandwidth_bytes_per_s, int(chan.mode))
    r = TransferReportC()
    check(lib().laivg_incremental_prefetch(dev.h, q.ctypes.data, int(budget_bytes), C.byref(ch),
                                           overlap_window_s, out.ctypes.data, C.byref(r)))
    return _report(r, out[: r.n_transferred].tolist())


def hybrid_search(dev: Device, q_out, L: int, k: int,
                  cost: CostModel | None = None):                 # tiered.hpp:125-128
    q = _check_q(dev, q_out)
    cost = cost or CostModel()
    nc = dev.ix.nc
    ids = np.empty(max(k, 1), np.uint64)
    sc = np.empty(max(k, 1), np.float32)
    fast = np.empty(max(nc, 1), np.uint32)
    slow = np.empty(max(nc, 1), np.uint32)
    cnt, nf, ns, hr = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_double()
    t = HybridTimingC()
    cm = CostModelC(cost.bandwidth_bytes_per_s, cost.t_cc, cost.t_gc, cost.parallel_slots)
    check(lib().laivg_hybrid_search(dev.h, q.ctypes.data, int(L), int(k), C.byref(cm),
                                    ids.ctypes.data, sc.ctypes.data, C.byref(cnt),
                                    fast.ctypes.data, C.byref(nf), slow.ctypes.data,
                                    C.byref(ns), C.byref(hr), C.byref(t)))
    res = HybridResult(TopK(k, [ScoredId(int(ids[i]), float(sc[i])) for i in range(cnt.value)]),
                       fast[: nf.value].tolist(), slow[: ns.value].tolist(), hr.value)
    return res, _timing(t)


@dataclass
class BatchResult:
    """Per-query results of hybrid_search_batch (extension point (2))."""
    ids: np.ndarray      # [nq][k] uint64 (unused slots: ~0)
    scores: np.ndarray   # [nq][k] float32
    counts: np.ndarray   # [nq]
    nfast: np.ndarray    # [nq] resident probed lists per query

    def topk(self, q: int) -> TopK:
        k = self.ids.shape[1]
        return TopK(k, [ScoredId(int(self.ids[q, i]), float(self.scores[q, i]))
                        for i in range(int(self.counts[q]))])


def hybrid_search_batch(dev: Device, Q, L: int, k: int, cost: CostModel | None = None):
    """hybrid_search for a batch of queries in one device pass (<= max_batch)."""
    Q = _c(Q, np.float32).reshape(-1, dev.ix.d)
    nq = Q.shape[0]
    cost = cost or CostModel()
    ids = np.empty((nq, max(k, 1)), np.uint64)
    sc = np.empty((nq, max(k, 1)), np.float32)
    cnt = np.empty(nq, np.uint32)
    nf = np.empty(nq, np.uint32)
    t = HybridTimingC()
    cm = CostModelC(cost.bandwidth_bytes_per_s, cost.t_cc, cost.t_gc, cost.parallel_slots)
    check(lib().laivg_hybrid_search_batch(dev.h, Q.ctypes.data, nq, int(L), int(k),
                                          C.byref(cm), ids.ctypes.data, sc.ctypes.data,
                                          cnt.ctypes.data, nf.ctypes.data, C.byref(t)))
    return BatchResult(ids, sc, cnt, nf), _timing(t)


def coverage(dev: Device, q_in, q_out, L: int) -> float:          # tiered.hpp:132-133
    a, b = _check_q(dev, q_in), _check_q(dev, q_out)
    out = C.c_double()
    check(lib().laivg_coverage(dev.h, a.ctypes.data, b.ctypes.data, int(L), C.byref(out)))
    return out.value


# --------------------------------------------------------------------------
# sched.hpp
# --------------------------------------------------------------------------
@dataclass
class MicroBatch:                                                 # sched.hpp:16-19
    queries: list[int] = field(default_factory=list)


@dataclass
class WorkerState:                                                # sched.hpp:21-26
    worker_id: int = 0
    resident_clusters: set[int] = field(default_factory=set)
    capacity_bytes: int = 0


def _batches_from_csr(order, off, nb):
    return [MicroBatch([int(x) for x in order[off[b]:off[b + 1]]]) for b in range(nb)]


def group_microbatches(queries, m: int) -> list[MicroBatch]:      # sched.hpp:31-32
    Q = _c(queries, np.float32)
    n, d = Q.shape
    if m < 1:
        raise ValueError("micro-batch size must be >= 1")
    order = np.empty(max(n, 1), np.uint64)
    off = np.empty(n + 1, np.uint64)
    nb = C.c_uint32()
    check(lib().laivg_group_microbatches(Q.ctypes.data, n, d, int(m), order.ctypes.data,
                                         off.ctypes.data, C.byref(nb)))
    return _batches_from_csr(order, off, nb.value)


def chunk_microbatches(n: int, m: int) -> list[MicroBatch]:      # sched.hpp:36
    if m < 1:
        raise ValueError("micro-batch size must be >= 1")
    order = np.empty(max(n, 1), np.uint64)
    off = np.empty(n + 2, np.uint64)
    nb = C.c_uint32()
    check(lib().laivg_chunk_microbatches(int(n), int(m), order.ctypes.data, off.ctypes.data,
                                         C.byref(nb)))
    return _batches_from_csr(order, off, nb.value)


def _csr(batches):
    off = np.zeros(len(batches) + 1, np.uint64)
    for i, b in enumerate(batches):
        off[i + 1] = off[i] + len(b.queries)
    mem = np.array([x for b in batches for x in b.queries] or [0], np.uint64)
    return off, mem


def _resident_matrix(workers, nc):
    r = np.zeros((max(len(workers), 1), nc), np.uint8)
    for i, w in enumerate(workers):
        for c in w.resident_clusters:
            if 0 <= c < nc:
                r[i, c] = 1
    return r


def assign_cache_aware(dev: Device, batches: list[MicroBatch], workers: list[WorkerState],
                       queries, L: int) -> list[int]:             # sched.hpp:42-45
    if not workers:
        raise ValueError("need at least one worker")
    off, mem = _csr(batches)
    res = _resident_matrix(workers, dev.ix.nc)
    Q = _c(queries, np.float32)
    out = np.empty(max(len(batches), 1), np.uint32)
    check(lib().laivg_assign_cache_aware(dev.h, off.ctypes.data, mem.ctypes.data, len(batches),
                                         res.ctypes.data, len(workers), Q.ctypes.data,
                                         Q.shape[0], int(L), out.ctypes.data))
    return out[: len(batches)].tolist()


def greedy_assign(overlap) -> list[int]:                          # sched.cpp:114-142
    """assign_cache_aware's greedy over a precomputed [nb, nw] overlap matrix."""
    ov = _c(overlap, np.uint64)
    if ov.ndim != 2:
        raise ValueError("overlap must be [batches, workers]")
    nb, nw = ov.shape
    out = np.empty(max(nb, 1), np.uint32)
    check(lib().laivg_greedy_assign(ov.ctypes.data, nb, nw, out.ctypes.data))
    return out[:nb].tolist()


def assign_round_robin(n_batches: int, n_workers: int) -> list[int]:  # sched.hpp:48
    out = np.empty(max(n_batches, 1), np.uint32)
    check(lib().laivg_assign_round_robin(n_batches, n_workers, out.ctypes.data))
    return out[:n_batches].tolist()


def assignment_overlap(dev: Device, batches, workers, assignment, queries,
                       L: int) -> int:                            # sched.hpp:51-55
    off, mem = _csr(batches)
    res = _resident_matrix(workers, dev.ix.nc)
    Q = _c(queries, np.float32)
    a = _c(assignment, np.uint32)
    out = C.c_uint64()
    check(lib().laivg_assignment_overlap(dev.h, off.ctypes.data, mem.ctypes.data, len(batches),
                                         res.ctypes.data, len(workers), a.ctypes.data,
                                         Q.ctypes.data, Q.shape[0], int(L), C.byref(out)))
    return int(out.value)


def split_budget(total_budget_bytes: int, batch: MicroBatch) -> list[int]:  # sched.hpp:59-60
    b = _c(batch.queries, np.uint64)
    out = np.empty(max(b.size, 1), np.uint64)
    check(lib().laivg_split_budget(int(total_budget_bytes), b.ctypes.data, b.size,
                                   out.ctypes.data))
    return [int(x) for x in out[: b.size]]


# --------------------------------------------------------------------------
# cache.hpp
# --------------------------------------------------------------------------
@dataclass
class CacheParams:                                                # cache.hpp:15-22
    h_init: float = 1.0
    h_inc: float = 1.0
    decay: float = 2.0
    cache_fraction: float = 0.5


class HotnessTable:                                               # cache.hpp:28-56
    def __init__(self, params: CacheParams | None = None):
        p = params or CacheParams()
        h = C.c_void_p()
        check(lib().laivg_hotness_create(p.h_init, p.h_inc, p.decay, p.cache_fraction,
                                         C.byref(h)))
        self.h = h
        self.params = p

    def __del__(self):
        try:
            if self.h:
                lib().laivg_hotness_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def on_fetch(self, c: int) -> None:
        check(lib().laivg_hotness_on_fetch(self.h, c))

    def end_of_round(self, used) -> None:
        u = _c(sorted(used) or [0], np.uint32)
        check(lib().laivg_hotness_end_of_round(self.h, u.ctypes.data, len(used)))

    def evict_to_fraction(self, dev: Device) -> list[int]:
        out = np.empty(max(dev.store.resident_count(), 1), np.uint32)
        n = C.c_uint32()
        check(lib().laivg_hotness_evict_to_fraction(self.h, dev.h, out.ctypes.data, C.byref(n)))
        return out[: n.value].tolist()

    def tracked(self, c: int) -> bool:
        return lib().laivg_hotness_get(self.h, c) >= 0.0

    def hotness(self, c: int) -> float:
        v = lib().laivg_hotness_get(self.h, c)
        if v < 0:
            raise KeyError(c)
        return float(np.float32(v))

    def forget(self, c: int) -> None:
        check(lib().laivg_hotness_forget(self.h, c))

    def clear(self) -> None:
        check(lib().laivg_hotness_clear(self.h))


# --------------------------------------------------------------------------
# synthetic workload + pinned memory
# --------------------------------------------------------------------------
def pinned_empty(shape, dtype) -> np.ndarray:
    """numpy array over portable pinned host memory (freed with the array)."""
    dt = np.dtype(dtype)
    n = int(np.prod(shape)) * dt.itemsize
    p = C.c_void_p()
    check(lib().laivg_host_alloc(n, C.byref(p)))
    buf = (C.c_char * max(n, 1)).from_address(p.value)
    buf._owner = _PinnedOwner(p.value)  # freed when the last view goes away
    return np.frombuffer(buf, dtype=dt, count=int(np.prod(shape))).reshape(shape)


class _PinnedOwner:
    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            lib().laivg_host_free(self.ptr)
        except Exception:
            pass


def synth_centroids(seed: int, nc: int, d: int) -> np.ndarray:
    out = np.empty((nc, d), np.float32)
    check(lib().laivg_synth_centroids(seed, nc, d, out.ctypes.data))
    return out


def synth_lists(seed: int, centroids: np.ndarray, per_list: int, spread: float,
                c_begin: int = 0, c_end: int | None = None, vecs=None, ids=None,
                threads: int = 0):
    centroids = _c(centroids, np.float32)
    nc, d = centroids.shape
    c_end = nc if c_end is None else c_end
    n = (c_end - c_begin) * per_list
    vecs = np.empty((n, d), np.float32) if vecs is None else vecs
    ids = np.empty(n, np.uint64) if ids is None else ids
    check(lib().laivg_synth_lists(seed, centroids.ctypes.data, nc, d, per_list, spread,
                                  c_begin, c_end, vecs.ctypes.data, ids.ctypes.data, threads))
    return vecs, ids


def synth_queries(seed: int, vecs: np.ndarray, nq: int, sigma: float):
    n, d = vecs.shape
    qi = np.empty((nq, d), np.float32)
    qo = np.empty((nq, d), np.float32)
    rows = np.empty(nq, np.uint64)
    check(lib().laivg_synth_queries(seed, vecs.ctypes.data, n, d, nq, sigma, qi.ctypes.data,
                                    qo.ctypes.data, rows.ctypes.data))
    return qi, qo, rows


def synth_queries_topical(seed: int, centroids: np.ndarray, vecs: np.ndarray, list_off,
                          nq: int, sigma: float, n_topics: int = 32, zipf_s: float = 1.0,
                          neigh: int = 16):
    """Topical (Zipf-skewed) q_in / q_out pairs: returns qi, qo, rows, topic."""
    cen = _c(centroids, np.float32)
    nc, d = cen.shape
    off = _c(list_off, np.uint64)
    qi = np.empty((nq, d), np.float32)
    qo = np.empty((nq, d), np.float32)
    rows = np.empty(nq, np.uint64)
    topic = np.empty(nq, np.uint32)
    check(lib().laivg_synth_queries_topical(seed, cen.ctypes.data, nc, vecs.ctypes.data,
                                            off.ctypes.data, d, n_topics, zipf_s, neigh, nq,
                                            sigma, qi.ctypes.data, qo.ctypes.data,
                                            rows.ctypes.data, topic.ctypes.data))
    return qi, qo, rows, topic


def group_microbatches_gpu(dev: Device, queries, m: int) -> list[MicroBatch]:
    """group_microbatches (sched.cpp:39-70) on the GPU; same batches."""
    Q = _c(queries, np.float32).reshape(-1, dev.ix.d)
    n = Q.shape[0]
    order = np.empty(max(n, 1), np.uint64)
    off = np.empty(n + 1, np.uint64)
    nb = C.c_uint32()
    check(lib().laivg_group_microbatches_gpu(dev.h, Q.ctypes.data, n, int(m), order.ctypes.data,
                                             off.ctypes.data, C.byref(nb)))
    return _batches_from_csr(order, off, nb.value)


def schedule(dev: Device, queries, m: int, L: int, resident):
    """The routing step of run_batch on the GPU: micro-batches of m
    (group_microbatches), each batch's probe-union overlap with every
    worker's resident set ([nw][nc] 0/1) as bitset popcounts, then the
    cache-aware greedy. Returns (batches, assignment, overlap[nb][nw])."""
    Q = _c(queries, np.float32).reshape(-1, dev.ix.d)
    n = Q.shape[0]
    res = np.ascontiguousarray(np.asarray(resident, np.uint8).reshape(-1, dev.ix.nc))
    nw = res.shape[0]
    order = np.empty(max(n, 1), np.uint64)
    off = np.empty(n + 1, np.uint64)
    nb = C.c_uint32()
    asg = np.empty(max(n, 1), np.uint32)
    ov = np.empty(max(n * nw, 1), np.uint64)
    check(lib().laivg_schedule(dev.h, Q.ctypes.data, n, int(m), int(L), res.ctypes.data, nw,
                               order.ctypes.data, off.ctypes.data, C.byref(nb), asg.ctypes.data,
                               ov.ctypes.data))
    k = nb.value
    return (_batches_from_csr(order, off, k), asg[:k].tolist(),
            ov[: k * nw].reshape(k, nw).copy())
