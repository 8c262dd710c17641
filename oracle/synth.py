"""ctypes binding of oracle/libsynth.so: the bench/test workload generator.

WORKLOAD GENERATION ONLY (SURVEY §8d planted clusters + queries). It is the
product's own generator source (paper_2502_20969_b200/csrc/synth.cpp) built
on its own, so bench.py's `--impl reference` arm draws the very datastore and
queries the GPU arm draws without loading liblaivg.so. Same signatures as the
``laiv.synth_*`` functions; tests/test_synth.py checks both bit for bit.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PATH = os.path.join(HERE, "libsynth.so")
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(PATH):
            import subprocess

            subprocess.check_call(["make", "-s", "-C", HERE, "synth"])
        L = C.CDLL(PATH)
        u32, u64, vp = C.c_uint32, C.c_uint64, C.c_void_p
        L.lsynth_last_error.restype = C.c_char_p
        L.lsynth_centroids.argtypes = [u64, u32, u32, vp]
        L.lsynth_lists.argtypes = [u64, vp, u32, u32, u64, C.c_float, u32, u32, vp, vp, C.c_int]
        L.lsynth_queries.argtypes = [u64, vp, u64, u32, u32, C.c_float, vp, vp, vp]
        L.lsynth_queries_topical.argtypes = [u64, vp, u32, vp, vp, u32, u32, C.c_double, u32,
                                             u32, C.c_float, vp, vp, vp, vp]
        _LIB = L
    return _LIB


def _check(rc: int) -> None:
    if rc != 0:
        raise ValueError(_lib().lsynth_last_error().decode())


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def synth_centroids(seed: int, nc: int, d: int) -> np.ndarray:
    out = np.empty((nc, d), np.float32)
    _check(_lib().lsynth_centroids(seed, nc, d, out.ctypes.data))
    return out


def synth_lists(seed: int, centroids, per_list: int, spread: float, c_begin: int = 0,
                c_end: int | None = None, vecs=None, ids=None, threads: int = 0):
    centroids = _c(centroids, np.float32)
    nc, d = centroids.shape
    c_end = nc if c_end is None else c_end
    n = (c_end - c_begin) * per_list
    vecs = np.empty((n, d), np.float32) if vecs is None else vecs
    ids = np.empty(n, np.uint64) if ids is None else ids
    _check(_lib().lsynth_lists(seed, centroids.ctypes.data, nc, d, per_list, spread, c_begin,
                               c_end, vecs.ctypes.data, ids.ctypes.data, threads))
    return vecs, ids


def synth_queries(seed: int, vecs, nq: int, sigma: float):
    n, d = vecs.shape
    qi = np.empty((nq, d), np.float32)
    qo = np.empty((nq, d), np.float32)
    rows = np.empty(nq, np.uint64)
    _check(_lib().lsynth_queries(seed, vecs.ctypes.data, n, d, nq, sigma, qi.ctypes.data,
                                 qo.ctypes.data, rows.ctypes.data))
    return qi, qo, rows


def synth_queries_topical(seed: int, centroids, vecs, list_off, nq: int, sigma: float,
                          n_topics: int = 32, zipf_s: float = 1.0, neigh: int = 16):
    cen = _c(centroids, np.float32)
    nc, d = cen.shape
    off = _c(list_off, np.uint64)
    qi = np.empty((nq, d), np.float32)
    qo = np.empty((nq, d), np.float32)
    rows = np.empty(nq, np.uint64)
    topic = np.empty(nq, np.uint32)
    _check(_lib().lsynth_queries_topical(seed, cen.ctypes.data, nc, vecs.ctypes.data,
                                         off.ctypes.data, d, n_topics, zipf_s, neigh, nq, sigma,
                                         qi.ctypes.data, qo.ctypes.data, rows.ctypes.data,
                                         topic.ctypes.data))
    return qi, qo, rows, topic
