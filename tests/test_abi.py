"""CPU-side checks of the product library: the C ABI loads and exports every
symbol include/laivg.h declares, host-only entry points match the reference
(golden fixtures / oracle), and the device path fails loudly without a GPU."""
import os
import re

import numpy as np
import pytest

from common import ROOT, golden, hybrid_d8_case, sha


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "laivg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(laivg_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported_and_bound():
    from paper_2502_20969_b200._lib import SIGNATURES, lib

    L = lib()
    syms = declared_symbols()
    assert len(syms) >= 55
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(SIGNATURES), set(syms) ^ set(SIGNATURES)
    assert L.laivg_version() >> 16 == 1


def test_library_is_in_tree_sm100a():
    from paper_2502_20969_b200._lib import LIB_PATH

    assert os.path.dirname(LIB_PATH) == os.path.join(ROOT, "paper_2502_20969_b200")
    data = open(LIB_PATH, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_split_budget_golden(laiv):
    g = golden("sched.npz")
    for i in range(len(g["split_total"])):
        n = int(g["split_n"][i])
        got = laiv.split_budget(int(g["split_total"][i]),
                                laiv.MicroBatch([int(x) for x in g["split_batch"][i, :n]]))
        assert got == [int(x) for x in g["split_out"][i, :n]]
    with pytest.raises(ValueError):
        laiv.split_budget(10, laiv.MicroBatch([]))


def test_group_microbatches_golden(orc, laiv):
    # acceptance.cpp:408-417: 256 x 768 queries in micro-batches of 4
    g = golden("sched.npz")
    q = orc.random_matrix(256, 768, 717)
    assert sha(q) == str(g["group_sha"])
    import time

    t0 = time.perf_counter()
    batches = laiv.group_microbatches(q, 4)
    assert time.perf_counter() - t0 < 0.1
    assert len(batches) == 64
    assert [x for b in batches for x in b.queries] == [int(x) for x in g["group_order"]]
    # test_sched.cpp:39-46 singletons for m = 1
    assert [b.queries for b in laiv.group_microbatches(q[:5], 1)] == [[0], [1], [2], [3], [4]]
    with pytest.raises(ValueError):
        laiv.group_microbatches(q, 0)


def test_group_microbatches_matches_oracle_random(orc, laiv):
    rng = np.random.default_rng(1)
    for t in range(5):
        q = rng.standard_normal((40, 16)).astype(np.float32)
        q[5] = q[9]  # exact duplicate -> distance tie broken by index
        m = int(rng.integers(1, 7))
        assert [b.queries for b in laiv.group_microbatches(q, m)] == orc.group_microbatches(q, m)


def test_group_microbatches_streaming_matches_reference(laiv):
    """n above the pair-matrix threshold (2048): per-seed rows, O(n) memory
    (ADVICE r01), bit-identical to the unmodified reference."""
    from oracle.oracle import RefLib

    if not RefLib.available():
        pytest.skip("oracle/_ref/libref.so not built")
    rng = np.random.default_rng(9)
    q = rng.standard_normal((3001, 24)).astype(np.float32)
    q[100:110] = q[7]  # exact distance ties: broken by index
    for m in (1, 4, 9):
        got = [b.queries for b in laiv.group_microbatches(q, m)]
        assert got == RefLib().group_microbatches(q, m)


def test_chunk_and_round_robin(laiv):
    assert [b.queries for b in laiv.chunk_microbatches(5, 2)] == [[0, 1], [2, 3], [4]]
    assert laiv.assign_round_robin(8, 3) == [b % 3 for b in range(8)]
    with pytest.raises(ValueError):
        laiv.assign_round_robin(3, 0)


def test_index_validation(laiv):
    cen = np.zeros((2, 4), np.float32)
    vecs = np.zeros((3, 4), np.float32)
    ids = np.array([0, 1, 2], np.uint64)
    off = np.array([0, 2, 3], np.uint64)
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.L2)
    assert ix.cluster_bytes(0) == 2 * (16 + 8) and ix.total_payload_bytes() == 3 * 24
    bad = vecs.copy()
    bad[1, 2] = np.nan
    with pytest.raises(ValueError):
        laiv.IvfIndex(cen, bad, ids, off, laiv.Metric.L2)
    with pytest.raises(ValueError):
        laiv.IvfIndex(cen, vecs, np.array([0, 1, 1], np.uint64), off, laiv.Metric.L2)
    with pytest.raises(ValueError):
        laiv.IvfIndex(cen, vecs, ids, np.array([0, 3, 2], np.uint64), laiv.Metric.L2)
    with pytest.raises(ValueError):
        laiv.IvfIndex(cen, vecs, ids, np.array([0, 3], np.uint64), laiv.Metric.L2)


def test_synth_is_deterministic_and_normalised(laiv):
    cen = laiv.synth_centroids(3, 16, 64)
    assert np.allclose(np.linalg.norm(cen, axis=1), 1.0, atol=1e-6)
    a, ia = laiv.synth_lists(3, cen, 20, 0.05, threads=1)
    b, ib = laiv.synth_lists(3, cen, 20, 0.05, threads=5)
    assert np.array_equal(a, b) and np.array_equal(ia, ib)
    part, _ = laiv.synth_lists(3, cen, 20, 0.05, c_begin=4, c_end=9)
    assert np.array_equal(part, a[4 * 20:9 * 20])
    assert list(ia[:3]) == [0, 1, 2] and int(ia[-1]) == 16 * 20 - 1
    qi, qo, rows = laiv.synth_queries(1, a, 8, 0.02)
    assert np.allclose(np.linalg.norm(qo, axis=1), 1.0, atol=1e-6)
    assert np.all(rows < a.shape[0])


def test_device_path_fails_loudly_without_gpu(orc, laiv):
    case, _, _ = hybrid_d8_case(orc, "l2")
    ix = laiv.IvfIndex(case.centroids, case.vecs, case.ids, case.list_off, laiv.Metric.L2)
    try:
        dev = laiv.Device(ix, 1 << 20)
    except laiv.CudaError:
        return  # CPU host: no silent fallback
    dev.close()
    pytest.skip("a GPU is present; covered by the -m gpu suite")
