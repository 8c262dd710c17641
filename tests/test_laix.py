"""LAIX index files: load_index / save_index (ivf.hpp:95-98,
ivf.cpp:351-458) through laivg_index_load / laivg_index_save.

Pinned to the reference: tests/golden/laix/ holds files written by the
reference's save_index and, for 140+ byte-level corruptions of one of them,
the exception class and message the reference's load_index throws (and the
store it loads when it does not). Host-only: no GPU needed.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2502_20969_b200 import laiv
from paper_2502_20969_b200._lib import LogicError

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "laix")
KIND = {1: RuntimeError, 2: ValueError, 3: LogicError}


def apply_ops(data: bytes, ops) -> bytes:  # the generator's byte edits
    b = bytearray(data)
    for op in ops:
        if op[0] == "truncate":
            del b[op[1]:]
        elif op[0] == "patch":
            b[op[1]:op[1] + len(op[2]) // 2] = bytes.fromhex(op[2])
        elif op[0] == "append":
            b += bytes.fromhex(op[1])
        elif op[0] == "replace":
            b = bytearray(bytes.fromhex(op[1]))
    return bytes(b)


def store_sha(ix):
    vecs, ids = ix.store()
    return hashlib.sha256(np.concatenate([ix.list_off.view(np.uint8), ids.view(np.uint8),
                                          vecs.reshape(-1).view(np.uint8)]).tobytes()).hexdigest()


def test_load_matches_reference_arrays():
    a = np.load(os.path.join(G, "a_ip_arrays.npz"))
    ix = laiv.load_index(os.path.join(G, "a_ip.laix"))
    assert ix.nc == 12 and ix.d == 6 and ix.metric == laiv.Metric.InnerProduct
    vecs, ids = ix.store()
    assert np.array_equal(ix.centroids, a["centroids"])
    assert np.array_equal(ix.list_off, a["list_off"])
    assert np.array_equal(ids, a["ids"])
    assert np.array_equal(vecs, a["vecs"])
    assert ix.total_payload_bytes() == 150 * (4 * 6 + 8)


@pytest.mark.parametrize("name", ["a_ip.laix", "b_l2_empty.laix"])
@pytest.mark.parametrize("threads", [1, 3, 0])
def test_round_trip_is_byte_exact(tmp_path, name, threads):
    # test_ivf.cpp:331-351: load then save reproduces the reference's bytes
    src = os.path.join(G, name)
    ix = laiv.load_index(src, threads)
    out = tmp_path / "x.laix"
    laiv.save_index(out, ix, threads)
    assert out.read_bytes() == open(src, "rb").read()


def test_save_from_arrays_matches_reference_bytes(tmp_path):
    a = np.load(os.path.join(G, "a_ip_arrays.npz"))
    ix = laiv.IvfIndex(a["centroids"], a["vecs"], a["ids"], a["list_off"],
                       laiv.Metric.InnerProduct)
    ix.save(tmp_path / "y.laix")
    assert (tmp_path / "y.laix").read_bytes() == open(os.path.join(G, "a_ip.laix"), "rb").read()


def test_empty_lists_file():
    ix = laiv.load_index(os.path.join(G, "b_l2_empty.laix"))
    assert ix.metric == laiv.Metric.L2
    assert ix.list_len(2) == 0 and ix.list_len(5) == 0
    assert int(ix.list_off[-1]) == 64


with open(os.path.join(G, "laix_cases.json")) as _f:
    CASES = json.load(_f)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_corruptions_match_reference(tmp_path, case):
    data = open(os.path.join(G, "a_ip.laix"), "rb").read()
    path = tmp_path / "case.laix"
    path.write_bytes(apply_ops(data, case["ops"]))
    if case["kind"] == 0:
        ix = laiv.load_index(path, 2)
        assert store_sha(ix) == case["store_sha"]
        return
    with pytest.raises(KIND[case["kind"]]) as e:
        laiv.load_index(path, 2)
    assert str(e.value) == case["msg"].replace("{path}", str(path))


def test_missing_file_and_unwritable_path(tmp_path):
    with pytest.raises(RuntimeError, match="cannot open: "):
        laiv.load_index(tmp_path / "nope.laix")
    ix = laiv.load_index(os.path.join(G, "a_ip.laix"))
    with pytest.raises(RuntimeError, match="cannot open for writing: "):
        ix.save(tmp_path / "no" / "dir" / "x.laix")


def test_large_store_round_trip_and_first_error_order(tmp_path):
    # many lists larger than one 16 MB read task, 16 threads; then the first
    # invalid row in file order wins over later ones
    rng = np.random.default_rng(3)
    nc, d = 9, 512
    lens = [0, 9000, 1, 12000, 0, 3, 8300, 2, 40]
    off = np.cumsum([0] + lens).astype(np.uint64)
    n = int(off[-1])
    vecs = rng.standard_normal((n, d)).astype(np.float32)
    ids = rng.permutation(np.arange(n, dtype=np.uint64) * 5 + 11)
    cen = rng.standard_normal((nc, d)).astype(np.float32)
    ix = laiv.IvfIndex(cen, vecs, ids, off, laiv.Metric.L2)
    p = tmp_path / "big.laix"
    ix.save(p, 16)
    back = laiv.load_index(p, 16)
    v2, i2 = back.store()
    assert np.array_equal(v2, vecs) and np.array_equal(i2, ids)
    assert np.array_equal(back.centroids, cen) and np.array_equal(back.list_off, off)
    # the constructor applies the same rule: a duplicate at row 20000 comes
    # before a NaN at row 25000, a NaN at row 100 before both
    bad = ids.copy()
    bad[20000] = bad[5]
    v = vecs.copy()
    v[25000, 7] = np.nan
    with pytest.raises(ValueError, match=f"^duplicate id {int(bad[5])}$"):
        laiv.IvfIndex(cen, v, bad, off, laiv.Metric.L2)
    v[100, 0] = np.inf
    with pytest.raises(ValueError, match=f"^non-finite component in row for id {int(bad[100])}$"):
        laiv.IvfIndex(cen, v, bad, off, laiv.Metric.L2)
