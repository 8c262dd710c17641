"""N > 1 path on CPU: two gloo ranks shard queries, all-gather their resident
sets, route micro-batches with the cache-aware greedy, and reduce timings with
max — the same host logic bench.py runs under torchrun on B200s. The routing
is checked against the oracle's assign_cache_aware (sched.cpp:87-144)."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from oracle.oracle import L2, Oracle
    from paper_2502_20969_b200 import laiv, shard

    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        orc = Oracle()
        nc, d, nq, L = 64, 8, 24, 4
        cen = orc.random_matrix(nc, d, 5)
        queries = orc.random_matrix(nq, d, 6)
        probes = np.array([orc.coarse_probe(cen, L2, qv, L) for qv in queries])
        batches = laiv.group_microbatches(queries, 4)
        rng = np.random.default_rng(100 + rank)  # each rank's own cache
        mine = (rng.random(nc) < 0.3).astype(np.uint8)
        resident = shard.gather_resident(mine)
        assign = shard.route(batches, probes, resident)
        want = orc.assign_cache_aware([b.queries for b in batches], resident, cen, L2, queries, L)
        idx = shard.shard_indices(nq, rank, world)
        mx = shard.max_over_ranks([rank + 0.5, -rank])
        # every rank must agree on the routing
        import torch

        t = torch.tensor(assign, dtype=torch.int64)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        agree = all(bool((p == t).all()) for p in parts)
        q.put((rank, assign, list(want), idx.tolist(), mx, agree, resident[rank].tolist(),
               mine.tolist()))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", repr(e)))


def test_two_rank_routing_and_sharding():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    out = sorted(out)
    for o in out:
        assert o[1] != "error", o
    (_, a0, w0, i0, m0, g0, r0, mine0), (_, a1, w1, i1, m1, g1, r1, mine1) = out
    assert g0 and g1 and a0 == a1 == w0 == w1       # same routing everywhere = oracle
    assert r0 == mine0 and r1 == mine1              # all_gather placed each rank's set
    assert sorted(i0 + i1) == list(range(24)) and not set(i0) & set(i1)
    assert m0 == m1 == [1.5, 0.0]
    loads = np.bincount(a0, minlength=2)
    assert loads.max() <= (len(a0) + 1) // 2        # cap = ceil(nb / nw)


def test_overlap_matrix_and_greedy_known_answers():
    from paper_2502_20969_b200 import laiv, shard

    # disjoint caches route to the matching worker (test_sched.cpp:140-176)
    probes = np.array([[0, 1], [2, 3]])
    batches = [laiv.MicroBatch([0]), laiv.MicroBatch([1])]
    resident = np.zeros((2, 4), np.uint8)
    resident[0, [2, 3]] = 1
    resident[1, [0, 1]] = 1
    assert shard.route(batches, probes, resident) == [1, 0]
    # empty caches degenerate to round robin (test_sched.cpp:178-188)
    b8 = [laiv.MicroBatch([i]) for i in range(8)]
    assert shard.route(b8, np.zeros((8, 2), int), np.zeros((3, 4), np.uint8)) == [
        i % 3 for i in range(8)]
    with pytest.raises(ValueError):
        laiv.greedy_assign(np.zeros((2, 0), np.uint64))
