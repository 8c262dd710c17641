"""Host-side plumbing of bench.py's multi-GPU runs (no GPU): per-rank core
slices are disjoint, cover the node's cores evenly, and emulated workers get
a W-way share of the host."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def affinity_of(rank, world):
    code = ("import json, os, sys; sys.path.insert(0, %r); import bench; "
            "bench.pin_rank_cores(%d, %d); print(json.dumps(sorted(os.sched_getaffinity(0))))"
            % (ROOT, rank, world))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         check=True, cwd=ROOT).stdout
    return json.loads(out.strip().splitlines()[-1])


def test_rank_core_slices_disjoint():
    cores = sorted(os.sched_getaffinity(0))
    for world in (1, 2, 4):
        if world > len(cores):
            continue
        slices = [affinity_of(r, world) for r in range(world)]
        if world == 1:
            assert slices[0] == cores
            continue
        seen = set()
        for sl in slices:
            assert len(sl) == len(cores) // world
            assert not (seen & set(sl))
            seen |= set(sl)
        assert seen <= set(cores)


def test_host_threads_split():
    sys.path.insert(0, ROOT)
    import bench

    n = os.cpu_count() or 1
    assert bench.host_threads(1) == n
    assert bench.host_threads(2) == max(1, n // 2)
    assert bench.host_threads(10 ** 6) == 1
