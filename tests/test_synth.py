"""The bench's reference arm draws its workload from oracle/libsynth.so (the
product's synth.cpp built alone, no liblaivg.so loaded): it must produce the
very bytes the product's laivg_synth_* produce."""
import numpy as np


def test_standalone_generator_bit_identical(laiv):
    from oracle import synth

    cen_a = laiv.synth_centroids(3, 24, 96)
    cen_b = synth.synth_centroids(3, 24, 96)
    assert np.array_equal(cen_a, cen_b)
    va, ia = laiv.synth_lists(3, cen_a, 50, 0.05, threads=3)
    vb, ib = synth.synth_lists(3, cen_b, 50, 0.05, threads=5)
    assert np.array_equal(va, vb) and np.array_equal(ia, ib)
    qa = laiv.synth_queries(9, va, 40, 0.01)
    qb = synth.synth_queries(9, vb, 40, 0.01)
    for x, y in zip(qa, qb):
        assert np.array_equal(x, y)
    off = np.arange(0, 24 * 50 + 1, 50, dtype=np.uint64)
    ta = laiv.synth_queries_topical(4, cen_a, va, off, 30, 0.01, 6, 1.0, 4)
    tb = synth.synth_queries_topical(4, cen_b, vb, off, 30, 0.01, 6, 1.0, 4)
    for x, y in zip(ta, tb):
        assert np.array_equal(x, y)
