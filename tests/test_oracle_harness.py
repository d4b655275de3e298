"""The block-parallel harness over the oracle (oracle/harness.py) returns exactly what one oracle call
returns: the CountSketch and G-stage are column-separable and the codes are a function of the global
row (R3), so blocking changes no operation and no order."""
import numpy as np

import oracle
from oracle import harness
import synth


def test_codes_blocks_identical():
    for d, row0 in [(100003, 0), (77, 5), (50000, (1 << 33) + 1)]:
        h, s = oracle.codes(d, 8192, 3, row0)
        hb, sb = harness.codes(d, 8192, 3, row0, threads=5)
        assert np.array_equal(h, hb) and np.array_equal(s, sb)


def test_cs_apply_and_gemm_blocks_bit_identical():
    d, n, k1, k2 = 20011, 13, 512, 26
    A = synth.gaussian_matrix(d, n, seed=4)
    b = synth.rhs(A, "hard", seed=4)
    h, s = oracle.codes(d, k1, 2)
    SA, T = oracle.cs_apply(h, s, A, k1, b=b, with_abs=True)
    for threads in (1, 3, 8, 40):
        SAb, Tb = harness.cs_apply(h, s, A, k1, b=b, with_abs=True, threads=threads)
        assert np.array_equal(SA, SAb) and np.array_equal(T, Tb)
    G = oracle.gauss(k2, k1, 2)
    Z, Zabs = oracle.gemm_comp(G, SA, T)
    Zb, Zabsb = harness.gemm(G, SA, T, threads=4)
    assert np.array_equal(Z, Zb) and np.array_equal(Zabs, Zabsb)


def test_ms_lstsq_blocks_identical():
    d, n = 1 << 14, 8
    A = synth.ill_conditioned(d, n, 1e4, seed=3)
    b = synth.rhs(A, "easy", seed=3)
    x, r = oracle.ms_lstsq(A, b, 2 * n * n, 2 * n, 1)
    xb, rb = harness.ms_lstsq(A, b, 2 * n * n, 2 * n, 1, threads=3)
    assert np.array_equal(x, xb) and r == rb


def test_fp32_and_b_only():
    d, k1 = 5000, 64
    h, s = oracle.codes(d, k1, 9)
    A = synth.gaussian_matrix(d, 5, seed=1, dtype=np.float32)
    assert np.array_equal(oracle.cs_apply(h, s, A, k1), harness.cs_apply(h, s, A, k1, threads=3))
    b = synth.gaussian_matrix(d, 1, seed=2)[:, 0]
    assert np.array_equal(oracle.cs_apply(h, s, np.zeros((d, 0)), k1, b=b),
                          harness.cs_apply(h, s, np.zeros((d, 0)), k1, b=b, threads=2))
