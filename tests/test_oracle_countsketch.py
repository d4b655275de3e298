"""Pins for the oracle's CountSketch apply (Eq 2 / Alg 2).

Each check is fixed by the paper or by mathematics, not by the oracle itself:
the SPEC worked example, dense brute force densify(S) @ A (numpy),
the k1 = 1 closed forms, the identity plan, exact integer sums, linearity,
the partition identity, and E||Sx||^2 = ||x||^2 with its closed-form
variance (2/k1)(||x||_2^4 - ||x||_4^4).
"""
import math
import os

import numpy as np
import pytest

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def densify(h, s, k1):
    """Explicit k1 x d CountSketch: column j is s_j e_{h_j} (Def 3)."""
    d = len(h)
    S = np.zeros((k1, d))
    S[h, np.arange(d)] = s
    return S


def test_spec_worked_example():
    vals = {}
    with open(os.path.join(GOLDEN, "countsketch_worked_example.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                k, *v = line.split()
                vals[k] = [float(t) for t in v]
    h = np.array(vals["r"], np.int32)
    s = np.array(vals["s"], np.int8)
    A = np.array(vals["A"])[:, None]
    Y = oracle.cs_apply(h, s, A, int(vals["k"][0]))
    assert np.array_equal(Y[:, 0], np.array(vals["Y"]))


@pytest.mark.parametrize("d,n,k1,seed", [(1, 1, 1, 1), (17, 3, 5, 2), (256, 4, 16, 3), (4096, 8, 64, 1), (1000, 5, 997, 4)])
def test_matches_dense_bruteforce(d, n, k1, seed):
    h, s = oracle.codes(d, k1, seed)
    A = synth.gaussian_matrix(d, n, seed=seed)
    SA, T = oracle.cs_apply(h, s, A, k1, with_abs=True)
    dense = densify(h, s, k1) @ A
    # numpy's matmul is itself rounded: bound by 2 d u sum|terms|
    assert np.all(np.abs(SA - dense) <= 4 * d * 1.2e-16 * T + 1e-300)
    assert np.allclose(T, np.abs(densify(h, s, k1)) @ np.abs(A), rtol=1e-13, atol=0)


def test_fp32_input_widened():
    d, n, k1 = 3000, 4, 32
    h, s = oracle.codes(d, k1, 6)
    A32 = synth.gaussian_matrix(d, n, seed=6, dtype=np.float32)
    SA, T = oracle.cs_apply(h, s, A32, k1, with_abs=True)
    dense = densify(h, s, k1) @ A32.astype(np.float64)
    assert np.all(np.abs(SA - dense) <= 4 * d * 1.2e-16 * T)


def test_k1_one_all_plus_is_column_sums():
    d, n = 5000, 6
    A = synth.gaussian_matrix(d, n, seed=3)
    h = np.zeros(d, np.int32)
    s = np.ones(d, np.int8)
    SA = oracle.cs_apply(h, s, A, 1)
    for c in range(n):
        exact = math.fsum(A[:, c])              # correctly rounded sum
        assert abs(SA[0, c] - exact) <= 2.3e-16 * abs(exact) + 1e-30 * d


def test_k1_one_hashed_signs_is_signed_sum():
    d, n = 4000, 3
    A = synth.gaussian_matrix(d, n, seed=4)
    h, s = oracle.codes(d, 1, seed=4)
    assert np.all(h == 0)
    SA = oracle.cs_apply(h, s, A, 1)
    for c in range(n):
        assert abs(SA[0, c] - math.fsum(s * A[:, c])) <= 1e-15 * np.abs(A[:, c]).sum()


def test_identity_plan_returns_A():
    d, n = 300, 4
    A = synth.gaussian_matrix(d, n, seed=5)
    SA = oracle.cs_apply(np.arange(d, dtype=np.int32), np.ones(d, np.int8), A, d)
    assert np.array_equal(SA, A)


def test_signed_permutation_plan():
    d, n = 64, 3
    A = synth.gaussian_matrix(d, n, seed=6)
    rng = np.random.default_rng(0)
    perm = rng.permutation(d).astype(np.int32)
    sg = rng.choice([-1, 1], d).astype(np.int8)
    SA = oracle.cs_apply(perm, sg, A, d)
    expect = np.zeros_like(A)
    expect[perm] = sg[:, None] * A
    assert np.array_equal(SA, expect)


def test_integer_matrix_exact():
    d, n, k1 = 20000, 5, 64
    A = synth.integer_matrix(d, n, seed=2, lo=-(1 << 20), hi=1 << 20)
    h, s = oracle.codes(d, k1, 1)
    SA = oracle.cs_apply(h, s, A, k1)
    exact = np.zeros((k1, n), np.int64)
    np.add.at(exact, h, s[:, None].astype(np.int64) * A.astype(np.int64))
    assert np.array_equal(SA, exact.astype(np.float64))


def test_single_nonzero_row():
    d, n, k1 = 1000, 3, 50
    A = np.zeros((d, n), order="F")
    A[417] = [1.5, -2.25, 3e-300]
    h, s = oracle.codes(d, k1, 8)
    SA = oracle.cs_apply(h, s, A, k1)
    expect = np.zeros((k1, n))
    expect[h[417]] = s[417] * A[417]
    assert np.array_equal(SA, expect)


def test_augmented_b_column_is_Sb():
    d, n, k1 = 2000, 3, 40
    A = synth.gaussian_matrix(d, n, seed=1)
    b = synth.rhs(A, "hard", seed=1)
    h, s = oracle.codes(d, k1, 2)
    SAb = oracle.cs_apply(h, s, A, k1, b=b)
    assert SAb.shape == (k1, n + 1)
    assert np.array_equal(SAb[:, :n], oracle.cs_apply(h, s, A, k1))
    assert np.array_equal(SAb[:, n], oracle.cs_apply(h, s, b[:, None], k1)[:, 0])


def test_linearity():
    d, n, k1 = 3000, 4, 128
    A = synth.gaussian_matrix(d, n, seed=1)
    B = synth.gaussian_matrix(d, n, seed=2)
    h, s = oracle.codes(d, k1, 3)
    lhs, T = oracle.cs_apply(h, s, 2.5 * A - 0.5 * B, k1, with_abs=True)
    rhs_ = 2.5 * oracle.cs_apply(h, s, A, k1) - 0.5 * oracle.cs_apply(h, s, B, k1)
    assert np.all(np.abs(lhs - rhs_) <= 1e-14 * (T + 1))


def test_partition_identity():
    # CA = sum_i C^(i) A^(i), C^(i) the slice of rows of block i
    d, n, k1 = 7001, 3, 256
    A = synth.integer_matrix(d, n, seed=3)
    h, s = oracle.codes(d, k1, 4)
    full = oracle.cs_apply(h, s, A, k1)
    for p in (1, 2, 4, 7):
        bounds = np.linspace(0, d, p + 1).astype(int)
        acc = np.zeros_like(full)
        for g in range(p):
            r0, r1 = bounds[g], bounds[g + 1]
            hg, sg = oracle.codes(r1 - r0, k1, 4, row0=r0)
            acc += oracle.cs_apply(hg, sg, np.asfortranarray(A[r0:r1]), k1)
        assert np.array_equal(acc, full)


def test_empty_buckets_exact_zero():
    d, n, k1 = 10, 2, 1000
    h, s = oracle.codes(d, k1, 1)
    SA = oracle.cs_apply(h, s, synth.gaussian_matrix(d, n), k1)
    empty = np.setdiff1d(np.arange(k1), h)
    assert np.all(SA[empty] == 0.0)


def test_norm_preserved_in_expectation():
    # E||Sx||^2 = ||x||^2, Var = (2/k1)(||x||_2^4 - ||x||_4^4) (derivation in DESIGN.md)
    d, k1, trials = 256, 16, 600
    x = synth.gaussian_matrix(d, 1, seed=9)[:, 0]
    vals = []
    for t in range(trials):
        h, s = oracle.codes(d, k1, seed=1000 + t)
        vals.append(float(np.sum(oracle.cs_apply(h, s, x[:, None], k1) ** 2)))
    vals = np.array(vals)
    n2, n4 = np.sum(x ** 2), np.sum(x ** 4)
    var = 2.0 / k1 * (n2 ** 2 - n4)
    assert abs(vals.mean() - n2) <= 5 * math.sqrt(var / trials)
    # sample variance within 25% of the closed form (600 samples)
    assert abs(vals.var() / var - 1.0) < 0.25


def test_bad_bucket_rejected():
    with pytest.raises(oracle.OracleError):
        oracle.cs_apply(np.array([0, 5], np.int32), np.ones(2, np.int8), np.ones((2, 1)), 3)
