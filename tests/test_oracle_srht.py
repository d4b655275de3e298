"""Pins for the oracle's SRHT (Def) and radix-4 FWHT (Alg 3).

The FWHT is pinned to scipy.linalg.hadamard (the Sylvester construction of P:L168-171,
a library routine) by dense brute force, and to H_d H_d = d I and Parseval
||H a||^2 = d ||a||^2; the SRHT to the dense product k^-1/2 P H D A, to the exact
expectation E||Sx||^2 = ||x||^2 over the draws of D and P, and its draws to sign
balance and uniform sampling.
"""
import numpy as np
import pytest
import scipy.linalg
import scipy.stats

import oracle
import synth


@pytest.mark.parametrize("q", range(0, 11))
def test_fwht_matches_sylvester_hadamard(q):
    d = 1 << q
    a = np.random.default_rng(q).standard_normal(d)
    H = scipy.linalg.hadamard(d).astype(np.float64)
    got = oracle.fwht_rad4(a)
    assert np.allclose(got, H @ a, rtol=0, atol=1e-12 * max(1.0, np.abs(a).sum()))


@pytest.mark.parametrize("q", [3, 8, 13])
def test_fwht_involution_and_parseval(q):
    d = 1 << q
    a = np.random.default_rng(100 + q).standard_normal(d)
    h = oracle.fwht_rad4(a)
    assert abs(np.dot(h, h) - d * np.dot(a, a)) <= 1e-12 * d * np.dot(a, a)
    assert np.allclose(oracle.fwht_rad4(h), d * a, rtol=0, atol=1e-11 * d * np.abs(a).max())


def test_fwht_integer_exact():
    d = 1 << 9
    a = np.random.default_rng(5).integers(-8, 9, size=d).astype(np.float64)
    H = scipy.linalg.hadamard(d).astype(np.int64)
    assert np.array_equal(oracle.fwht_rad4(a), (H @ a.astype(np.int64)).astype(np.float64))


def test_srht_matches_dense_product():
    d, n, k = 256, 5, 24
    A = synth.gaussian_matrix(d, n, seed=3)
    b = synth.rhs(A, "hard", seed=3)
    D, p = oracle.srht_draws(d, k, seed=11)
    H = scipy.linalg.hadamard(d).astype(np.float64)
    P = np.zeros((k, d))
    P[np.arange(k), p] = 1.0
    S = (P @ H @ np.diag(D.astype(np.float64))) / np.sqrt(k)
    Y = oracle.srht_apply(A, k, seed=11, b=b)
    ref = S @ np.column_stack([A, b])
    assert np.allclose(Y, ref, rtol=0, atol=1e-12 * np.abs(ref).max())


def test_srht_draws_statistics():
    d, k = 1 << 16, 1 << 14
    D, p = oracle.srht_draws(d, k, seed=1)
    assert set(np.unique(D)) == {-1, 1}
    assert abs(D.astype(np.float64).mean()) < 5 / np.sqrt(d)
    assert p.min() >= 0 and p.max() < d
    counts = np.bincount(p >> 10, minlength=64)   # 64 equal bins
    _, pval = scipy.stats.chisquare(counts)
    assert pval > 1e-4


def test_srht_norm_expectation():
    # E||S x||^2 = (1/k) sum_j E (H D x)_{p_j}^2 = ||H D x||^2 / d = ||x||^2 (uniform p_j, H^T H = d I)
    d, k, trials = 128, 16, 400
    x = np.random.default_rng(2).standard_normal(d)
    vals = np.array([np.sum(oracle.srht_apply(x, k, seed=s) ** 2) for s in range(trials)])
    nx = np.dot(x, x)
    assert abs(vals.mean() - nx) <= 5 * vals.std() / np.sqrt(trials)


def test_srht_linearity_and_identity_rows():
    d, k = 64, 64
    rng = np.random.default_rng(9)
    A = rng.standard_normal((d, 3))
    Y = oracle.srht_apply(A, k, seed=4)
    Y2 = oracle.srht_apply(2.0 * A[:, :1] - A[:, 1:2], k, seed=4)
    assert np.allclose(Y2[:, 0], 2 * Y[:, 0] - Y[:, 1], atol=1e-12)
