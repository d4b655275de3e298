"""Pins for the oracle's rand_cholQR least squares (Alg 5).

rand_cholQR computes the TRUE least-squares solution (no sketch distortion), so
the oracle is pinned to numpy.linalg.lstsq on A itself (a library QR solve), to the
QR factor of A (R^T R = A^T A, |R| = |qr(A).R| up to row signs), to the identity-sketch
special case (Y = A: R0 is A's own R, Q0 = Q, G = I, R1 = I), and to its stability
claim at kappa = 1e10, where the normal equations break down (Fig 8 setup).
"""
import numpy as np
import pytest
import scipy.linalg

import oracle
import synth


def _sketch(A, k1, k2, seed):
    return oracle.ms_apply(A, k1, k2, seed)


@pytest.mark.parametrize("kappa", [1.0, 1e2, 1e6])
@pytest.mark.parametrize("mode", ["easy", "hard"])
def test_matches_library_lstsq(kappa, mode):
    d, n = 3000, 8
    A = synth.ill_conditioned(d, n, kappa, seed=4)
    b = synth.rhs(A, mode, seed=4)
    x = oracle.rand_cholqr_lstsq(A, b, _sketch(A, 2 * n * n, 2 * n, seed=7))
    xs, *_ = np.linalg.lstsq(A, b, rcond=None)
    nb = np.linalg.norm(b)
    r = np.linalg.norm(b - A @ xs)
    # fitted values agree within the perturbation bound of backward-stable LS solvers,
    # ||delta(A x)|| <~ u (||b|| + kappa ||r||) (Wedin; Higham, Accuracy and Stability, ch. 20)
    assert np.linalg.norm(A @ (x - xs)) <= 10 * n * 2.2e-16 * (nb + kappa * r)
    # forward error within the LS perturbation bound ~ kappa u (1 + kappa ||r|| / (||A|| ||x||))
    bound = 50 * 2.2e-16 * kappa * (1 + kappa * r / (np.linalg.norm(A, 2) * np.linalg.norm(xs)))
    assert np.linalg.norm(x - xs) <= bound * np.linalg.norm(xs) + 1e-300


def test_R_is_the_qr_factor_of_A():
    d, n = 2000, 12
    A = synth.ill_conditioned(d, n, 1e2, seed=5)
    b = synth.rhs(A, "easy", seed=5)
    _, R = oracle.rand_cholqr_lstsq(A, b, _sketch(A, 2 * n * n, 2 * n, seed=3), return_R=True)
    assert np.all(np.tril(R, -1) == 0)
    AtA = A.T @ A
    assert np.abs(R.T @ R - AtA).max() <= 1e-12 * np.abs(AtA).max()
    Rn = np.linalg.qr(A, mode="r")
    assert np.allclose(np.abs(R), np.abs(Rn), rtol=1e-10, atol=1e-12 * np.abs(Rn).max())
    # Q = A R^-1 is orthonormal (Alg 4's output)
    Q = scipy.linalg.solve_triangular(R, A.T, trans="T", lower=False).T
    assert np.abs(Q.T @ Q - np.eye(n)).max() <= 1e-12


def test_identity_sketch_reduces_to_qr_lstsq():
    # Y = A: R0 = R(A), Q0 = A R0^-1 = Q, G = I, R1 = I, R = R0 -> x = R^-1 Q^T b
    d, n = 500, 6
    A = synth.gaussian_matrix(d, n, seed=6)
    b = synth.rhs(A, "hard", seed=6)
    x, R = oracle.rand_cholqr_lstsq(A, b, A, return_R=True)
    R0 = oracle.householder_qr(A)
    assert np.allclose(R, R0, rtol=1e-13, atol=1e-13 * np.abs(R0).max())
    xq, _ = oracle.sketch_solve(np.column_stack([A, b]), n)
    assert np.allclose(x, xq, rtol=1e-12, atol=1e-14)


def test_stable_where_normal_equations_fail():
    # stable for kappa(A) < u^-1; NE only for kappa < u^-1/2 (fail past ~1e8)
    d, n = 1 << 14, 16
    A = synth.ill_conditioned(d, n, 1e10, seed=3)
    b = synth.rhs(A, "consistent", seed=3)
    nb = np.linalg.norm(b)
    x = oracle.rand_cholqr_lstsq(A, b, _sketch(A, 2 * n * n, 2 * n, seed=1))
    xs, *_ = np.linalg.lstsq(A, b, rcond=None)
    r_rc = oracle.residual_norm(A, b, x) / nb
    r_qr = oracle.residual_norm(A, b, xs) / nb
    assert r_rc <= max(100 * r_qr, 1e-13), (r_rc, r_qr)
    try:
        r_ne = oracle.residual_norm(A, b, oracle.normal_eq(A, b)) / nb
    except oracle.OracleError as e:
        assert e.status == oracle.ENOTPD
    else:
        assert r_ne > 1e3 * r_rc


def test_singular_sketch():
    d, n = 200, 4
    A = synth.gaussian_matrix(d, n, seed=1)
    A[:, 2] = A[:, 1]
    with pytest.raises(oracle.OracleError) as e:
        oracle.rand_cholqr_lstsq(A, np.ones(d), _sketch(A, 32, 8, seed=1))
    assert e.value.status == oracle.ESINGULAR
