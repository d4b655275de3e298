"""Pins for the oracle's least-squares layer.

Householder QR against numpy.linalg.qr (library); the sketched solve against
numpy.linalg.lstsq on the same sketch (library); the identity sketch against
plain QR least squares; the distortion chain of P:L107-111 with the
embedding constant measured per instance (Reading R8); the normal equations
against scipy.linalg.cho_solve (library) and their breakdown past
kappa ~ 1e8 (Fig 8 setup d = 2^17, n = 16, b = Ae).
"""
import numpy as np
import pytest
import scipy.linalg

import oracle
import synth


def test_householder_matches_numpy_qr():
    rng = np.random.default_rng(3)
    for m, nc in [(1, 1), (5, 5), (64, 8), (256, 129)]:
        W = rng.standard_normal((m, nc))
        R = oracle.householder_qr(W)
        Rn = np.linalg.qr(W, mode="r")
        assert np.allclose(np.abs(R), np.abs(Rn), rtol=1e-12, atol=1e-12 * np.abs(Rn).max())
        assert np.allclose(R.T @ R, W.T @ W, rtol=0, atol=1e-12 * np.abs(W.T @ W).max())
        assert np.all(np.tril(R, -1) == 0)


def test_householder_hand_cases():
    # A = [[3],[4]] -> R = [[5]] up to sign
    R = oracle.householder_qr(np.array([[3.0], [4.0]]))
    assert abs(abs(R[0, 0]) - 5.0) < 1e-15


def test_sketch_solve_matches_lstsq():
    rng = np.random.default_rng(4)
    m, n = 40, 7
    Z = rng.standard_normal((m, n + 1))
    x, r = oracle.sketch_solve(Z, n)
    xs, res, *_ = np.linalg.lstsq(Z[:, :n], Z[:, n], rcond=None)
    assert np.allclose(x, xs, rtol=1e-12, atol=1e-12)
    assert abs(r - np.sqrt(res[0])) < 1e-12 * np.linalg.norm(Z[:, n])


def test_sketch_solve_singular():
    Z = np.zeros((10, 4))
    Z[:, 0] = 1.0
    Z[:, 3] = 1.0
    with pytest.raises(oracle.OracleError) as e:
        oracle.sketch_solve(Z, 3)
    assert e.value.status == oracle.ESINGULAR


def test_identity_sketch_is_qr_lstsq():
    # S = I degenerates Alg 1 to the QR-based true least squares
    d, n = 200, 5
    A = synth.gaussian_matrix(d, n, seed=2)
    b = synth.rhs(A, "hard", seed=2)
    SAb = oracle.cs_apply(np.arange(d, dtype=np.int32), np.ones(d, np.int8), A, d, b=b)
    x, r = oracle.sketch_solve(SAb, n)
    xs, res, *_ = np.linalg.lstsq(A, b, rcond=None)
    assert np.allclose(x, xs, rtol=1e-12, atol=1e-13)
    assert abs(r - oracle.residual_norm(A, b, x)) < 1e-11 * r


def _qr_basis(A, b):
    Q, _ = np.linalg.qr(np.column_stack([A, b]))
    return Q


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("mode", ["easy", "hard"])
@pytest.mark.parametrize("k2_per_n", [2, 16])
def test_distortion_chain(seed, mode, k2_per_n):
    # ||b-Ax_t|| <= ||b-Ax_s|| <= sqrt((1+eps)/(1-eps)) ||b-Ax_t||
    # with the embedding measured on span([A b]) (Reading R8): singular values
    # smin <= smax of S Q give the same chain with factor smax/smin, and
    # eps = max(smax^2-1, 1-smin^2) gives the paper's form when eps < 1.
    d, n = 4096, 8
    k1, k2 = 2 * n * n, k2_per_n * n
    A = synth.ill_conditioned(d, n, 1e2, seed=seed)
    b = synth.rhs(A, mode, seed=seed)
    x, _ = oracle.ms_lstsq(A, b, k1, k2, seed=100 + seed)
    r_s = oracle.residual_norm(A, b, x)
    xt, *_ = np.linalg.lstsq(A, b, rcond=None)
    r_t = oracle.residual_norm(A, b, xt)
    SQ = oracle.ms_apply(_qr_basis(A, b), k1, k2, seed=100 + seed)
    sv = np.linalg.svd(SQ, compute_uv=False)
    assert r_t <= r_s * (1 + 1e-12)
    assert r_s <= sv[0] / sv[-1] * r_t * (1 + 1e-10)
    eps = max(sv[0] ** 2 - 1, 1 - sv[-1] ** 2)
    if eps < 1:
        assert r_s <= np.sqrt((1 + eps) / (1 - eps)) * r_t * (1 + 1e-10)


def test_normal_eq_matches_cho_solve():
    d, n = 3000, 6
    A = synth.ill_conditioned(d, n, 1e2, seed=1)
    b = synth.rhs(A, "easy", seed=1)
    x = oracle.normal_eq(A, b)
    xs = scipy.linalg.cho_solve(scipy.linalg.cho_factor(A.T @ A), A.T @ b)
    assert np.allclose(x, xs, rtol=1e-11, atol=0)
    # kappa = 1e2 normal equations agree with QR least squares
    xq, *_ = np.linalg.lstsq(A, b, rcond=None)
    assert np.linalg.norm(x - xq) <= 1e-10 * np.linalg.norm(xq)


def test_normal_eq_not_pd():
    # A^T A = [[1 + 1e-18, 1], [1, 1]] rounds to the singular [[1,1],[1,1]]:
    # the second Cholesky pivot is exactly 0 (S:L69 NotPositiveDefinite)
    A = np.asfortranarray(np.array([[1.0, 1.0], [1e-9, 0.0]]))
    with pytest.raises(oracle.OracleError) as e:
        oracle.normal_eq(A, np.ones(2))
    assert e.value.status == oracle.ENOTPD


def test_kappa_sweep_fig8():
    # Fig 8: d = 2^17, n = 16, b = Ae; NE fails past kappa ~ 1e8,
    # sketch-and-solve (multisketch) tracks QR.
    d, n = 1 << 17, 16
    k1, k2 = 2 * n * n, 2 * n
    for kappa in (1e2, 1e6, 1e10):
        A = synth.ill_conditioned(d, n, kappa, seed=3)
        b = synth.rhs(A, "consistent", seed=3)
        nb = np.linalg.norm(b)
        x_ms, _ = oracle.ms_lstsq(A, b, k1, k2, seed=1)
        r_ms = oracle.residual_norm(A, b, x_ms) / nb
        assert r_ms <= 1e-6, (kappa, r_ms)
        try:
            r_ne = oracle.residual_norm(A, b, oracle.normal_eq(A, b)) / nb
        except oracle.OracleError as e:
            assert e.status == oracle.ENOTPD and kappa > 1e8
            continue
        if kappa <= 1e6:
            assert r_ne <= 1e-6
        else:
            assert r_ne > 1e-2 or r_ne > 1e3 * max(r_ms, 1e-16), (kappa, r_ne)


def test_residual_norm_closed_forms():
    # or_residual_norm (P:L338's ||b - Ax||) pinned to values fixed by arithmetic, not by a re-typed
    # formula: (i) integer cases whose residual is a Pythagorean vector (exact); (ii) x = 0 gives
    # ||b|| and x solving A x = b exactly gives 0; (iii) a residual orthogonal to range(A) built from a
    # Householder reflector: b = A x + t u with u a unit vector orthogonal to A's columns -> |t|.
    A = np.array([[1.0, 0.0], [0.0, 1.0], [0.0, 0.0], [0.0, 0.0]])
    assert oracle.residual_norm(A, np.array([4.0, -2.0, 3.0, 4.0]), np.array([4.0, -2.0])) == 5.0
    Ai = np.array([[2.0, 1.0], [1.0, 3.0], [0.0, 1.0]])
    x = np.array([1.0, 2.0])
    r = np.array([5.0, 12.0, 0.0])                  # ||r|| = 13 exactly
    assert oracle.residual_norm(Ai, Ai @ x + r, x) == 13.0
    rng = np.random.default_rng(11)
    B = rng.standard_normal((50, 4))
    b = rng.standard_normal(50)
    assert oracle.residual_norm(B, b, np.zeros(4)) == pytest.approx(float(np.sqrt(np.sum(b * b))), rel=1e-15, abs=0)
    assert oracle.residual_norm(Ai, Ai @ x, x) == 0.0
    # (iii): the last column of a full QR of B is orthogonal to B's range
    Q, _ = np.linalg.qr(np.column_stack([B, rng.standard_normal(50)]), mode="reduced")
    u = Q[:, -1] - B @ np.linalg.lstsq(B, Q[:, -1], rcond=None)[0]
    u /= np.linalg.norm(u)
    xs = rng.standard_normal(4)
    for t, tol in ((1e-8, 1e-5), (0.5, 1e-12), (3.0, 1e-12)):   # b's rounding (~1e-15) sets the tolerance
        assert oracle.residual_norm(B, B @ xs + t * u, xs) == pytest.approx(t, rel=tol, abs=0)
    # a dropped term or a wrong sign in the accumulation fails one of the above; a transposed operand
    # fails the non-square integer case (A^T has the wrong shape for x)
