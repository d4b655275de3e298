"""GPU parity of rc_lstsq (rand_cholQR least squares, Alg 5) against the oracle.

Both sides run Alg 5 on the same multisketch (plan seed, k1 = 2n^2, k2 = 2n); x must agree in
fitted values within the LS perturbation bound (R16b, the Wedin term), and R = R1 R0
within rounding of the R factor of A.  The row-chunked pass is exercised with many chunks and
a ragged tail (CSK_RC_CHUNK).
"""
import numpy as np
import pytest

import oracle
import synth
from tests._util import check_fitted, check_le, gpu_colmajor, host, ls_tol

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2508_14209_b200 as csk  # noqa: E402

U = 2.2e-16


def _case(d, n, kappa, mode, seed):
    A = synth.ill_conditioned(d, n, kappa, seed=seed)
    b = synth.rhs(A, mode, seed=seed)
    return A, b


def _oracle(A, b, k1, k2, seed):
    Y = oracle.ms_apply(A, k1, k2, seed)
    return oracle.rand_cholqr_lstsq(A, b, Y, return_R=True)


@pytest.mark.parametrize("kappa", [1e2, 1e10])
@pytest.mark.parametrize("mode", ["easy", "hard", "consistent"])
def test_rc_lstsq_matches_oracle(kappa, mode):
    d, n = 1 << 15, 16
    k1, k2 = 2 * n * n, 2 * n
    A, b = _case(d, n, kappa, mode, seed=4)
    plan = csk.cs_plan(d, k1, 1)
    x, R = csk.rc_lstsq(plan, k2, gpu_colmajor(A), gpu_colmajor(b), want_R=True)
    xo, Ro = _oracle(A, b, k1, k2, seed=1)
    nb = np.linalg.norm(b)
    rr = oracle.residual_norm(A, b, xo) / nb
    tol = max(1e-8, 64 * U * kappa * rr)
    check_fitted(A, host(x) - xo, nb, tol)
    Rg = host(R)
    assert np.all(np.tril(Rg, -1) == 0)
    if kappa <= 1e2:
        assert np.abs(Rg - Ro).max() <= 1e-10 * np.abs(Ro).max()


@pytest.mark.parametrize("chunk", ["1024", "3000", "100000"])
def test_rc_lstsq_chunked_ragged(monkeypatch, chunk):
    d, n = 20011, 24
    k1, k2 = 2 * n * n, 2 * n
    A, b = _case(d, n, 1e4, "hard", seed=5)
    monkeypatch.setenv("CSK_RC_CHUNK", chunk)
    plan = csk.cs_plan(d, k1, 3)
    x = host(csk.rc_lstsq(plan, k2, gpu_colmajor(A), gpu_colmajor(b)))
    xo, _ = _oracle(A, b, k1, k2, seed=3)
    nb = np.linalg.norm(b)
    rr = oracle.residual_norm(A, b, xo) / nb
    check_fitted(A, x - xo, nb, max(1e-8, 64 * U * 1e4 * rr))


def test_rc_lstsq_is_true_least_squares():
    # no sketch distortion: x is the LS solution of A itself, unlike ms_lstsq
    d, n = 50000, 32
    k1, k2 = 2 * n * n, 2 * n
    A, b = _case(d, n, 1e3, "hard", seed=6)
    plan = csk.cs_plan(d, k1, 1)
    x = host(csk.rc_lstsq(plan, k2, gpu_colmajor(A), gpu_colmajor(b)))
    xs, *_ = np.linalg.lstsq(A, b, rcond=None)
    nb = np.linalg.norm(b)
    r = np.linalg.norm(b - A @ xs)
    assert np.linalg.norm(A @ (x - xs)) <= 64 * U * (nb + 1e3 * r)
    xm, _ = csk.ms_lstsq(plan, k2, gpu_colmajor(A), gpu_colmajor(b))
    r_ms = oracle.residual_norm(A, b, host(xm))
    r_rc = oracle.residual_norm(A, b, x)
    assert r_rc <= r * (1 + 1e-12) and r_ms > r_rc * (1 + 1e-6)


def test_rc_lstsq_stable_at_kappa_1e10():
    # Fig 8 setup: b = Ae; rand_cholQR keeps a QR-level residual where NE fails
    d, n = 1 << 17, 16
    A, b = _case(d, n, 1e10, "consistent", seed=3)
    plan = csk.cs_plan(d, 2 * n * n, 1)
    x = host(csk.rc_lstsq(plan, 2 * n, gpu_colmajor(A), gpu_colmajor(b)))
    nb = np.linalg.norm(b)
    xs, *_ = np.linalg.lstsq(A, b, rcond=None)
    r_qr = oracle.residual_norm(A, b, xs) / nb
    assert oracle.residual_norm(A, b, x) / nb <= max(100 * r_qr, 1e-13)


def test_rc_lstsq_errors():
    d, n = 4096, 8
    A, b = _case(d, n, 1e2, "easy", seed=1)
    plan = csk.cs_plan(d, 128, 1)
    with pytest.raises(csk.CskError) as e:
        csk.rc_lstsq(plan, n, gpu_colmajor(A), gpu_colmajor(b))      # k2 < n + 1
    assert e.value.status == csk.csk.ESHAPE
    As = A.copy(order="F")
    As[:, 3] = As[:, 2]
    with pytest.raises(csk.CskError) as e:
        csk.rc_lstsq(plan, 2 * n, gpu_colmajor(As), gpu_colmajor(b))
    assert e.value.status == csk.csk.ESINGULAR


@pytest.mark.parametrize("path", ["fused", "blas"])
@pytest.mark.parametrize("d,n", [(70001, 128), (30000, 100), (4099, 64), (513, 5), (64, 8)])
def test_rc_lstsq_paths_and_shapes(monkeypatch, path, d, n):
    # fused DMMA pass (n <= 128: 8-column blocks padded to 16/32/64/128) and the cuBLAS chunked
    # pass must both reproduce the oracle; ragged 64-row tiles and padded column blocks included
    k1, k2 = 2 * n * n, 2 * n
    if path == "blas":
        monkeypatch.setenv("CSK_RC_PATH", "0")
    A, b = _case(d, n, 1e6, "easy", seed=7)
    plan = csk.cs_plan(d, k1, 5)
    x, R = csk.rc_lstsq(plan, k2, gpu_colmajor(A), gpu_colmajor(b), want_R=True)
    xo, Ro = _oracle(A, b, k1, k2, seed=5)
    nb = np.linalg.norm(b)
    rr = oracle.residual_norm(A, b, xo) / nb
    check_fitted(A, host(x) - xo, nb, max(1e-8, 64 * U * 1e6 * rr))
    Rg = host(R)
    AtA = A.T @ A
    assert np.abs(Rg.T @ Rg - AtA).max() <= 1e-11 * np.abs(AtA).max()


@pytest.mark.parametrize("p", [1, 3])
def test_rc_phases_row_partitioned(p):
    # the distributed form on one GPU: sum_g Z_g -> rc_r0 -> sum_g rc_gram(A_g) -> rc_finish
    # must reproduce rc_lstsq (and the oracle) -- P:L373-381 linearity of both reductions
    d, n = 30011, 20
    k1, k2 = 2 * n * n, 2 * n
    A, b = _case(d, n, 1e8, "hard", seed=9)
    Ad, bd = gpu_colmajor(A), gpu_colmajor(b)
    bounds = [g * d // p for g in range(p + 1)]
    Z = None
    for g in range(p):
        r0, r1 = bounds[g], bounds[g + 1]
        plan = csk.cs_plan(r1 - r0, k1, 2, row0=r0)
        Zg = csk.ms_apply(plan, k2, Ad[r0:r1], b=bd[r0:r1])
        Z = Zg if Z is None else Z + Zg
    R0 = csk.rc_r0(Z, n)
    C = sum(csk.rc_gram(Ad[bounds[g]:bounds[g + 1]], bd[bounds[g]:bounds[g + 1]], R0) for g in range(p))
    x, R = csk.rc_finish(C, R0, want_R=True)
    xo, Ro = _oracle(A, b, k1, k2, seed=2)
    nb = np.linalg.norm(b)
    rr = oracle.residual_norm(A, b, xo) / nb
    check_fitted(A, host(x) - xo, nb, max(1e-8, 64 * U * 1e8 * rr))
    x1 = host(csk.rc_lstsq(csk.cs_plan(d, k1, 2), k2, Ad, bd))
    check_fitted(A, host(x) - x1, nb, max(1e-8, 64 * U * 1e8 * rr))


@pytest.mark.parametrize("path", ["trsm", "blas"])
@pytest.mark.parametrize("n,k1", [(160, 2 * 160 * 160), (256, 4096), (129, 2 * 129 * 129)])
def test_rc_lstsq_wide(monkeypatch, path, n, k1):
    # 128 < n <= 256: the DMMA TRSM-to-workspace kernel + cuBLAS Gram ("trsm"), or the row-chunked
    # cuBLAS DTRSM pass ("blas"); both must match the oracle.  (n = 256 with a smaller k1 keeps the
    # oracle's compensated G-stage to seconds; rand_cholQR needs only a subspace embedding.)
    if path == "blas":
        monkeypatch.setenv("CSK_RC_PATH", "0")
    d = 30011
    k2 = 2 * n
    A, b = _case(d, n, 1e4, "easy", seed=11)
    plan = csk.cs_plan(d, k1, 6)
    x = host(csk.rc_lstsq(plan, k2, gpu_colmajor(A), gpu_colmajor(b)))
    xo, _ = _oracle(A, b, k1, k2, seed=6)
    nb = np.linalg.norm(b)
    rr = oracle.residual_norm(A, b, xo) / nb
    check_fitted(A, x - xo, nb, max(1e-8, 64 * U * 1e4 * rr))
