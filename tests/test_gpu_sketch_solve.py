"""GPU parity of the other sketch-and-solve operators (Fig 5 bars):
Gaussian sketch (gs_apply / gs_lstsq), CountSketch-only (cs_lstsq, GEQRF on k1 x (n+1)) and the
Count+SRHT multisketch (msh_apply / msh_lstsq), each against the oracle composition of the same
steps (oracle.gauss + gemm_comp, cs_apply + sketch_solve, cs_apply + srht_apply + sketch_solve).
"""
import numpy as np
import pytest

import oracle
import synth
from tests._util import check_fitted, check_le, gpu_colmajor, host, ls_tol, unpack

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2508_14209_b200 as csk  # noqa: E402

U = 2.2e-16


def _ls_tol(A, b, xo, kappa):
    nb = np.linalg.norm(b)
    rr = oracle.residual_norm(A, b, xo) / nb
    return nb, max(1e-8, 64 * U * kappa * rr)


@pytest.mark.parametrize("d,n,k,chunk", [(4096, 6, 16, None), (10000, 9, 20, "1000"), (777, 3, 8, "64")])
def test_gs_apply_matches_oracle(monkeypatch, d, n, k, chunk):
    if chunk:
        monkeypatch.setenv("CSK_GS_CHUNK", chunk)
    A = synth.gaussian_matrix(d, n, seed=2)
    b = synth.rhs(A, "easy", seed=2)
    Z = host(csk.gs_apply(gpu_colmajor(A), k, seed=5, b=gpu_colmajor(b)))
    Ab = np.column_stack([A, b])
    G = oracle.gauss(k, d, seed=5)
    Zo, Zabs = oracle.gemm_comp(G, Ab, np.abs(Ab))
    assert np.all(np.abs(Z - Zo) <= 1e-12 * Zabs)


def test_gs_apply_row_partition():
    d, n, k = 6000, 4, 12
    A = synth.integer_matrix(d, n, seed=3)
    full = host(csk.gs_apply(gpu_colmajor(A), k, seed=1))
    acc = np.zeros_like(full)
    for r0, r1 in [(0, 1000), (1000, 3500), (3500, 6000)]:
        acc += host(csk.gs_apply(gpu_colmajor(A[r0:r1]), k, seed=1, row0=r0))
    Zo, Zabs = oracle.gemm_comp(oracle.gauss(k, d, seed=1), A, np.abs(A))
    assert np.all(np.abs(acc - Zo) <= 1e-12 * Zabs)
    assert np.all(np.abs(full - Zo) <= 1e-12 * Zabs)


@pytest.mark.parametrize("kappa", [1e2, 1e8])
def test_gs_lstsq_matches_oracle(kappa):
    d, n = 1 << 14, 12
    k = 2 * n
    A = synth.ill_conditioned(d, n, kappa, seed=4)
    b = synth.rhs(A, "hard", seed=4)
    x, r = csk.gs_lstsq(gpu_colmajor(A), gpu_colmajor(b), k, seed=3)
    Zo = oracle.gemm_comp(oracle.gauss(k, d, seed=3), np.column_stack([A, b]))
    xo, ro = oracle.sketch_solve(Zo, n)
    nb, tol = _ls_tol(A, b, xo, kappa)
    check_fitted(A, host(x) - xo, nb, tol)
    assert abs(r - ro) <= tol * nb


@pytest.mark.parametrize("kappa", [1e2, 1e10])
@pytest.mark.parametrize("mode", ["easy", "consistent"])
def test_cs_lstsq_matches_oracle(kappa, mode):
    d, n = 1 << 14, 8
    k1 = 2 * n * n
    A = synth.ill_conditioned(d, n, kappa, seed=5)
    b = synth.rhs(A, mode, seed=5)
    plan = csk.cs_plan(d, k1, 2)
    x, r = csk.cs_lstsq(plan, gpu_colmajor(A), gpu_colmajor(b))
    h, s, = oracle.codes(d, k1, 2)
    xo, ro = oracle.sketch_solve(oracle.cs_apply(h, s, A, k1, b=b), n)
    nb, tol = _ls_tol(A, b, xo, kappa)
    check_fitted(A, host(x) - xo, nb, tol)
    assert abs(r - ro) <= tol * nb + 1e-300


@pytest.mark.parametrize("d,n", [(1 << 14, 8), (30011, 16)])
def test_msh_apply_matches_oracle(d, n):
    k1, k2 = 2 * n * n, 2 * n     # k1 = 128 / 512: powers of two
    A = synth.gaussian_matrix(d, n, seed=6)
    b = synth.rhs(A, "easy", seed=6)
    plan = csk.cs_plan(d, k1, 4)
    Z = host(csk.msh_apply(plan, k2, gpu_colmajor(A), gpu_colmajor(b)))
    h, s = oracle.codes(d, k1, 4)
    Ab = np.column_stack([A, b])
    SA, T = oracle.cs_apply(h, s, Ab, k1, with_abs=True)
    Zo = oracle.srht_apply(SA, k2, seed=4)
    # |dZ| <= 1e-12 * k2^-1/2 sum_m T[m, c]: the SRHT of the CountSketch's |terms| bound
    bound = 1e-12 * T.sum(axis=0)[None, :] / np.sqrt(k2)
    assert np.all(np.abs(Z - Zo) <= bound)


def test_msh_lstsq_matches_oracle():
    d, n = 1 << 15, 16
    k1, k2 = 2 * n * n, 2 * n
    A = synth.ill_conditioned(d, n, 1e6, seed=7)
    b = synth.rhs(A, "hard", seed=7)
    plan = csk.cs_plan(d, k1, 1)
    x, r = csk.msh_lstsq(plan, k2, gpu_colmajor(A), gpu_colmajor(b))
    h, s = oracle.codes(d, k1, 1)
    Zo = oracle.srht_apply(oracle.cs_apply(h, s, A, k1, b=b), k2, seed=1)
    xo, ro = oracle.sketch_solve(Zo, n)
    nb, tol = _ls_tol(A, b, xo, 1e6)
    check_fitted(A, host(x) - xo, nb, tol)


def test_msh_needs_power_of_two_k1():
    A = gpu_colmajor(synth.gaussian_matrix(1000, 3, seed=1))
    plan = csk.cs_plan(1000, 18, 1)
    with pytest.raises(csk.CskError) as e:
        csk.msh_apply(plan, 8, A)
    assert e.value.status == csk.csk.ESHAPE
