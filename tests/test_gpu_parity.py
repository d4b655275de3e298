"""GPU parity: the CUDA path through the C-ABI against the CPU oracle.

Bit-exact: codes (hash), the counting sort, integer-valued A.  Tolerances
(BASELINE.json north_star): fp64 |dSA| <= 1e-12 * sum|terms|, fp32 <= 1e-5;
G within 1e-13/sqrt(k2); Z within 1e-12 |G| T; least squares
||A (x_gpu - x_oracle)|| / ||b|| <= 1e-8 (R16).
"""
import ctypes
import os
import subprocess

import numpy as np
import pytest

import oracle
import synth
from tests._util import assert_within_T, check_fitted, check_le, gpu_colmajor, host, ls_tol, unpack

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2508_14209_b200 as csk  # noqa: E402

VARIANTS = ["L", "T", "S", "G", "B", "X"]


# ------------------------------------------------------------------ codes
@pytest.mark.parametrize("d,k1,seed,row0", [(4096, 64, 1, 0), (10007, 1000, 7, 3), (1, 1, 2, 0), (5, 8192, 1, 6),
                                            (100003, 8192, 1, 1 << 20), (64, 3, 9, (1 << 33) + 1)])
def test_codes_bit_exact(d, k1, seed, row0):
    plan = csk.cs_plan(d, k1, seed, row0=row0)
    code, _, _ = plan.export()
    h, s = unpack(code)
    ho, so = oracle.codes(d, k1, seed, row0)
    assert np.array_equal(h, ho) and np.array_equal(s, so)


def _curand_probe():
    here = os.path.join(os.path.dirname(__file__), "helpers")
    so = os.path.join(here, "build", "libcurand_probe.so")
    if not os.path.exists(so):
        os.makedirs(os.path.dirname(so), exist_ok=True)
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                               "-Xcompiler", "-fPIC", "-o", so, os.path.join(here, "curand_probe.cu")])
    return ctypes.CDLL(so)


def test_oracle_philox_matches_curand():
    # library pin of the oracle's hash: cuRAND Philox4x32-10 ("cuRAND")
    lib = _curand_probe()
    q = np.array([0, 1, 2, 12345, (1 << 32) + 7, (1 << 40) + 3], dtype=np.uint64)
    out = np.zeros((len(q), 4), np.uint32)
    for seed in (1, 0xDEADBEEFCAFEF00D):
        assert lib.curand_probe(ctypes.c_uint64(seed), q.ctypes.data_as(ctypes.c_void_p),
                                out.ctypes.data_as(ctypes.c_void_p), len(q)) == 0
        for i, qi in enumerate(q):
            ctr = [int(qi) & 0xFFFFFFFF, int(qi) >> 32, 0, 0]
            key = [seed & 0xFFFFFFFF, seed >> 32]
            assert list(oracle.philox4x32_10(ctr, key)) == list(out[i])


@pytest.mark.parametrize("d,k1", [(4096, 64), (100000, 8192), (3000, 1), (77777, 131072), (1 << 20, 65536)])
def test_sort_bit_exact(d, k1):
    plan = csk.cs_plan(d, k1, 3, sort=True)
    code, offsets, perm = plan.export()
    h, _ = unpack(code)
    oo, po = oracle.count_sort(h, k1)
    assert np.array_equal(offsets, oo)
    assert np.array_equal(perm, po)


# ------------------------------------------------------------- cs_apply
def _check_apply(plan, h, s, A, b, variant, dtype=np.float64, rel=1e-12, lda_pad=0, ldsa_pad=0):
    d = A.shape[0] if A is not None else len(b)
    Ad = None
    if A is not None:
        if lda_pad:
            big = np.zeros((d + lda_pad, A.shape[1]), dtype=dtype, order="F")
            big[:d] = A
            Ad = gpu_colmajor(big)[:d]
        else:
            Ad = gpu_colmajor(A.astype(dtype))
    bd = None if b is None else gpu_colmajor(b.astype(dtype))
    ncols = (0 if A is None else A.shape[1]) + (b is not None)
    SA = None
    if ldsa_pad:
        SA = torch.full((ncols, plan.k1 + ldsa_pad), 7.0, dtype=Ad.dtype if Ad is not None else bd.dtype,
                        device="cuda").t()[: plan.k1]
    SA = csk.cs_apply(plan, Ad, b=bd, SA=SA, variant=variant)
    torch.cuda.synchronize()
    got = host(SA)
    Aor = A if A is not None else np.zeros((d, 0))
    exp, T = oracle.cs_apply(h, s, Aor.astype(dtype), plan.k1, b=None if b is None else b.astype(dtype),
                             with_abs=True)
    assert_within_T(got, exp, T, rel)
    return got, exp


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("d,n,k1", [(4096, 8, 64), (10007, 37, 1000), (5000, 1, 8192), (1000, 3, 1), (777, 70, 4096),
                                    (3000, 5, 65536)])
def test_cs_apply_fp64(variant, d, n, k1):
    plan = csk.cs_plan(d, k1, 1, sort=(variant == "G"))
    h, s = oracle.codes(d, k1, 1)
    A = synth.gaussian_matrix(d, n, seed=2)
    _check_apply(plan, h, s, A, None, variant)


@pytest.mark.parametrize("variant", VARIANTS)
def test_cs_apply_with_b_and_padding(variant):
    d, n, k1 = 9001, 12, 512
    plan = csk.cs_plan(d, k1, 5, sort=(variant == "G"))
    h, s = oracle.codes(d, k1, 5)
    A = synth.gaussian_matrix(d, n, seed=3)
    b = synth.rhs(A, "hard", seed=3)
    _check_apply(plan, h, s, A, b, variant, lda_pad=3, ldsa_pad=5)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("d,n,k1", [(9001, 12, 512), (100003, 64, 8192), (4099, 100, 777), (5000, 200, 4096)])
def test_cs_apply_contiguous_Ab(variant, d, n, k1):
    # [A b] stored as one d x (n+1) column-major buffer (the TMA variant's fast layout)
    plan = csk.cs_plan(d, k1, 5, sort=(variant == "G"))
    h, s = oracle.codes(d, k1, 5)
    Ab = synth.gaussian_matrix(d, n + 1, seed=3)
    buf = gpu_colmajor(Ab)
    SA = csk.cs_apply(plan, buf[:, :n], b=buf[:, n], variant=variant)
    exp, T = oracle.cs_apply(h, s, Ab[:, :n], k1, b=Ab[:, n], with_abs=True)
    assert_within_T(host(SA), exp, T, 1e-12)


@pytest.mark.parametrize("variant", ["B", "X"])
def test_cs_apply_contiguous_Ab_fp32(variant):
    d, n, k1 = 50001, 64, 4096
    plan = csk.cs_plan(d, k1, 6)
    h, s = oracle.codes(d, k1, 6)
    Ab = synth.gaussian_matrix(d, n + 1, seed=4, dtype=np.float32)
    buf = gpu_colmajor(Ab)
    SA = csk.cs_apply(plan, buf[:, :n], b=buf[:, n], variant=variant)
    exp, T = oracle.cs_apply(h, s, Ab[:, :n], k1, b=Ab[:, n], with_abs=True)
    assert_within_T(host(SA), exp, T, 1e-5)


@pytest.mark.parametrize("variant", ["B", "X"])
def test_cs_apply_chunk_major_layout(variant):
    # k1 * ncols * 8 > L2/2 switches the TMA variants to one SA^T slice per column chunk (C3 regime)
    d, n, k1 = 30011, 200, 65536
    plan = csk.cs_plan(d, k1, 8)
    h, s = oracle.codes(d, k1, 8)
    Ab = synth.integer_matrix(d, n + 1, seed=8, lo=-1000, hi=1000)
    buf = gpu_colmajor(Ab)
    SA = csk.cs_apply(plan, buf[:, :n], b=buf[:, n], variant=variant)
    exp = oracle.cs_apply(h, s, Ab[:, :n], k1, b=Ab[:, n])
    assert np.array_equal(host(SA), exp)


@pytest.mark.parametrize("variant", VARIANTS)
def test_cs_apply_only_b(variant):
    d, k1 = 3333, 100
    plan = csk.cs_plan(d, k1, 5, sort=(variant == "G"))
    h, s = oracle.codes(d, k1, 5)
    b = synth.gaussian_matrix(d, 1, seed=4)[:, 0]
    _check_apply(plan, h, s, None, b, variant)


@pytest.mark.parametrize("variant", VARIANTS)
def test_cs_apply_integer_exact(variant):
    d, n, k1 = 50000, 9, 2048
    plan = csk.cs_plan(d, k1, 3, sort=(variant == "G"))
    h, s = oracle.codes(d, k1, 3)
    A = synth.integer_matrix(d, n, seed=5, lo=-(1 << 20), hi=1 << 20)
    got, exp = _check_apply(plan, h, s, A, None, variant, rel=0.0)
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("variant", VARIANTS)
def test_cs_apply_fp32(variant):
    d, n, k1 = 20000, 6, 1024
    plan = csk.cs_plan(d, k1, 4, sort=(variant == "G"))
    h, s = oracle.codes(d, k1, 4)
    A = synth.gaussian_matrix(d, n, seed=6, dtype=np.float32)
    _check_apply(plan, h, s, A, None, variant, dtype=np.float32, rel=1e-5)


def test_worked_example_forced_plan():
    # d=4, k=2, r=[0,1,0,1], s=[+,+,-,+], A=[1,2,3,4]^T -> Y=[-2, 6]^T
    for variant in VARIANTS:
        plan = csk.cs_plan_from_arrays([0, 1, 0, 1], [1, 1, -1, 1], 2, sort=True)
        Y = csk.cs_apply(plan, gpu_colmajor(np.array([[1.0], [2.0], [3.0], [4.0]])), variant=variant)
        assert host(Y)[:, 0].tolist() == [-2.0, 6.0]


def test_identity_plan_returns_A():
    d, n = 300, 4
    A = synth.gaussian_matrix(d, n, seed=5)
    plan = csk.cs_plan_from_arrays(np.arange(d), np.ones(d), d)
    for variant in VARIANTS:
        if variant == "G":
            continue
        assert np.array_equal(host(csk.cs_apply(plan, gpu_colmajor(A), variant=variant)), A)


def test_sorted_variant_deterministic():
    d, n, k1 = 200000, 4, 4096
    plan = csk.cs_plan(d, k1, 9, sort=True)
    A = gpu_colmajor(synth.gaussian_matrix(d, n, seed=9))
    a = host(csk.cs_apply(plan, A, variant="G"))
    b = host(csk.cs_apply(plan, A, variant="G"))
    assert np.array_equal(a, b)


@pytest.mark.parametrize("p", [1, 2, 4, 7])
def test_partition_invariance_on_one_gpu(p):
    # CA = sum_i C^(i) A^(i) with row0-plans (the multi-GPU identity, one device)
    d, n, k1 = 100001, 5, 4096
    A = synth.integer_matrix(d, n, seed=11)
    full = host(csk.cs_apply(csk.cs_plan(d, k1, 1), gpu_colmajor(A)))
    bounds = np.linspace(0, d, p + 1).astype(int)
    acc = np.zeros_like(full)
    for g in range(p):
        r0, r1 = bounds[g], bounds[g + 1]
        acc += host(csk.cs_apply(csk.cs_plan(r1 - r0, k1, 1, row0=int(r0)), gpu_colmajor(A[r0:r1])))
    assert np.array_equal(acc, full)


def test_error_paths():
    plan = csk.cs_plan(100, 10, 1)
    A = torch.zeros((3, 100), dtype=torch.float64, device="cuda").t()
    lib = csk.lib()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    SA = torch.zeros((3, 10), dtype=torch.float64, device="cuda").t()
    assert lib.cs_apply(plan.handle, 0, 3, ctypes.c_void_p(A.data_ptr()), 99, None,
                        ctypes.c_void_p(SA.data_ptr()), 10, -1, st) == csk.csk.ESHAPE
    assert lib.cs_apply(plan.handle, 0, 3, ctypes.c_void_p(A.data_ptr()), 100, None,
                        ctypes.c_void_p(SA.data_ptr()), 9, -1, st) == csk.csk.ESHAPE
    assert lib.cs_apply(plan.handle, 0, 3, None, 100, None, ctypes.c_void_p(SA.data_ptr()), 10, -1,
                        st) == csk.csk.EINVAL
    assert lib.cs_apply(plan.handle, 7, 3, ctypes.c_void_p(A.data_ptr()), 100, None,
                        ctypes.c_void_p(SA.data_ptr()), 10, -1, st) == csk.csk.EDTYPE
    assert lib.cs_apply(plan.handle, 0, 3, ctypes.c_void_p(A.data_ptr()), 100, None,
                        ctypes.c_void_p(SA.data_ptr()), 10, 3, st) == csk.csk.EUNSUPPORTED  # G without sort
    out = ctypes.c_void_p()
    assert lib.cs_plan(0, 10, 1, 0, 0, st, ctypes.byref(out)) == csk.csk.EINVAL
    assert lib.cs_plan(10, 1 << 31, 1, 0, 0, st, ctypes.byref(out)) == csk.csk.EINVAL
    with pytest.raises(csk.CskError) as e:
        csk.cs_plan_from_arrays([0, 5], [1, 1], 3)
    assert e.value.status == csk.csk.EINVAL
    Z = torch.zeros((5, 8), dtype=torch.float64, device="cuda").t()
    x = torch.zeros(8, dtype=torch.float64, device="cuda")
    assert lib.ms_solve(4, 4, ctypes.c_void_p(Z.data_ptr()), 8, ctypes.c_void_p(x.data_ptr()), None,
                        st) == csk.csk.ESHAPE


# ------------------------------------------------------------ multisketch
def test_gauss_matches_oracle():
    # identity plan (k1 = d) and A = I give S A = I, so Z = G exactly
    for k2, k1 in [(8, 32), (3, 5), (128, 256)]:
        plan_seeded = csk.cs_plan(k1, k1, 77)      # G is drawn from the plan's seed
        Z = host(csk.ms_apply(plan_seeded, k2, gpu_colmajor(np.eye(k1))))
        h, s = oracle.codes(k1, k1, 77)
        S = np.zeros((k1, k1))
        S[h, np.arange(k1)] = s
        G = oracle.gauss(k2, k1, 77)
        # G S with S a signed permutation is exact, so Z - G S is the Box-Muller difference itself:
        # |dN| <= 1e-13, |dG| = |dN| / sqrt(k2)
        check_le(np.abs(Z - G @ S).max(), 1e-13 / np.sqrt(k2), "max |G_gpu - G_oracle|")


@pytest.mark.parametrize("d,n,k1,k2", [(4096, 8, 128, 16), (20000, 16, 512, 32), (5000, 3, 18, 6),
                                       (30011, 129, 4096, 260), (200003, 64, 131072, 130), (7001, 5, 1000, 1),
                                       (9000, 70, 4096, 65), (12000, 10, 600, 191), (4099, 65, 777, 64),
                                       (100003, 64, 8192, 128), (30011, 128, 32768, 256)])
def test_ms_apply_matches_oracle(d, n, k1, k2):
    # the hand-written DMMA G-stage (gstage.cu) on the CountSketch's row-major SA^T: one chunk (C2-like),
    # two chunks (129 + b), chunk-major (k1 = 131072), k2 not a multiple of 8, k1 not a multiple of 32
    plan = csk.cs_plan(d, k1, 3)
    A = synth.gaussian_matrix(d, n, seed=1)
    b = synth.rhs(A, "easy", seed=1)
    Z = host(csk.ms_apply(plan, k2, gpu_colmajor(A), b=gpu_colmajor(b)))
    Zo, Zabs = oracle.ms_apply(A, k1, k2, seed=3, b=b, with_abs=True)
    assert_within_T(Z, Zo, Zabs, 1e-12)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("d,n,k1,k2", [(9000, 70, 4096, 65), (50000, 100, 2048, 200), (3001, 4, 64, 8)])
def test_ms_apply_every_countsketch_variant(monkeypatch, variant, d, n, k1, k2):
    # every CountSketch variant feeds the same G-stage: row-major workspaces directly (T, B, X; T's
    # one-row layout wider than 72 columns is re-cut into 64-column chunks), column-major ones (L, S, G)
    # through the row-major conversion
    monkeypatch.setenv("CSK_VARIANT", str(csk.csk.VARIANTS[variant]))
    plan = csk.cs_plan(d, k1, 4, sort=(variant == "G"))
    A = synth.gaussian_matrix(d, n, seed=5)
    b = synth.rhs(A, "hard", seed=5)
    Z = host(csk.ms_apply(plan, k2, gpu_colmajor(A), b=gpu_colmajor(b)))
    Zo, Zabs = oracle.ms_apply(A, k1, k2, seed=4, b=b, with_abs=True)
    assert_within_T(Z, Zo, Zabs, 1e-12)


def test_ms_apply_gstage_large_k2_and_k1():
    # k2 = 512, k1 = 131072 (C3's G-stage shape): 4 M-tiles, stream-K over 5 chunk-major chunks
    d, n, k1, k2 = 300007, 256, 131072, 512
    plan = csk.cs_plan(d, k1, 6)
    A = synth.gaussian_matrix(d, n, seed=2)
    b = synth.rhs(A, "hard", seed=2)
    Z = host(csk.ms_apply(plan, k2, gpu_colmajor(A), b=gpu_colmajor(b)))
    Zo, Zabs = oracle.ms_apply(A, k1, k2, seed=6, b=b, with_abs=True)
    assert_within_T(Z, Zo, Zabs, 1e-12)


@pytest.mark.parametrize("ctas", ["1", "3", "7", "1000"])
def test_ms_apply_gstage_any_split_deterministic(monkeypatch, ctas):
    # the stream-K split (1 CTA = no split, ragged splits, more CTAs than k-blocks): same tolerance,
    # and each split is bitwise reproducible (fixed-order partial sums)
    monkeypatch.setenv("CSK_GS_CTAS", ctas)
    d, n, k1, k2 = 60000, 70, 4000, 140
    plan = csk.cs_plan(d, k1, 2)
    Ai = synth.integer_matrix(d, n, seed=3)
    A = synth.gaussian_matrix(d, n, seed=3)
    Ad = gpu_colmajor(A)
    Z1 = host(csk.ms_apply(plan, k2, Ad))
    Z2 = host(csk.ms_apply(plan, k2, Ad))
    Zo, Zabs = oracle.ms_apply(A, k1, k2, seed=2, with_abs=True)
    assert_within_T(Z1, Zo, Zabs, 1e-12)
    # the CountSketch's atomics reorder SA's sums, so bitwise reproducibility is checked on integer A
    Zi1 = host(csk.ms_apply(plan, k2, gpu_colmajor(Ai)))
    Zi2 = host(csk.ms_apply(plan, k2, gpu_colmajor(Ai)))
    assert np.array_equal(Zi1, Zi2)
    del Z2


@pytest.mark.parametrize("d,n,k1", [(40000, 33, 2048), (1 << 20, 8, 128)])
def test_ms_apply_fp32_input(d, n, k1):
    # fp32 [A b]: the sketch accumulates in bounded-depth fp32 copies summed in fp64 (R12), the G-stage
    # runs in fp64, Z is rounded once.  (2^20, 8, 128): 128 copies, the warp-per-element combine
    k2 = 2 * n
    plan = csk.cs_plan(d, k1, 8)
    A = synth.gaussian_matrix(d, n, seed=4, dtype=np.float32)
    b = synth.gaussian_matrix(d, 1, seed=5, dtype=np.float32)[:, 0]
    Z = host(csk.ms_apply(plan, k2, gpu_colmajor(A), b=gpu_colmajor(b)))
    assert Z.dtype == np.float32
    Zo, Zabs = oracle.ms_apply(A, k1, k2, seed=8, b=b, with_abs=True)
    assert_within_T(Z, Zo, Zabs, 1e-5)


# every small-solve kernel (csrc/qr_wy.cu default, forced wider clusters, and the older
# multisketch.cu kernels kept for m > 512) against the oracle's Householder QR
SOLVERS = {
    "wy": {},
    "wy_p4": {"CSK_QR_WY_P": "4"},
    "wy_p16": {"CSK_QR_WY_P": "16"},
    "wy_p16_l2_staging": {"CSK_QR_WY_P": "16", "CSK_QR_PUSH": "0"},   # V/T staged through L2 only (no DSMEM push)
    "cluster": {"CSK_QR_WY": "0"},
    "single": {"CSK_QR_WY": "0", "CSK_QR_SINGLE": "1"},
}


@pytest.fixture(params=list(SOLVERS), ids=list(SOLVERS))
def solver_env(request, monkeypatch):
    for k, v in SOLVERS[request.param].items():
        monkeypatch.setenv(k, v)
    return request.param


def test_ms_solve_matches_oracle(solver_env):
    rng = np.random.default_rng(5)
    for m, n in [(16, 8), (128, 64), (256, 128), (40, 3), (512, 256), (300, 150), (33, 32), (2, 1), (70, 9)]:
        Z = rng.standard_normal((m, n + 1))
        x, r = csk.ms_solve(gpu_colmajor(Z), n)
        xo, ro = oracle.sketch_solve(Z, n)
        err = np.linalg.norm(Z[:, :n] @ (host(x) - xo))
        check_le(err / np.linalg.norm(Z[:, n]), 1e-12, f"ms_solve {m}x{n} ||Z_A dx||/||z||")
        check_le(abs(r - ro) / np.linalg.norm(Z[:, n]), 1e-12, f"ms_solve {m}x{n} |d sk_resid|/||z||")


@pytest.mark.parametrize("kappa", [1e6, 1e12])
def test_ms_solve_ill_conditioned(solver_env, kappa):
    # Z1 = U diag(sigma) V^T with sigma log-spaced over [1/kappa, 1]; z = Z1 x* + noise.
    # Backward-stable solves agree in fitted values to O(u kappa ||r||) (Wedin; R16)
    m, n = 256, 128
    Z1 = synth.ill_conditioned(m, n, kappa, seed=11)
    z = synth.rhs(Z1, "hard", seed=11)
    Z = np.column_stack([Z1, z])
    x, r = csk.ms_solve(gpu_colmajor(Z), n)
    xo, ro = oracle.sketch_solve(Z, n)
    nz = np.linalg.norm(z)
    rr = ro / nz
    tol = max(1e-12, 64 * 2.2e-16 * kappa * rr)
    check_fitted(Z1, host(x) - xo, nz, tol)
    check_le(abs(r - ro) / nz, tol, "|d sk_resid| / ||z||")


def test_ms_solve_singular(solver_env):
    Z = np.zeros((10, 4))
    Z[:, 0] = 1.0
    Z[:, 3] = 1.0
    with pytest.raises(csk.CskError) as e:
        csk.ms_solve(gpu_colmajor(Z), 3)
    assert e.value.status == csk.csk.ESINGULAR


def test_ms_solve_async_matches_oracle_and_reports_status(solver_env):
    # the asynchronous form: same launches, the status and |R_nn| left on the device
    rng = np.random.default_rng(8)
    for m, n in [(128, 64), (256, 128), (40, 3), (512, 256)]:
        Z = rng.standard_normal((m, n + 1))
        x, st, r = csk.ms_solve_async(gpu_colmajor(Z), n)
        torch.cuda.synchronize()
        xo, ro = oracle.sketch_solve(Z, n)
        assert int(st.item()) == csk.csk.OK
        assert np.linalg.norm(Z[:, :n] @ (host(x) - xo)) <= 1e-12 * np.linalg.norm(Z[:, n]), (m, n)
        assert abs(float(r.item()) - ro) <= 1e-12 * np.linalg.norm(Z[:, n]), (m, n)
    Z = np.zeros((10, 4))
    Z[:, 0] = 1.0
    Z[:, 3] = 1.0
    _, st, _ = csk.ms_solve_async(gpu_colmajor(Z), 3)
    assert int(st.item()) == csk.csk.ESINGULAR
    with pytest.raises(csk.CskError) as e:   # the status must live on the device
        csk.ms_solve_async(gpu_colmajor(Z), 3, status=torch.zeros(1, dtype=torch.int32))
    assert e.value.status == csk.csk.EINVAL


@pytest.mark.parametrize("kappa", [1e2, 1e10])
@pytest.mark.parametrize("mode", ["easy", "hard", "consistent"])
def test_ms_lstsq_matches_oracle(kappa, mode):
    d, n = 1 << 15, 16
    k1, k2 = 2 * n * n, 2 * n
    A = synth.ill_conditioned(d, n, kappa, seed=4)
    b = synth.rhs(A, mode, seed=4)
    plan = csk.cs_plan(d, k1, 1)
    x, r = csk.ms_lstsq(plan, k2, gpu_colmajor(A), gpu_colmajor(b))
    xo, ro = oracle.ms_lstsq(A, b, k1, k2, seed=1)
    nb = np.linalg.norm(b)
    # R16: fitted values agree to 1e-8 relative; for kappa = 1e10 with a noisy b the
    # problem itself amplifies O(u) input rounding by kappa * ||r|| / ||b|| (Wedin), so
    # the bound is max(1e-8, 64 u kappa ||r|| / ||b||) (R16b)
    rr = oracle.residual_norm(A, b, xo) / nb
    tol = ls_tol(kappa, rr)                 # = 1e-8 for the consistent b and for kappa = 1e2
    if mode == "consistent" or kappa <= 1e2:
        assert tol == 1e-8
    check_fitted(A, host(x) - xo, nb, tol)
    check_le(abs(r - ro) / nb, tol, "|d sk_resid| / ||b||")   # |d ||r||| <= ||A dx||, same first-order bound


def test_ms_lstsq_host_inputs_streamed():
    d, n = 300000, 8
    k1, k2 = 2 * n * n, 2 * n
    A = synth.gaussian_matrix(d, n, seed=8)
    b = synth.rhs(A, "hard", seed=8)
    plan = csk.cs_plan(d, k1, 2)
    xd, rd = csk.ms_lstsq(plan, k2, gpu_colmajor(A), gpu_colmajor(b))
    At = torch.from_numpy(np.ascontiguousarray(A.T)).pin_memory().t()
    bt = torch.from_numpy(b).pin_memory()
    xh, rh = csk.ms_lstsq(plan, k2, At, bt)
    assert not xh.is_cuda
    xo, ro = oracle.ms_lstsq(A, b, k1, k2, seed=2)
    nb = np.linalg.norm(b)
    check_fitted(A, xh.numpy() - xo, nb, 1e-8)
    check_fitted(A, host(xd) - xo, nb, 1e-8)
    # pageable host memory works too
    xp, _ = csk.ms_lstsq(plan, k2, torch.from_numpy(np.ascontiguousarray(A.T)).t(), torch.from_numpy(b))
    check_fitted(A, xp.numpy() - xo, nb, 1e-8)


# -------------------------------------------------------- normal equations
def test_ne_lstsq_matches_oracle():
    d, n = 1 << 15, 16
    A = synth.ill_conditioned(d, n, 1e2, seed=2)
    b = synth.rhs(A, "easy", seed=2)
    xo = oracle.normal_eq(A, b)
    nb = np.linalg.norm(b)
    # b stored apart from A (SYRK + GEMV) and as column n of [A b] (one SYRK)
    x1 = host(csk.ne_lstsq(gpu_colmajor(A), gpu_colmajor(b)))
    Ab = gpu_colmajor(np.column_stack([A, b]))
    x2 = host(csk.ne_lstsq(Ab[:, :n], Ab[:, n]))
    for x in (x1, x2):
        check_fitted(A, x - xo, nb, 1e-8)


def test_ne_lstsq_breaks_down_at_kappa_1e10():
    # the normal equations fail for kappa(A) > 1e8 (ENOTPD or a useless x)
    d, n = 1 << 17, 16
    A = synth.ill_conditioned(d, n, 1e10, seed=3)
    b = synth.rhs(A, "consistent", seed=3)
    try:
        x = host(csk.ne_lstsq(gpu_colmajor(A), gpu_colmajor(b)))
    except csk.CskError as e:
        assert e.status == csk.csk.ENOTPD
        return
    assert oracle.residual_norm(A, b, x) / np.linalg.norm(b) > 1e-2


def test_profile_hooks_time_the_main_kernel():
    d, n, k1 = 1 << 16, 8, 64
    A = synth.gaussian_matrix(d, n, seed=2)
    plan = csk.cs_plan(d, k1, 1)
    Ad = gpu_colmajor(A)
    csk.profile_enable(True)
    for _ in range(3):
        csk.cs_apply(plan, Ad)
    ms, launches = csk.profile_read()
    csk.profile_enable(False)
    assert launches == 3 and ms > 0.0
    csk.cs_apply(plan, Ad)                    # disabled: nothing recorded
    assert csk.profile_read() == (0.0, 0)


# ------------------------------------------------ B32 shapes: odd widths, narrow rows, k1 up to 16384
@pytest.mark.parametrize("d,n,with_b,k1", [(100003, 64, True, 8192), (50000, 4, True, 2048), (40961, 5, False, 64),
                                           (9999, 64, True, 10240), (3000, 64, True, 16384), (100003, 32, False, 2048),
                                           (40000, 17, False, 512), (5000, 2, False, 64)])
def test_cs_apply_b32_shapes(d, n, with_b, k1):
    A = synth.gaussian_matrix(d, n, seed=3)
    b = synth.rhs(A, "hard", seed=3) if with_b else None
    plan = csk.cs_plan(d, k1, 7)
    h, s = oracle.codes(d, k1, 7)
    for variant in ("auto", "B"):
        _check_apply(plan, h, s, A, b, variant)
    Ai = synth.integer_matrix(d, n, seed=6)
    got = host(csk.cs_apply(plan, gpu_colmajor(Ai)))
    assert np.array_equal(got, oracle.cs_apply(h, s, Ai, k1))


@pytest.mark.parametrize("acc", ["1", "0"])
@pytest.mark.parametrize("d,n,with_b,k1,off", [(1 << 21, 64, True, 2048, 0), (300007, 40, False, 512, 0),
                                               (100003, 129, True, 1024, 0), (50001, 7, True, 4096, 1),
                                               (1 << 20, 256, True, 131072, 0), (70008, 65, True, 8192, 0),
                                               (4104, 3, False, 64, 0), (64008, 66, True, 4096, 8),
                                               (1 << 20, 8, True, 128, 0), (1 << 20, 16, False, 512, 8),
                                               (777777, 30, True, 1800, 0)])
def test_cs_apply_fp32_accumulation(monkeypatch, acc, d, n, with_b, k1, off):
    # fp32 input: fp32 sums in row-block copies of bounded bucket depth, combined in fp64 ("1", the
    # default: 64-row tiles, 32-B loads), or fp64 accumulation ("0"); both within 1e-5 * sum|terms|
    # (BASELINE.json).  off = 1 misaligns A by one float (no 32-B loads: the fp64-accumulating
    # 16-row kernel); off = 8 keeps 32-B alignment with an offset base; k1 = 131072 is chunk-major.
    monkeypatch.setenv("CSK_F32ACC", acc)
    A = synth.gaussian_matrix(d, n, seed=3, dtype=np.float32)
    b = synth.rhs(A.astype(np.float64), "easy", seed=3).astype(np.float32) if with_b else None
    plan = csk.cs_plan(d, k1, 4)
    h, s = oracle.codes(d, k1, 4)
    big = np.zeros((d + off, n), dtype=np.float32, order="F")
    big[off:] = A
    Ad = gpu_colmajor(big)[off:]
    bd = None if b is None else gpu_colmajor(b)
    exp, T = oracle.cs_apply(h, s, A, k1, b=b, with_abs=True)
    Ai = synth.integer_matrix(d, n, seed=6, dtype=np.float32)
    # "B" forces the bounded-depth copies even where the measured table picks X/T (tiny fp32 SA^T)
    for variant in ("auto", "B"):
        SA = host(csk.cs_apply(plan, Ad, b=bd, variant=variant))
        assert_within_T(SA, exp, T, 1e-5)
        got = host(csk.cs_apply(plan, gpu_colmajor(Ai), variant=variant))
        assert np.array_equal(got.astype(np.float64), oracle.cs_apply(h, s, Ai, k1))


# ------------------------------------------------ CSK_PLAN_HASH (codes hashed on the fly)
@pytest.mark.parametrize("d,n,with_b,k1,row0", [(100003, 64, True, 8192, 0), (4099, 100, False, 777, 5),
                                                (77777, 128, True, 4096, (1 << 33) + 3), (5000, 300, True, 65536, 1),
                                                (31, 3, False, 7, 2), (1 << 20, 20, True, 1 << 17, 0)])
def test_hash_plan_matches_oracle(d, n, with_b, k1, row0):
    # the on-the-fly kernel (wide rows, narrow chunk-major slices, ragged tails, unaligned row0)
    plan = csk.cs_plan(d, k1, 7, row0=row0, hash=True)
    h, s = oracle.codes(d, k1, 7, row0)
    A = synth.gaussian_matrix(d, n, seed=4)
    b = synth.rhs(A, "hard", seed=4) if with_b else None
    _check_apply(plan, h, s, A, b, "B")
    Ai = synth.integer_matrix(d, n, seed=8)
    got = host(csk.cs_apply(plan, gpu_colmajor(Ai)))
    assert np.array_equal(got, oracle.cs_apply(h, s, Ai, k1))


def test_hash_plan_materialises_codes_for_other_consumers():
    d, n, k1 = 20011, 9, 1000
    A = synth.integer_matrix(d, n, seed=2)
    h, s = oracle.codes(d, k1, 3, 11)
    exp = oracle.cs_apply(h, s, A, k1)
    for variant in ["L", "T", "S", "X", "auto"]:   # each a fresh hash plan: the first use builds the codes
        plan = csk.cs_plan(d, k1, 3, row0=11, hash=True)
        assert np.array_equal(host(csk.cs_apply(plan, gpu_colmajor(A), variant=variant)), exp)
    plan = csk.cs_plan(d, k1, 3, row0=11, hash=True)
    code, _, _ = plan.export()
    hh, ss = unpack(code)
    assert np.array_equal(hh, h) and np.array_equal(ss, s)
    # fp32 input and odd lda (no 16-B loads) also go through the stored codes
    plan = csk.cs_plan(d, k1, 3, row0=11, hash=True)
    got = host(csk.cs_apply(plan, gpu_colmajor(A.astype(np.float32))))
    assert np.array_equal(got.astype(np.float64), exp)


def test_hash_plan_ms_lstsq_matches_stored_codes():
    d, n, k2 = 1 << 16, 16, 32
    k1 = 2 * n * n
    A = synth.ill_conditioned(d, n, 1e6, seed=3)
    b = synth.rhs(A, "hard", seed=3)
    x0, r0 = csk.ms_lstsq(csk.cs_plan(d, k1, 5), k2, gpu_colmajor(A), gpu_colmajor(b))
    x1, r1 = csk.ms_lstsq(csk.cs_plan(d, k1, 5, hash=True), k2, gpu_colmajor(A), gpu_colmajor(b))
    # same codes; the reduction order is not deterministic, so within the LS tolerance (R16)
    nb = np.linalg.norm(b)
    check_fitted(A, host(x0) - host(x1), nb, 1e-8)
    assert abs(r0 - r1) <= 1e-8 * nb


# ------------------------------------------------ narrow B32 / fp32 instantiations (2-3 CTAs per SM)
@pytest.mark.parametrize("narrow", ["1", "0"])
@pytest.mark.parametrize("d,n,with_b,k1", [(300007, 1, True, 64), (262147, 8, True, 128), (131101, 16, False, 512),
                                           (200001, 17, True, 578), (150011, 24, True, 1152), (100003, 32, True, 2048),
                                           (90001, 33, True, 2178), (80021, 33, False, 999)])
def test_cs_apply_narrow_rows(monkeypatch, narrow, d, n, with_b, k1):
    # n + b <= 17 / 33 columns run the KJ = 9 / 17 kernels (CSK_B32_NARROW=0: the one-CTA kernel), fp64
    # within 1e-12 T and exact on integer A; fp32 within 1e-5 T (KJF = 5 / 9); ragged last tiles
    monkeypatch.setenv("CSK_B32_NARROW", narrow)
    plan = csk.cs_plan(d, k1, 11)
    h, s = oracle.codes(d, k1, 11)
    A = synth.gaussian_matrix(d, n, seed=7)
    b = synth.rhs(A, "easy", seed=7) if with_b else None
    _check_apply(plan, h, s, A, b, "B")
    Ai = synth.integer_matrix(d, n, seed=8)
    got = host(csk.cs_apply(plan, gpu_colmajor(Ai), variant="B"))
    assert np.array_equal(got, oracle.cs_apply(h, s, Ai, k1))
    _check_apply(plan, h, s, A.astype(np.float32), None if b is None else b.astype(np.float32), "B",
                 dtype=np.float32, rel=1e-5)


# ------------------------------------------------ spread SA^T copies (small k1)
@pytest.mark.parametrize("spread_kb", ["0", "256", "8192"])
@pytest.mark.parametrize("d,n,k1,with_b", [(200003, 8, 128, True), (100003, 20, 512, False), (70001, 33, 97, True)])
def test_cs_apply_spread_copies(monkeypatch, spread_kb, d, n, k1, with_b):
    # CTA c reduces into copy c mod S of a small SA^T and the copies are folded in fixed order: the
    # result is the same sum (within 1e-12 T; exact on integer A) for no copies, the default target
    # and one copy per CTA; also through ms_apply (the G-stage reads the folded copy 0)
    monkeypatch.setenv("CSK_SPREAD_KB", spread_kb)
    plan = csk.cs_plan(d, k1, 3)
    h, s = oracle.codes(d, k1, 3)
    A = synth.gaussian_matrix(d, n, seed=4)
    b = synth.rhs(A, "easy", seed=4) if with_b else None
    _check_apply(plan, h, s, A, b, "B")
    Ai = synth.integer_matrix(d, n, seed=5)
    got = host(csk.cs_apply(plan, gpu_colmajor(Ai), variant="B"))
    assert np.array_equal(got, oracle.cs_apply(h, s, Ai, k1))
    k2 = 2 * (n + 1)
    Z = host(csk.ms_apply(plan, k2, gpu_colmajor(A), b=None if b is None else gpu_colmajor(b)))
    Zo, Zabs = oracle.ms_apply(A, k1, k2, seed=3, b=b, with_abs=True)
    assert_within_T(Z, Zo, Zabs, 1e-12)
