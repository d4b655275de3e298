"""Full-size parity: BASELINE.json's configs C2, C3, C4 and C5 through the C-ABI, in the launch
configuration bench.py times (cs_apply / ms_apply on a contiguous column-major [A b]), against the
oracle on the same bytes.

* C2 (d=2^24, n=64 + b, k1=8192, k2=128) and C4 (d=2^23, n=128 + b, k1=32768, k2=256, kappa=1e10):
  SA elementwise within 1e-12 * T, Z within 1e-12 * |G| T, and the C4 least-squares solution within
  DESIGN.md R16b of the oracle's; C2 in fp32 within 1e-5 * T (the fp32 copies path).
* C3 (d=2^22, n=256 + b, k1=131072, k2=512): a column subset that spans every chunk boundary of the
  chunk-major layout (the CountSketch and the G-stage are column-separable, Eq 2).
* C5 (d=2^27, n=64 + b: 8.7e9 elements, past 2^31): integer-valued A, row-partitioned plans
  p in {1, 2, 4, 8} summed on the device are bit-identical to each other and to the oracle,
  which is streamed over row blocks (codes by global row, R3).

The oracle runs through oracle/harness.py (column blocks / row blocks over all host cores; the blocks
are the oracle's own loops, bit-identical to one call).
"""
import concurrent.futures as cf

import numpy as np
import pytest

import oracle
from oracle import harness
import synth
from tests._util import assert_within_T, check_fitted, check_le, host, ls_tol, record_slack, unpack

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2508_14209_b200 as csk  # noqa: E402

SEED, DATA = 1, 2


def _free():
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def _host_colmajor(t):
    """(d, n) column-major CUDA tensor -> Fortran-ordered numpy array (no reorder on the host)."""
    return t.cpu().numpy()


def _full(d, n, k1, k2, kappa=None, check_ls=False):
    if kappa is None:
        buf = synth.gaussian_matrix_torch(d, n + 1, seed=DATA)
    else:
        buf = synth.colmajor_empty(torch, d, n + 1, torch.float64, "cuda")
        buf[:, :n] = synth.ill_conditioned_torch(d, n, kappa, seed=DATA)
        buf[:, n] = synth.rhs_torch(buf[:, :n], "easy", seed=DATA)
    A, b = buf[:, :n], buf[:, n]
    plan = csk.cs_plan(d, k1, SEED)
    SA = csk.cs_apply(plan, A, b=b)
    Z = csk.ms_apply(plan, k2, A, b=b)
    x = csk.ms_lstsq(plan, k2, A, b)[0] if check_ls else None
    code, _, _ = plan.export()
    Ah = _host_colmajor(buf)
    del buf, A, b
    _free()
    h, s = harness.codes(d, k1, SEED)
    hg, sg = unpack(code)
    assert np.array_equal(hg, h) and np.array_equal(sg, s), "codes differ at full size"
    SAo, T = harness.cs_apply(h, s, Ah[:, :n], k1, b=Ah[:, n], with_abs=True)
    assert_within_T(host(SA), SAo, T, 1e-12)
    G = oracle.gauss(k2, k1, SEED)
    Zo, Zabs = harness.gemm(G, SAo, T)
    assert_within_T(host(Z), Zo, Zabs, 1e-12)
    if check_ls:
        xo, _ = oracle.sketch_solve(Zo, n)
        bh = Ah[:, n]
        nb = np.linalg.norm(bh)
        rr = float(np.linalg.norm(bh - Ah[:, :n] @ xo)) / nb
        check_fitted(Ah[:, :n], host(x) - xo, nb, ls_tol(kappa or 1.0, rr), "C4 full size ||A dx||/||b||")


def test_c2_full_size():
    _full(1 << 24, 64, 8192, 128)


def test_c2_full_size_fp32():
    # C2's fp32 form (BASELINE: "also fp32"): the bounded-depth fp32 copies summed in fp64 (R12) within
    # 1e-5 * T of the exact fp64 sums of the same fp32 values, and the multisketch Z within 1e-5 |G| T
    d, n, k1, k2 = 1 << 24, 64, 8192, 128
    buf = synth.gaussian_matrix_torch(d, n + 1, seed=DATA)
    b32 = synth.colmajor_empty(torch, d, n + 1, torch.float32, "cuda")
    b32.copy_(buf)
    del buf
    _free()
    A, b = b32[:, :n], b32[:, n]
    plan = csk.cs_plan(d, k1, SEED)
    SA = host(csk.cs_apply(plan, A, b=b))
    Z = host(csk.ms_apply(plan, k2, A, b=b))
    assert SA.dtype == np.float32 and Z.dtype == np.float32
    Ah = _host_colmajor(b32).astype(np.float64)
    del b32, A, b
    _free()
    h, s = harness.codes(d, k1, SEED)
    SAo, T = harness.cs_apply(h, s, Ah[:, :n], k1, b=Ah[:, n], with_abs=True)
    assert_within_T(SA.astype(np.float64), SAo, T, 1e-5)
    G = oracle.gauss(k2, k1, SEED)
    Zo, Zabs = harness.gemm(G, SAo, T)
    assert_within_T(Z.astype(np.float64), Zo, Zabs, 1e-5)


def test_c4_full_size_with_least_squares():
    _full(1 << 23, 128, 32768, 256, kappa=1e10, check_ls=True)


def test_c3_full_size_column_subset():
    d, n, k1, k2 = 1 << 22, 256, 131072, 512
    buf = synth.gaussian_matrix_torch(d, n + 1, seed=DATA)
    A, b = buf[:, :n], buf[:, n]
    plan = csk.cs_plan(d, k1, SEED)
    SA = host(csk.cs_apply(plan, A, b=b))
    Z = host(csk.ms_apply(plan, k2, A, b=b))
    # both sides of every chunk boundary of the chunk-major layout (52-column chunks) and b
    cols = [0, 1, 51, 52, 103, 104, 155, 156, 207, 208, 255, 256]
    sub = _host_colmajor(buf[:, cols])
    del buf, A, b
    _free()
    h, s = harness.codes(d, k1, SEED)
    SAo, T = harness.cs_apply(h, s, sub, k1, with_abs=True)
    assert_within_T(SA[:, cols], SAo, T, 1e-12)
    G = oracle.gauss(k2, k1, SEED)
    Zo, Zabs = harness.gemm(G, SAo, T)
    assert_within_T(Z[:, cols], Zo, Zabs, 1e-12)


def test_c5_integer_partitions_bit_exact_past_2_31_elements():
    d, n, k1 = 1 << 27, 64, 8192
    assert d * (n + 1) > 1 << 33
    buf = synth.colmajor_empty(torch, d, n + 1, torch.float64, "cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(1234)
    for c in range(n + 1):
        buf[:, c] = torch.randint(-8, 9, (d,), generator=g, device="cuda", dtype=torch.float64)
    A, b = buf[:, :n], buf[:, n]
    results = {}
    for p in (1, 2, 4, 8):
        acc = torch.zeros((n + 1, k1), dtype=torch.float64, device="cuda").t()
        edges = np.linspace(0, d, p + 1).astype(np.int64)
        for r0, r1 in zip(edges[:-1], edges[1:]):
            r0, r1 = int(r0), int(r1)
            plan = csk.cs_plan(r1 - r0, k1, SEED, row0=r0)
            acc += csk.cs_apply(plan, A[r0:r1], b=b[r0:r1])   # views with lda = d (offsets past 2^31)
            plan.close()
        results[p] = host(acc)
    for p in (2, 4, 8):
        assert np.array_equal(results[p], results[1]), f"p={p} differs from p=1"
    # the oracle, streamed in row blocks of the global matrix (exact integer sums in any order)
    blk = 1 << 23
    nthreads = min(8, harness.host_threads())

    def oracle_block(r0):
        Ah = _host_colmajor(buf[r0:r0 + blk])
        h, s = oracle.codes(blk, k1, SEED, r0)
        return oracle.cs_apply(h, s, Ah[:, :n], k1, b=Ah[:, n])

    SAo = np.zeros((k1, n + 1))
    with cf.ThreadPoolExecutor(nthreads) as ex:
        for part in ex.map(oracle_block, range(0, d, blk)):
            SAo += part
    record_slack(float(np.abs(results[1] - SAo).max()), 0.0, "C5 integer SA, bit-exact")
    assert np.array_equal(results[1], SAo)
    del buf, A, b
    _free()
