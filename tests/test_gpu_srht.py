"""GPU parity of srht_apply (SRHT, Def P:L164-173; one-pass blocked FWHT) against the oracle.

Tolerance: every output is k^-1/2 sum_i +-a_i, so |dY| <= 1e-12 * T with T = k^-1/2 sum_i |a_i|
(the |S||A| of the SRHT; the FWHT's own bound is ~log2(d) u T).  Integer-valued A with k a power
of 4 (so k^-1/2 is a power of two) is bit-exact, including across row partitions.
"""
import numpy as np
import pytest

import oracle
import synth
from tests._util import gpu_colmajor, host

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2508_14209_b200 as csk  # noqa: E402


def _T(A, k):
    return np.abs(A).sum(axis=0)[None, :] / np.sqrt(k)


@pytest.mark.parametrize("d,n,k", [(1 << 12, 3, 16), (1 << 14, 5, 256), (1 << 16, 33, 300), (1 << 15, 2, 700),
                                   (1 << 13, 1, 1024), (1024, 4, 40), (8, 2, 5), (1, 1, 3)])
def test_srht_matches_oracle(d, n, k):
    A = synth.gaussian_matrix(d, n, seed=3)
    b = synth.rhs(A, "hard", seed=3)
    Y = host(csk.srht_apply(gpu_colmajor(A), k, seed=9, b=gpu_colmajor(b)))
    Yo = oracle.srht_apply(A, k, seed=9, b=b)
    Ab = np.column_stack([A, b])
    assert Y.shape == (k, n + 1)
    assert np.all(np.abs(Y - Yo) <= 1e-12 * _T(Ab, k))


@pytest.mark.parametrize("d,k", [(1 << 14, 64), (1 << 16, 256), (512, 16)])
def test_srht_integer_exact(d, k):
    A = synth.integer_matrix(d, 6, seed=4)
    Y = host(csk.srht_apply(gpu_colmajor(A), k, seed=2))
    assert np.array_equal(Y, oracle.srht_apply(A, k, seed=2))


@pytest.mark.parametrize("p", [2, 4, 8])
def test_srht_row_partition_sums_to_global(p):
    d, n, k = 1 << 16, 4, 256
    A = synth.integer_matrix(d, n, seed=5)
    full = host(csk.srht_apply(gpu_colmajor(A), k, seed=7))
    acc = np.zeros_like(full)
    db = d // p
    for g in range(p):
        acc += host(csk.srht_apply(gpu_colmajor(A[g * db:(g + 1) * db]), k, seed=7, dglob=d, row0=g * db))
    assert np.array_equal(acc, full)
    assert np.array_equal(full, oracle.srht_apply(A, k, seed=7))


def test_srht_only_b_and_padded_ld():
    d, n, k = 1 << 13, 3, 32
    A = synth.gaussian_matrix(d, n, seed=6)
    big = np.zeros((d + 6, n), order="F")
    big[:d] = A
    Ad = gpu_colmajor(big)[:d]
    Y = torch.full((n + 5, k), 3.0, dtype=torch.float64, device="cuda").t()[:, :n]   # ldy = k, ragged alloc
    csk.srht_apply(Ad, k, seed=1, Y=Y)
    Yo = oracle.srht_apply(A, k, seed=1)
    assert np.all(np.abs(host(Y) - Yo) <= 1e-12 * _T(A, k))
    yb = host(csk.srht_apply(None, k, seed=1, b=gpu_colmajor(A[:, 0])))
    assert np.all(np.abs(yb[:, 0] - Yo[:, 0]) <= 1e-12 * _T(A[:, :1], k)[0])


def test_srht_errors():
    A = gpu_colmajor(synth.gaussian_matrix(3000, 2, seed=1))
    with pytest.raises(csk.CskError) as e:
        csk.srht_apply(A, 16, seed=1)                      # d not a power of two
    assert e.value.status == csk.csk.ESHAPE
    A2 = gpu_colmajor(synth.gaussian_matrix(1 << 13, 2, seed=1))
    with pytest.raises(csk.CskError) as e:
        csk.srht_apply(A2[:6000], 16, seed=1, dglob=1 << 14, row0=100)   # unaligned block
    assert e.value.status == csk.csk.ESHAPE
    with pytest.raises(csk.CskError) as e:
        csk.srht_apply(A2, 2000, seed=1)
    assert e.value.status == csk.csk.EUNSUPPORTED


@pytest.mark.parametrize("path", ["warp", "r64"])
@pytest.mark.parametrize("lda_pad", [0, 1])
def test_srht_kernel_paths(monkeypatch, path, lda_pad):
    # k = 130: the TMA-fed warp kernel (16-B aligned columns) or the register warp kernel (odd lda);
    # "r64" forces the radix-64 CTA kernel (the default for k > 512)
    if path == "r64":
        monkeypatch.setenv("CSK_SRHT_KERNEL", "2")
    d, n, k = 1 << 15, 7, 130
    A = synth.gaussian_matrix(d, n, seed=8)
    big = np.zeros((d + lda_pad, n), order="F")
    big[:d] = A
    Y = host(csk.srht_apply(gpu_colmajor(big)[:d], k, seed=5))
    Yo = oracle.srht_apply(A, k, seed=5)
    assert np.all(np.abs(Y - Yo) <= 1e-12 * _T(A, k))
