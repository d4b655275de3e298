"""CPU oracle for the hot path of arXiv 2508.14209 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The
product package ``paper_2508_14209_b200`` never imports it, and the two share
no code (the only shared module is ``synth``, the seeded input generators,
which holds none of the method's arithmetic).

The arithmetic lives in ``oracle/oracle.c`` (plain C loops, fp64, every
function citing the PAPER.md passage it follows); this module only builds it
with gcc and marshals numpy arrays through ctypes.

Functions and the passage each follows (P:Lx = PAPER.md line x):
  philox4x32_10   counter-based hash (Reading R1; P:L226 cuRAND)
  codes           Def 3 via the documented hash (Reading R3)
  count_sort      stable counting sort of rows by bucket (north_star form 1)
  cs_apply        Eq 2 / Alg 2, Neumaier-compensated
  gauss           N(0, 1/k2) Gaussian stage, Box-Muller (Reading R4)
  gemm_comp       Z = G Y, compensated dots
  householder_qr  economy QR (Alg 1 line 2)
  sketch_solve    Alg 1 lines 2-3 on [SA | Sb]
  ms_lstsq        the whole multisketch sketch-and-solve (Alg 1 with S = G S1)
  normal_eq       normal equations, ENOTPD on a non-positive pivot
  residual_norm   ||b - Ax||
  rand_cholqr_lstsq  rand_cholQR least squares, Alg 5, in the paper's order
  srht_draws      the SRHT's D signs and sampled rows (Readings R16-R17)
  fwht_rad4       Alg 3 radix-4 FWHT
  srht_apply      SRHT S = k^-1/2 P H D (Def) applied to [A b]
No function here is "parity unpinned"; each pin is listed in oracle.c's header.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared", "-std=c11"]
_lock = threading.Lock()
_lib = None

OK, EINVAL, ENOTPD, ESINGULAR = 0, 1, 6, 7


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"oracle {what} failed with status {status}")
        self.status = status


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (called by __graft_entry__.build())."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *_CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB_PATH)
            P = ctypes.c_void_p
            I64 = ctypes.c_int64
            lib.or_philox4x32_10.argtypes = [P, P, P]
            lib.or_codes.argtypes = [I64, I64, ctypes.c_uint64, I64, P, P]
            lib.or_count_sort.argtypes = [I64, I64, P, P, P]
            lib.or_cs_apply.argtypes = [I64, I64, I64, P, P, P, I64, P, ctypes.c_int, P, I64, P]
            lib.or_gauss.argtypes = [I64, I64, ctypes.c_uint64, P, I64]
            lib.or_gemm_comp.argtypes = [I64, I64, I64, P, I64, P, I64, P, I64, P, P]
            lib.or_householder_qr.argtypes = [I64, I64, P, I64, P, I64]
            lib.or_sketch_solve.argtypes = [I64, I64, P, I64, P, P]
            lib.or_normal_eq.argtypes = [I64, I64, P, I64, P, P]
            lib.or_residual_norm.argtypes = [I64, I64, P, I64, P, P]
            lib.or_residual_norm.restype = ctypes.c_double
            lib.or_rand_cholqr_lstsq.argtypes = [I64, I64, P, I64, P, P, I64, I64, P, P, I64]
            lib.or_srht_draws.argtypes = [I64, I64, ctypes.c_uint64, P, P]
            lib.or_fwht_rad4.argtypes = [I64, P]
            lib.or_srht_apply.argtypes = [I64, I64, I64, ctypes.c_uint64, P, I64, P, P, I64]
            _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _check(st: int, what: str):
    if st != OK:
        raise OracleError(st, what)


def _fortran(a, dtype):
    return np.asfortranarray(np.asarray(a, dtype=dtype))


# ---------------------------------------------------------------------------
def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    assert c.shape == (4,) and k.shape == (2,)
    out = np.zeros(4, dtype=np.uint32)
    _load().or_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def codes(d: int, k1: int, seed: int, row0: int = 0):
    """(h, s): bucket int32[d] in [0,k1), sign int8[d] in {-1,+1} of global rows row0..row0+d-1."""
    h = np.zeros(d, dtype=np.int32)
    s = np.zeros(d, dtype=np.int8)
    _check(_load().or_codes(d, k1, seed, row0, _ptr(h), _ptr(s)), "codes")
    return h, s


def count_sort(h: np.ndarray, k1: int):
    h = np.ascontiguousarray(h, dtype=np.int32)
    offsets = np.zeros(k1 + 1, dtype=np.int64)
    perm = np.zeros(h.shape[0], dtype=np.int32)
    _check(_load().or_count_sort(h.shape[0], k1, _ptr(h), _ptr(offsets), _ptr(perm)), "count_sort")
    return offsets, perm


def cs_apply(h, s, A, k1: int, b=None, with_abs: bool = False):
    """SA (k1 x ncols, fp64, column-major) for A d x n (fp64 or fp32) and optional b.

    Returns SA, or (SA, T) with T = |S||[A b]| (sum of |terms|) if with_abs."""
    h = np.ascontiguousarray(h, dtype=np.int32)
    s = np.ascontiguousarray(s, dtype=np.int8)
    A = np.asarray(A)
    is_f32 = A.dtype == np.float32
    dt = np.float32 if is_f32 else np.float64
    if A.ndim == 1:
        A = A[:, None]
    A = _fortran(A, dt)
    d, n = A.shape
    bb = None if b is None else np.ascontiguousarray(b, dtype=dt)
    ncols = n + (1 if bb is not None else 0)
    SA = np.zeros((k1, ncols), dtype=np.float64, order="F")
    T = np.zeros((k1, ncols), dtype=np.float64, order="F") if with_abs else None
    _check(_load().or_cs_apply(d, n, k1, _ptr(h), _ptr(s), _ptr(A), max(d, 1), _ptr(bb), int(is_f32),
                               _ptr(SA), k1, _ptr(T)), "cs_apply")
    return (SA, T) if with_abs else SA


def gauss(k2: int, k1: int, seed: int) -> np.ndarray:
    G = np.zeros((k2, k1), dtype=np.float64, order="F")
    _check(_load().or_gauss(k2, k1, seed, _ptr(G), k2), "gauss")
    return G


def gemm_comp(G, Y, Yabs=None):
    G = _fortran(G, np.float64)
    Y = _fortran(Y, np.float64)
    m, k = G.shape
    k2_, n = Y.shape
    assert k == k2_
    Z = np.zeros((m, n), dtype=np.float64, order="F")
    Zabs = None
    Ya = None
    if Yabs is not None:
        Ya = _fortran(Yabs, np.float64)
        Zabs = np.zeros((m, n), dtype=np.float64, order="F")
    _check(_load().or_gemm_comp(m, n, k, _ptr(G), m, _ptr(Y), k, _ptr(Z), m, _ptr(Ya), _ptr(Zabs)), "gemm")
    return Z if Yabs is None else (Z, Zabs)


def householder_qr(W):
    """R factor (LAPACK sign convention) of the economy QR of W (m x nc)."""
    W = np.array(W, dtype=np.float64, order="F", copy=True)
    m, nc = W.shape
    R = np.zeros((nc, nc), dtype=np.float64, order="F")
    _check(_load().or_householder_qr(m, nc, _ptr(W), m, _ptr(R), nc), "householder_qr")
    return R


def sketch_solve(Zaug, n: int):
    """x, sketched residual |R[n,n]| from the augmented sketch [SA | Sb] (m x (n+1))."""
    Z = np.array(Zaug, dtype=np.float64, order="F", copy=True)
    m = Z.shape[0]
    assert Z.shape[1] == n + 1
    x = np.zeros(n, dtype=np.float64)
    r = np.zeros(1, dtype=np.float64)
    _check(_load().or_sketch_solve(m, n, _ptr(Z), m, _ptr(x), _ptr(r)), "sketch_solve")
    return x, float(r[0])


def ms_apply(A, k1: int, k2: int, seed: int, b=None, row0: int = 0, with_abs: bool = False):
    """Multisketch Z = G S [A b] (Count-Gauss) for rows row0.. of the global sketch."""
    A2 = np.asarray(A)
    d = A2.shape[0]
    h, s = codes(d, k1, seed, row0)
    SA, T = cs_apply(h, s, A2, k1, b=b, with_abs=True)
    G = gauss(k2, k1, seed)
    if with_abs:
        return gemm_comp(G, SA, T)
    return gemm_comp(G, SA)


def ms_lstsq(A, b, k1: int, k2: int, seed: int):
    """Oracle of the multisketched sketch-and-solve (Alg 1 with S = G S1): x, sketched residual."""
    A2 = np.asarray(A, dtype=np.float64)
    Z = ms_apply(A2, k1, k2, seed, b=b)
    return sketch_solve(Z, A2.shape[1])


def normal_eq(A, b):
    A = _fortran(A, np.float64)
    d, n = A.shape
    bb = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(n, dtype=np.float64)
    _check(_load().or_normal_eq(d, n, _ptr(A), d, _ptr(bb), _ptr(x)), "normal_eq")
    return x


def residual_norm(A, b, x) -> float:
    A = _fortran(A, np.float64)
    d, n = A.shape
    bb = np.ascontiguousarray(b, dtype=np.float64)
    xx = np.ascontiguousarray(x, dtype=np.float64)
    return float(_load().or_residual_norm(d, n, _ptr(A), d, _ptr(bb), _ptr(xx)))


def rand_cholqr_lstsq(A, b, Y, return_R: bool = False):
    """rand_cholQR least squares (Alg 5) given the sketch Y = S A (k x n)."""
    A = _fortran(A, np.float64)
    d, n = A.shape
    Yf = _fortran(Y, np.float64)
    k = Yf.shape[0]
    assert Yf.shape[1] == n
    bb = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(n, dtype=np.float64)
    R = np.zeros((n, n), dtype=np.float64, order="F")
    _check(_load().or_rand_cholqr_lstsq(d, n, _ptr(A), d, _ptr(bb), _ptr(Yf), k, k, _ptr(x), _ptr(R), n),
           "rand_cholqr_lstsq")
    return (x, R) if return_R else x


def srht_draws(d: int, k: int, seed: int):
    """(D signs int8[d], sampled rows int64[k]) of the SRHT."""
    D = np.zeros(d, dtype=np.int8)
    p = np.zeros(k, dtype=np.int64)
    _check(_load().or_srht_draws(d, k, seed, _ptr(D), _ptr(p)), "srht_draws")
    return D, p


def fwht_rad4(a) -> np.ndarray:
    v = np.array(a, dtype=np.float64, copy=True)
    _check(_load().or_fwht_rad4(v.shape[0], _ptr(v)), "fwht_rad4")
    return v


def srht_apply(A, k: int, seed: int, b=None) -> np.ndarray:
    """Y = k^-1/2 P H D [A b] (k x ncols)."""
    A = _fortran(A, np.float64)
    if A.ndim == 1:
        A = A.reshape(-1, 1, order="F")
    d, n = A.shape
    bb = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
    Y = np.zeros((k, n + (b is not None)), dtype=np.float64, order="F")
    _check(_load().or_srht_apply(d, n, k, seed, _ptr(A), d, _ptr(bb), _ptr(Y), k), "srht_apply")
    return Y
