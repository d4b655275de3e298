"""Column-block / row-block parallel driver over the UNCHANGED oracle (test infrastructure).

Nothing here does arithmetic of the method: every number comes from an oracle function
(oracle.codes, oracle.cs_apply, oracle.gauss, oracle.gemm_comp, oracle.sketch_solve) called on a
slice of the problem, and the slices are independent by definition:

* the CountSketch and the G-stage act column by column (SA[:, c] = S A[:, c], Z[:, c] = G SA[:, c],
  Eq 2), so a column block is the same loop the oracle runs for those columns,
  in the same order -- the results are bit-identical to one oracle call on the whole matrix;
* the codes are a function of the global row index (R3), so row blocks with their row0
  are slices of the same code array.

ctypes releases the GIL inside the oracle's C functions, so a thread pool runs the blocks on all
host cores.  Used by the full-size parity tests and bench.py's cpu_baseline (all-core leg).
"""
from __future__ import annotations

import concurrent.futures as cf
import os

import numpy as np

from . import codes as _codes
from . import cs_apply as _cs_apply
from . import gauss as _gauss
from . import gemm_comp as _gemm_comp
from . import sketch_solve as _sketch_solve


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _col_blocks(ncols: int, threads: int):
    nb = max(1, min(threads, ncols))
    edges = np.linspace(0, ncols, nb + 1).astype(int)
    return [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a]


def codes(d: int, k1: int, seed: int, row0: int = 0, threads: int | None = None):
    """oracle.codes over row blocks (each block its own row0): identical to one call."""
    threads = threads or host_threads()
    h = np.empty(d, dtype=np.int32)
    s = np.empty(d, dtype=np.int8)
    edges = np.linspace(0, d, max(1, min(threads, d // 4096 + 1)) + 1).astype(int)

    def run(i):
        a, b = int(edges[i]), int(edges[i + 1])
        if b > a:
            h[a:b], s[a:b] = _codes(b - a, k1, seed, row0 + a)

    with cf.ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, range(len(edges) - 1)))
    return h, s


def cs_apply(h, s, A, k1: int, b=None, with_abs: bool = False, threads: int | None = None):
    """oracle.cs_apply on column blocks of [A b] (A column-major d x n, b optional)."""
    threads = threads or host_threads()
    n = 0 if A is None else A.shape[1]
    ncols = n + (b is not None)
    d = A.shape[0] if A is not None else len(b)
    SA = np.zeros((k1, ncols), dtype=np.float64, order="F")
    T = np.zeros((k1, ncols), dtype=np.float64, order="F") if with_abs else None

    def run(blk):
        a, e = blk
        a_hi = min(e, n)
        Ab = A[:, a:a_hi] if a < n else np.zeros((d, 0), dtype=A.dtype if A is not None else b.dtype)
        bb = b if e > n else None
        r = _cs_apply(h, s, Ab, k1, b=bb, with_abs=with_abs)
        if with_abs:
            SA[:, a:e], T[:, a:e] = r
        else:
            SA[:, a:e] = r

    with cf.ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, _col_blocks(ncols, threads)))
    return (SA, T) if with_abs else SA


def gemm(G, Y, Yabs=None, threads: int | None = None):
    """oracle.gemm_comp on column blocks of Y (Z[:, c] = G Y[:, c])."""
    threads = threads or host_threads()
    m, ncols = G.shape[0], Y.shape[1]
    Z = np.zeros((m, ncols), dtype=np.float64, order="F")
    Zabs = np.zeros((m, ncols), dtype=np.float64, order="F") if Yabs is not None else None

    def run(blk):
        a, e = blk
        if Yabs is None:
            Z[:, a:e] = _gemm_comp(G, Y[:, a:e])
        else:
            Z[:, a:e], Zabs[:, a:e] = _gemm_comp(G, Y[:, a:e], Yabs[:, a:e])

    with cf.ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, _col_blocks(ncols, threads)))
    return Z if Yabs is None else (Z, Zabs)


def ms_apply(A, k1: int, k2: int, seed: int, b=None, row0: int = 0, with_abs: bool = False,
             threads: int | None = None):
    """oracle.ms_apply with its codes, CountSketch and G-stage run in blocks (identical result)."""
    d = A.shape[0]
    h, s = codes(d, k1, seed, row0, threads)
    SA, T = cs_apply(h, s, A, k1, b=b, with_abs=True, threads=threads)
    G = _gauss(k2, k1, seed)
    return gemm(G, SA, T if with_abs else None, threads)


def ms_lstsq(A, b, k1: int, k2: int, seed: int, threads: int | None = None):
    """oracle.ms_lstsq (Alg 1 with S = G S1) with the data-parallel steps in blocks."""
    Z = ms_apply(A, k1, k2, seed, b=b, threads=threads)
    return _sketch_solve(Z, A.shape[1])
