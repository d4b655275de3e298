"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds none of the method's arithmetic (no hash, no sketch, no
solve): it only draws the matrices A and right-hand sides b that both sides
consume as *bytes*.  The recipe is stated in DESIGN.md ("Input recipe"):

* Gaussian A: i.i.d. N(0,1) entries ("we fix a random matrix A").
* Integer A: i.i.d. uniform integers in [lo, hi] (exactness tests).
* Ill-conditioned A (Reading R9, "fixed kappa(A) = 10^2"):
  A = sqrt(d) U diag(sigma) V^T, U = Q of a d x n Gaussian, V = Q of an
  n x n Gaussian, sigma_i = kappa^{-(i-1)/(n-1)} (geometric spectrum).
* b = A e + eta, e = ones: consistent (eta = 0), easy
  (eta ~ N(0, 0.01)), hard (eta ~ N(3, 2)).

Host (numpy) generators feed the parity tests at sizes the oracle finishes;
device (torch) generators feed full-size runs, whose bytes are copied to the
host for sampled oracle checks.  Matrices are column-major: numpy arrays in
Fortran order, torch tensors of shape (d, n) with strides (1, d).
Seeds: data seed 2 by default; streams 2 Gaussian A, 3 integer A, 4 eta, 5 U/V.
"""
from __future__ import annotations

import math

import numpy as np

STREAM_GAUSS_A = 2
STREAM_INT_A = 3
STREAM_NOISE = 4
STREAM_UV = 5
NOISE = {"consistent": (0.0, 0.0), "easy": (0.0, 0.01), "hard": (3.0, 2.0)}


def _rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(seed), int(stream)]))


def singular_values(n: int, kappa: float) -> np.ndarray:
    if n == 1:
        return np.ones(1)
    return kappa ** (-np.arange(n, dtype=np.float64) / (n - 1))


# ----------------------------------------------------------------- host side
def gaussian_matrix(d: int, n: int, seed: int = 2, dtype=np.float64) -> np.ndarray:
    a = _rng(seed, STREAM_GAUSS_A).standard_normal((n, d)).astype(dtype)
    return np.asfortranarray(a.T)


def integer_matrix(d: int, n: int, seed: int = 2, lo: int = -8, hi: int = 8, dtype=np.float64) -> np.ndarray:
    a = _rng(seed, STREAM_INT_A).integers(lo, hi + 1, size=(n, d)).astype(dtype)
    return np.asfortranarray(a.T)


def ill_conditioned(d: int, n: int, kappa: float, seed: int = 2) -> np.ndarray:
    g = _rng(seed, STREAM_UV)
    U, _ = np.linalg.qr(g.standard_normal((d, n)))
    V, _ = np.linalg.qr(g.standard_normal((n, n)))
    A = math.sqrt(d) * (U * singular_values(n, kappa)[None, :]) @ V.T
    return np.asfortranarray(A)


def rhs(A: np.ndarray, mode: str = "easy", seed: int = 2) -> np.ndarray:
    mu, var = NOISE[mode]
    b = A @ np.ones(A.shape[1])
    if var > 0.0:
        b = b + _rng(seed, STREAM_NOISE).normal(mu, math.sqrt(var), size=A.shape[0])
    return np.ascontiguousarray(b)


# --------------------------------------------------------------- device side
def _torch_gen(torch, seed: int, stream: int, device):
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) * 1_000_003 + int(stream))
    return g


def colmajor_empty(torch, d: int, n: int, dtype, device):
    """Uninitialised (d, n) tensor in column-major storage (lda = d)."""
    return torch.empty((n, d), dtype=dtype, device=device).t()


def gaussian_matrix_torch(d: int, n: int, seed: int = 2, dtype=None, device="cuda"):
    import torch
    dtype = dtype or torch.float64
    g = _torch_gen(torch, seed, STREAM_GAUSS_A, device)
    return torch.randn((n, d), dtype=dtype, device=device, generator=g).t()


def ill_conditioned_torch(d: int, n: int, kappa: float, seed: int = 2, device="cuda"):
    import torch
    g = _torch_gen(torch, seed, STREAM_UV, device)
    U = torch.linalg.qr(torch.randn((n, d), dtype=torch.float64, device=device, generator=g).t())[0]
    V = torch.linalg.qr(torch.randn((n, n), dtype=torch.float64, device=device, generator=g))[0]
    sig = torch.as_tensor(singular_values(n, kappa), dtype=torch.float64, device=device)
    B = (V * sig[None, :]).t() * math.sqrt(d)          # diag(sigma) V^T scaled, n x n
    At = torch.matmul(B.t(), U.t()).contiguous()       # (U B)^T, n x d row-major
    del U
    return At.t()                                       # d x n column-major


def rhs_torch(A, mode: str = "easy", seed: int = 2):
    import torch
    mu, var = NOISE[mode]
    b = A.sum(dim=1).contiguous()     # A e
    if var > 0.0:
        g = _torch_gen(torch, seed, STREAM_NOISE, A.device)
        b += mu + math.sqrt(var) * torch.randn(b.shape, dtype=b.dtype, device=A.device, generator=g)
    return b


# ------------------------------------------------- row-partitioned device inputs (multi-GPU bench)
def row_block_size(d_global: int) -> int:
    """Rows per generator block of a d_global-row matrix: a function of the global shape only, so
    every row partition (any world size dividing d_global / block) sees the same global matrix."""
    return max(1, min(1 << 22, d_global // 8))


def gaussian_rows_torch(d_global: int, row0: int, rows: int, ncols: int, seed: int = 2, device="cuda",
                        out=None):
    """Rows [row0, row0 + rows) of the d_global x ncols Gaussian matrix whose row block q (of
    row_block_size rows) is drawn from generator (seed, q): identical bytes for any partition."""
    import torch
    blk = row_block_size(d_global)
    if out is None:
        out = colmajor_empty(torch, rows, ncols, torch.float64, device)
    q0, q1 = row0 // blk, (row0 + rows - 1) // blk
    for q in range(q0, q1 + 1):
        g = _torch_gen(torch, seed * 7919 + q, STREAM_GAUSS_A, device)
        nb = min(blk, d_global - q * blk)
        block = torch.randn((ncols, nb), dtype=torch.float64, device=device, generator=g).t()
        a, e = max(row0, q * blk), min(row0 + rows, q * blk + nb)
        out[a - row0:e - row0] = block[a - q * blk:e - q * blk]
        del block
    return out


def noise_rows_torch(d_global: int, row0: int, rows: int, mode: str = "easy", seed: int = 2, device="cuda"):
    """eta of b = A e + eta for rows [row0, row0 + rows), drawn per global row block like the matrix."""
    import torch
    mu, var = NOISE[mode]
    eta = torch.zeros(rows, dtype=torch.float64, device=device)
    if var == 0.0:
        return eta
    blk = row_block_size(d_global)
    q0, q1 = row0 // blk, (row0 + rows - 1) // blk
    for q in range(q0, q1 + 1):
        g = _torch_gen(torch, seed * 7919 + q, STREAM_NOISE, device)
        nb = min(blk, d_global - q * blk)
        block = mu + math.sqrt(var) * torch.randn(nb, dtype=torch.float64, device=device, generator=g)
        a, e = max(row0, q * blk), min(row0 + rows, q * blk + nb)
        eta[a - row0:e - row0] = block[a - q * blk:e - q * blk]
    return eta
