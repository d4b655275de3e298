"""Test helpers (marshalling between numpy/oracle and torch/CUDA) and the parity-slack record.

Every tolerance check goes through ``record_slack(measured, tol)`` so the measured disagreement is
reported beside the bound it is tested against (conftest.py writes them all to
``gpurun_out/parity_slack.json`` at session end and prints a summary).
"""
import os

import numpy as np

SLACK = []


def record_slack(measured, tol, what=""):
    """Record one parity check: measured disagreement vs its tolerance (both in the same unit)."""
    test = os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]
    SLACK.append({"test": test, "what": what, "measured": float(measured), "tol": float(tol),
                  "ratio": float(measured) / float(tol) if tol else (0.0 if measured == 0 else float("inf"))})


def gpu_colmajor(a, device="cuda"):
    """numpy (d, n) -> torch CUDA tensor with column-major storage."""
    import torch
    a = np.asarray(a)
    if a.ndim == 1:
        return torch.from_numpy(np.ascontiguousarray(a)).to(device)
    t = torch.from_numpy(np.ascontiguousarray(a.T)).to(device)
    return t.t()


def host(t):
    """torch tensor -> numpy array (column-major 2-D tensors come back as (d, n))."""
    return t.detach().cpu().numpy()


def unpack(code):
    code = np.asarray(code).view(np.uint32)
    h = (code & 0x7FFFFFFF).astype(np.int32)
    s = np.where(code >> 31, -1, 1).astype(np.int8)
    return h, s


def assert_within_T(got, expect, T, rel):
    """|got - expect| <= rel * T elementwise (T = sum of |terms|); T == 0 entries must be exactly 0."""
    got = np.asarray(got, dtype=np.float64)
    err = np.abs(got - expect)
    bound = rel * T
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(T > 0, err / np.where(T > 0, T, 1.0), np.where(err > 0, np.inf, 0.0))
    record_slack(float(np.max(r)) if r.size else 0.0, rel, "max |got - exp| / T (elementwise)")
    bad = err > bound
    if bad.any():
        idx = np.argwhere(bad)[:5]
        raise AssertionError(f"{bad.sum()} entries exceed {rel}*T; first {idx.tolist()}: "
                             f"err={err[bad][:5]}, bound={bound[bad][:5]}")


U = 2.2e-16   # fp64 unit roundoff (rounded up), as used in the LS tolerances


def ls_tol(kappa, rr):
    """DESIGN.md R16/R16b: ||A (x_gpu - x_oracle)|| / ||b|| <= max(1e-8, 64 u kappa ||r|| / ||b||).
    For a consistent b (r = 0) and for well-conditioned problems this is BASELINE's 1e-8."""
    return max(1e-8, 64 * U * kappa * rr)


def check_fitted(A, dx, nb, tol, what="||A dx|| / ||b||"):
    """Fitted-value agreement of two LS solutions (R16), recorded beside its tolerance."""
    m = float(np.linalg.norm(A @ dx) / nb)
    record_slack(m, tol, what)
    assert m <= tol, f"{what} = {m:.3e} > {tol:.3e}"


def check_le(measured, tol, what):
    measured = float(measured)
    record_slack(measured, tol, what)
    assert measured <= tol, f"{what} = {measured:.3e} > {tol:.3e}"
