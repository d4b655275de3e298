"""Test helpers (marshalling between numpy/oracle and torch/CUDA)."""
import numpy as np


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
    bad = err > bound
    if bad.any():
        idx = np.argwhere(bad)[:5]
        raise AssertionError(f"{bad.sum()} entries exceed {rel}*T; first {idx.tolist()}: "
                             f"err={err[bad][:5]}, bound={bound[bad][:5]}")
