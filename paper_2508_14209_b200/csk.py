"""Thin ctypes binding over libcsk.so (include/csk.h).  Argument marshalling only:
every step of the path runs in the library's CUDA kernels.  There is no CPU
fallback -- loading fails loudly if the library is missing, and every call
that needs a GPU raises if CUDA is unavailable.

Tensors are torch tensors; matrices are column-major, i.e. shape (d, n) with
stride (1, lda) -- e.g. ``torch.empty((n, d)).t()``.  Vectors are contiguous.
Streams default to torch's current stream on the tensor's device.
"""
from __future__ import annotations

import ctypes
import os
import re
import threading

from . import _build

OK, EINVAL, ESHAPE, EDTYPE, ENOMEM, ECUDA, ENOTPD, ESINGULAR, EUNSUPPORTED = range(9)
F64, F32 = 0, 1
VAR_AUTO, VAR_ATOMIC_COL, VAR_ATOMIC_ROW, VAR_SMEM, VAR_SORTED, VAR_BULK_ROW, VAR_TMA_ROW = -1, 0, 1, 2, 3, 4, 5
VARIANTS = {"auto": VAR_AUTO, "L": VAR_ATOMIC_COL, "T": VAR_ATOMIC_ROW, "S": VAR_SMEM, "G": VAR_SORTED,
            "B": VAR_BULK_ROW, "X": VAR_TMA_ROW}
PLAN_SORT = 0x2
PLAN_HASH = 0x4

_lock = threading.Lock()
_lib = None


class CskError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: {_STATUS_NAMES.get(status, status)}: {detail}")
        self.status = status


_STATUS_NAMES = {OK: "CSK_OK", EINVAL: "CSK_EINVAL", ESHAPE: "CSK_ESHAPE", EDTYPE: "CSK_EDTYPE",
                 ENOMEM: "CSK_ENOMEM", ECUDA: "CSK_ECUDA", ENOTPD: "CSK_ENOTPD", ESINGULAR: "CSK_ESINGULAR",
                 EUNSUPPORTED: "CSK_EUNSUPPORTED"}


def header_symbols() -> list[str]:
    """Function names declared in include/csk.h (the boundary)."""
    hdr = os.path.join(_build.ROOT, "include", "csk.h")
    text = open(hdr).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b([a-z_][a-z0-9_]*)\s*\(", text)) - {"if", "sizeof"})


def lib():
    """Load libcsk.so (building it in-tree with nvcc if it is missing or stale)."""
    global _lib
    with _lock:
        if _lib is None:
            path = _build.LIB
            if _build.needs_build():
                path = _build.build()
            L = ctypes.CDLL(path)
            P, I64, U64, U32, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
            sigs = {
                "cs_plan": [I64, I64, U64, I64, U32, P, P],
                "cs_plan_from_arrays": [I64, I64, P, P, U32, P, P],
                "cs_plan_export": [P, P, P, P, P],
                "cs_plan_info": [P, P, P, P],
                "cs_apply": [P, I32, I64, P, I64, P, P, I64, I32, P],
                "ms_apply": [P, I64, I32, I64, P, I64, P, P, I64, P],
                "ms_solve": [I64, I64, P, I64, P, P, P],
                "ms_solve_async": [I64, I64, P, I64, P, P, P, P],
                "ms_lstsq": [P, I64, I64, P, I64, P, P, P, P],
                "ne_lstsq": [I64, I64, P, I64, P, P, P],
                "rc_lstsq": [P, I64, I64, P, I64, P, P, P, I64, P],
                "srht_apply": [I64, I64, I64, I64, U64, I64, P, I64, P, P, I64, P],
                "rc_r0": [I64, I64, P, I64, P, I64, P],
                "rc_gram": [I64, I64, P, I64, P, P, I64, P, I64, P],
                "rc_finish": [I64, P, I64, P, I64, P, P, I64, P],
                "gs_apply": [I64, I64, I64, U64, I64, P, I64, P, P, I64, P],
                "gs_lstsq": [I64, I64, U64, I64, P, I64, P, P, P, P],
                "cs_lstsq": [P, I64, P, I64, P, P, P, P],
                "msh_apply": [P, I64, I64, P, I64, P, P, I64, P],
                "msh_lstsq": [P, I64, I64, P, I64, P, P, P, P],
            }
            for name, argt in sigs.items():
                f = getattr(L, name)
                f.argtypes = argt
                f.restype = ctypes.c_int
            L.cs_plan_destroy.argtypes = [P]
            L.cs_plan_destroy.restype = None
            L.csk_status_str.argtypes = [ctypes.c_int]
            L.csk_status_str.restype = ctypes.c_char_p
            L.csk_last_error.restype = ctypes.c_char_p
            L.csk_launch_count.argtypes = [ctypes.c_int]
            L.csk_launch_count.restype = ctypes.c_uint64
            L.csk_version.restype = ctypes.c_char_p
            L.csk_profile_enable.argtypes = [ctypes.c_int]
            L.csk_profile_enable.restype = None
            L.csk_profile_read.argtypes = [P, P]
            L.csk_profile_read.restype = ctypes.c_int
            _lib = L
    return _lib


def _check(st: int, where: str):
    if st != OK:
        raise CskError(st, where, lib().csk_last_error().decode())


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2508_14209_b200 needs a CUDA GPU (no CPU fallback)")
    return torch


def _stream(stream, device=None):
    if stream is None:
        torch = _torch()
        return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _colmajor(t, name):
    """(pointer, ld) of a column-major (d, n) tensor; vectors have ld = len."""
    if t is None:
        return None, 0
    if t.dim() == 1:
        if t.stride(0) != 1 and t.shape[0] > 1:
            raise ValueError(f"{name} must be contiguous")
        return ctypes.c_void_p(t.data_ptr()), t.shape[0]
    if t.dim() != 2 or (t.stride(0) != 1 and t.shape[0] > 1):
        raise ValueError(f"{name} must be column-major: shape (d, n), stride (1, ld)")
    ld = t.stride(1) if t.shape[1] > 1 else t.shape[0]
    return ctypes.c_void_p(t.data_ptr()), max(ld, t.shape[0])


def _dtype_code(t):
    import torch
    if t.dtype == torch.float64:
        return F64
    if t.dtype == torch.float32:
        return F32
    raise TypeError(f"unsupported dtype {t.dtype}")


# ---------------------------------------------------------------- validation
# Every pointer handed to the library is checked here first (shape, dtype, device): the C side
# validates sizes and leading dimensions, but it cannot see how many elements a buffer holds.
def _need(t, name, dtype=None, rows=None, min_cols=None, cols=None, device=None, allow_host=False):
    import torch
    if t is None:
        raise ValueError(f"{name} is required")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if t.dtype not in (torch.float64, torch.float32):
        raise TypeError(f"{name}: unsupported dtype {t.dtype}")
    if not t.is_cuda and not allow_host:
        raise ValueError(f"{name} must be a CUDA tensor")
    if device is not None and t.is_cuda and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    r = t.shape[0]
    c = 1 if t.dim() == 1 else t.shape[1]
    if rows is not None and r != rows:
        raise ValueError(f"{name} has {r} rows, expected {rows}")
    if cols is not None and c != cols:
        raise ValueError(f"{name} has {c} columns, expected {cols}")
    if min_cols is not None and c < min_cols:
        raise ValueError(f"{name} has {c} columns, needs >= {min_cols}")
    return t


def _vec(t, name, n, dtype=None, device=None, allow_host=False):
    if t is None:
        raise ValueError(f"{name} is required")
    if t.dim() != 1:
        raise ValueError(f"{name} must be a vector")
    return _need(t, name, dtype=dtype, rows=n, device=device, allow_host=allow_host)


def _inputs(A, b, d, allow_host=False):
    """Validate [A b] against d rows: same dtype, same device; returns (ref tensor, n, ncols)."""
    if A is None and b is None:
        raise ValueError("A and b cannot both be None")
    ref = A if A is not None else b
    if A is not None:
        if A.dim() != 2:
            raise ValueError("A must be a (d, n) matrix")
        _need(A, "A", rows=d, allow_host=allow_host)
    if b is not None:
        _vec(b, "b", d, dtype=ref.dtype, allow_host=allow_host)
        if A is not None and b.is_cuda != A.is_cuda:
            raise ValueError("A and b must both be on the GPU or both on the host")
        if A is not None and A.is_cuda and b.device != A.device:
            raise ValueError("A and b must be on the same device")
    n = 0 if A is None else A.shape[1]
    return ref, n, n + (1 if b is not None else 0)


def launch_count(reset: bool = False) -> int:
    return int(lib().csk_launch_count(1 if reset else 0))


def profile_enable(on: bool = True):
    """Bracket every dominant cs_apply kernel launch with CUDA events (roofline timing)."""
    lib().csk_profile_enable(1 if on else 0)


def profile_read():
    """(summed kernel ms, number of bracketed launches) since profile_enable; clears them."""
    ms = ctypes.c_double()
    cnt = ctypes.c_uint64()
    _check(lib().csk_profile_read(ctypes.byref(ms), ctypes.byref(cnt)), "csk_profile_read")
    return ms.value, int(cnt.value)


class Plan:
    """Owning handle of a csk_plan_t (cs_plan / cs_plan_from_arrays)."""

    def __init__(self, handle: int, d: int, k1: int, row0: int, seed: int | None, sorted_: bool):
        self._h = ctypes.c_void_p(handle)
        self.d, self.k1, self.row0, self.seed, self.sorted = d, k1, row0, seed, sorted_

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h and self._h.value:
            lib().cs_plan_destroy(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def export(self, stream=None):
        """(code int32[d], offsets int64[k1+1] | None, perm int32[d] | None) as numpy arrays."""
        import numpy as np
        code = np.zeros(self.d, np.int32)
        offsets = np.zeros(self.k1 + 1, np.int64) if self.sorted else None
        perm = np.zeros(self.d, np.int32) if self.sorted else None
        ptr = lambda a: None if a is None else a.ctypes.data_as(ctypes.c_void_p)
        _check(lib().cs_plan_export(self._h, ptr(code), ptr(offsets), ptr(perm), _stream(stream)), "cs_plan_export")
        return code, offsets, perm


def cs_plan(d: int, k1: int, seed: int, row0: int = 0, sort: bool = False, stream=None, hash: bool = False) -> Plan:
    """hash=True: CSK_PLAN_HASH (no stored codes; the fp64 row-tile kernel hashes rows on the fly)."""
    _torch()
    h = ctypes.c_void_p()
    flags = (PLAN_SORT if sort else 0) | (PLAN_HASH if hash else 0)
    _check(lib().cs_plan(d, k1, seed, row0, flags, _stream(stream), ctypes.byref(h)), "cs_plan")
    return Plan(h.value, d, k1, row0, seed, sort)


def cs_plan_from_arrays(h, s, k1: int, sort: bool = False, stream=None) -> Plan:
    import numpy as np
    _torch()
    h = np.ascontiguousarray(h, dtype=np.int32)
    s = np.ascontiguousarray(s, dtype=np.int8)
    out = ctypes.c_void_p()
    _check(lib().cs_plan_from_arrays(h.shape[0], k1, h.ctypes.data_as(ctypes.c_void_p),
                                     s.ctypes.data_as(ctypes.c_void_p), PLAN_SORT if sort else 0, _stream(stream),
                                     ctypes.byref(out)), "cs_plan_from_arrays")
    return Plan(out.value, h.shape[0], k1, 0, None, sort)


def cs_apply(plan: Plan, A, b=None, SA=None, variant="auto", stream=None):
    """SA = S [A b] (k1 x ncols column-major, allocated if not given)."""
    torch = _torch()
    ref, n, ncols = _inputs(A, b, plan.d)
    if SA is None:
        SA = torch.empty((ncols, plan.k1), dtype=ref.dtype, device=ref.device).t()
    _need(SA, "SA", dtype=ref.dtype, rows=plan.k1, min_cols=ncols, device=ref.device)
    pA, lda = _colmajor(A, "A") if A is not None else (None, plan.d)
    pb, _ = _colmajor(b, "b")
    pS, ldsa = _colmajor(SA, "SA")
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    _check(lib().cs_apply(plan.handle, _dtype_code(ref), n, pA, lda, pb, pS, ldsa, v, _stream(stream, ref.device)),
           "cs_apply")
    return SA


def ms_apply(plan: Plan, k2: int, A, b=None, Z=None, stream=None):
    """Z = G S [A b] (k2 x ncols column-major).  A, b may be CPU tensors (streamed)."""
    torch = _torch()
    ref, n, ncols = _inputs(A, b, plan.d, allow_host=True)
    dev = ref.device if ref.is_cuda else torch.device("cuda", torch.cuda.current_device())
    if Z is None:
        Z = torch.empty((ncols, k2), dtype=ref.dtype, device=dev).t()
    _need(Z, "Z", dtype=ref.dtype, rows=k2, min_cols=ncols, device=dev)
    pA, lda = _colmajor(A, "A") if A is not None else (None, plan.d)
    pb, _ = _colmajor(b, "b")
    pZ, ldz = _colmajor(Z, "Z")
    _check(lib().ms_apply(plan.handle, k2, _dtype_code(ref), n, pA, lda, pb, pZ, ldz, _stream(stream, dev)),
           "ms_apply")
    return Z


def ms_solve(Z, n: int, x=None, stream=None):
    """(x, sketched residual) from the augmented sketch Z = [GSA | GSb] (k2 x (n+1))."""
    torch = _torch()
    _need(Z, "Z", dtype=torch.float64, min_cols=n + 1)
    if x is None:
        x = torch.empty(n, dtype=torch.float64, device=Z.device)
    _vec(x, "x", n, dtype=torch.float64, device=Z.device)
    pZ, ldz = _colmajor(Z, "Z")
    r = ctypes.c_double()
    _check(lib().ms_solve(Z.shape[0], n, pZ, ldz, ctypes.c_void_p(x.data_ptr()), ctypes.byref(r),
                          _stream(stream, Z.device)), "ms_solve")
    return x, r.value


def ms_solve_async(Z, n: int, x=None, status=None, sk_resid=None, stream=None):
    """ms_solve without the host sync: (x, status, sk_resid) as device tensors (int32, fp64)."""
    torch = _torch()
    _need(Z, "Z", dtype=torch.float64, min_cols=n + 1)
    if x is None:
        x = torch.empty(n, dtype=torch.float64, device=Z.device)
    _vec(x, "x", n, dtype=torch.float64, device=Z.device)
    if status is None:
        status = torch.empty(1, dtype=torch.int32, device=Z.device)
    if sk_resid is None:
        sk_resid = torch.empty(1, dtype=torch.float64, device=Z.device)
    if status.dtype != torch.int32 or status.numel() < 1:
        raise TypeError("status must be an int32 tensor with >= 1 element")
    if sk_resid.dtype != torch.float64 or sk_resid.numel() < 1:
        raise TypeError("sk_resid must be a float64 tensor with >= 1 element")
    pZ, ldz = _colmajor(Z, "Z")
    _check(lib().ms_solve_async(Z.shape[0], n, pZ, ldz, ctypes.c_void_p(x.data_ptr()),
                                ctypes.c_void_p(sk_resid.data_ptr()), ctypes.c_void_p(status.data_ptr()),
                                _stream(stream, Z.device)), "ms_solve_async")
    return x, status, sk_resid


def ms_lstsq(plan: Plan, k2: int, A, b, x=None, stream=None):
    """Multisketched sketch-and-solve: (x, sketched residual).  A, b, x may be CPU tensors."""
    torch = _torch()
    _need(A, "A", dtype=torch.float64, rows=plan.d, allow_host=True)
    _inputs(A, b, plan.d, allow_host=True)
    n = A.shape[1]
    dev = A.device if A.is_cuda else torch.device("cuda", torch.cuda.current_device())
    if x is None:
        x = torch.empty(n, dtype=torch.float64, device=dev if A.is_cuda else "cpu")
    _vec(x, "x", n, dtype=torch.float64, allow_host=True)
    pA, lda = _colmajor(A, "A")
    pb, _ = _colmajor(b, "b")
    r = ctypes.c_double()
    _check(lib().ms_lstsq(plan.handle, k2, n, pA, lda, pb, ctypes.c_void_p(x.data_ptr()), ctypes.byref(r),
                          _stream(stream, dev)), "ms_lstsq")
    return x, r.value


def ne_lstsq(A, b, x=None, stream=None):
    """Normal-equations least squares (cuBLAS Gram + Cholesky); raises CskError(ENOTPD) on breakdown."""
    torch = _torch()
    _need(A, "A", dtype=torch.float64)
    d, n = A.shape
    _inputs(A, b, d)
    if x is None:
        x = torch.empty(n, dtype=torch.float64, device=A.device)
    _vec(x, "x", n, dtype=torch.float64, device=A.device)
    pA, lda = _colmajor(A, "A")
    pb, _ = _colmajor(b, "b")
    _check(lib().ne_lstsq(d, n, pA, lda, pb, ctypes.c_void_p(x.data_ptr()), _stream(stream, A.device)), "ne_lstsq")
    return x


def rc_lstsq(plan: Plan, k2: int, A, b, x=None, want_R: bool = False, stream=None):
    """rand_cholQR least squares (Alg 5): the true LS solution x (and R = R1 R0 if want_R)."""
    torch = _torch()
    _need(A, "A", dtype=torch.float64, rows=plan.d)
    d, n = A.shape
    _inputs(A, b, d)
    if x is None:
        x = torch.empty(n, dtype=torch.float64, device=A.device)
    _vec(x, "x", n, dtype=torch.float64, device=A.device)
    R = torch.empty((n, n), dtype=torch.float64, device=A.device).t() if want_R else None
    pA, lda = _colmajor(A, "A")
    pb, _ = _colmajor(b, "b")
    pR, ldr = _colmajor(R, "R") if want_R else (None, n)
    _check(lib().rc_lstsq(plan.handle, k2, n, pA, lda, pb, ctypes.c_void_p(x.data_ptr()), pR, ldr,
                          _stream(stream, A.device)), "rc_lstsq")
    return (x, R) if want_R else x


def srht_apply(A, k: int, seed: int, b=None, Y=None, dglob: int | None = None, row0: int = 0, stream=None):
    """SRHT Y = k^-1/2 P H D [A b] (k x ncols) of the rows [row0, row0 + d) of a dglob-row matrix."""
    torch = _torch()
    d = A.shape[0] if A is not None else b.shape[0]
    ref, n, ncols = _inputs(A, b, d)
    _need(ref, "A" if A is not None else "b", dtype=torch.float64)
    dev = ref.device
    if Y is None:
        Y = torch.empty((ncols, k), dtype=torch.float64, device=dev).t()
    _need(Y, "Y", dtype=torch.float64, rows=k, min_cols=ncols, device=dev)
    pA, lda = _colmajor(A, "A") if A is not None else (None, max(d, 1))
    pb, _ = _colmajor(b, "b")
    pY, ldy = _colmajor(Y, "Y")
    _check(lib().srht_apply(d, dglob if dglob is not None else d, row0, k, seed, n, pA, lda, pb, pY, ldy,
                            _stream(stream, dev)), "srht_apply")
    return Y


def gs_apply(A, k: int, seed: int, b=None, Z=None, row0: int = 0, stream=None):
    """Gaussian sketch Z = G [A b] (k x ncols), G k x d ~ N(0, 1/k) generated by row chunks."""
    torch = _torch()
    d = A.shape[0] if A is not None else b.shape[0]
    ref, n, ncols = _inputs(A, b, d)
    _need(ref, "A" if A is not None else "b", dtype=torch.float64)
    dev = ref.device
    if Z is None:
        Z = torch.empty((ncols, k), dtype=torch.float64, device=dev).t()
    _need(Z, "Z", dtype=torch.float64, rows=k, min_cols=ncols, device=dev)
    pA, lda = _colmajor(A, "A") if A is not None else (None, max(d, 1))
    pb, _ = _colmajor(b, "b")
    pZ, ldz = _colmajor(Z, "Z")
    _check(lib().gs_apply(d, row0, k, seed, n, pA, lda, pb, pZ, ldz, _stream(stream, dev)), "gs_apply")
    return Z


def _solve_out(n, dev, x):
    torch = _torch()
    x = torch.empty(n, dtype=torch.float64, device=dev) if x is None else x
    return _vec(x, "x", n, dtype=torch.float64, device=dev)


def _ls_inputs(A, b, d=None):
    import torch
    _need(A, "A", dtype=torch.float64, rows=d)
    if A.dim() != 2:
        raise ValueError("A must be a (d, n) matrix")
    _inputs(A, b, A.shape[0])
    if b is None:
        raise ValueError("b is required")


def gs_lstsq(A, b, k: int, seed: int, x=None, stream=None):
    """Gaussian sketch-and-solve: (x, sketched residual)."""
    _ls_inputs(A, b)
    d, n = A.shape
    x = _solve_out(n, A.device, x)
    pA, lda = _colmajor(A, "A")
    pb, _ = _colmajor(b, "b")
    r = ctypes.c_double()
    _check(lib().gs_lstsq(d, k, seed, n, pA, lda, pb, ctypes.c_void_p(x.data_ptr()), ctypes.byref(r),
                          _stream(stream, A.device)), "gs_lstsq")
    return x, r.value


def cs_lstsq(plan: Plan, A, b, x=None, stream=None):
    """CountSketch-only sketch-and-solve (GEQRF of the k1 x (n+1) sketch): (x, sketched residual)."""
    _ls_inputs(A, b, plan.d)
    n = A.shape[1]
    x = _solve_out(n, A.device, x)
    pA, lda = _colmajor(A, "A")
    pb, _ = _colmajor(b, "b")
    r = ctypes.c_double()
    _check(lib().cs_lstsq(plan.handle, n, pA, lda, pb, ctypes.c_void_p(x.data_ptr()), ctypes.byref(r),
                          _stream(stream, A.device)), "cs_lstsq")
    return x, r.value


def msh_apply(plan: Plan, k2: int, A, b=None, Z=None, stream=None):
    """Count+SRHT multisketch Z = SRHT_k2 (S1 [A b])."""
    torch = _torch()
    _need(A, "A", dtype=torch.float64, rows=plan.d)
    _, n, ncols = _inputs(A, b, plan.d)
    if Z is None:
        Z = torch.empty((ncols, k2), dtype=torch.float64, device=A.device).t()
    _need(Z, "Z", dtype=torch.float64, rows=k2, min_cols=ncols, device=A.device)
    pA, lda = _colmajor(A, "A")
    pb, _ = _colmajor(b, "b")
    pZ, ldz = _colmajor(Z, "Z")
    _check(lib().msh_apply(plan.handle, k2, n, pA, lda, pb, pZ, ldz, _stream(stream, A.device)), "msh_apply")
    return Z


def msh_lstsq(plan: Plan, k2: int, A, b, x=None, stream=None):
    """Count+SRHT multisketch sketch-and-solve: (x, sketched residual)."""
    _ls_inputs(A, b, plan.d)
    n = A.shape[1]
    x = _solve_out(n, A.device, x)
    pA, lda = _colmajor(A, "A")
    pb, _ = _colmajor(b, "b")
    r = ctypes.c_double()
    _check(lib().msh_lstsq(plan.handle, k2, n, pA, lda, pb, ctypes.c_void_p(x.data_ptr()), ctypes.byref(r),
                           _stream(stream, A.device)), "msh_lstsq")
    return x, r.value


def rc_r0(Z, n: int, stream=None):
    """R0 (n x n, upper) of the Householder QR of the (all-reduced) sketch Z = [GSA | GSb]."""
    torch = _torch()
    _need(Z, "Z", dtype=torch.float64, min_cols=n + 1)
    R0 = torch.zeros((n, n), dtype=torch.float64, device=Z.device).t()
    pZ, ldz = _colmajor(Z, "Z")
    _check(lib().rc_r0(Z.shape[0], n, pZ, ldz, ctypes.c_void_p(R0.data_ptr()), n, _stream(stream, Z.device)), "rc_r0")
    return R0


def rc_gram(A, b, R0, stream=None):
    """[Q0^T Q0 | Q0^T b] ((n+1) x (n+1); upper triangle + column n) over this block's rows, Q0 = A R0^-1."""
    torch = _torch()
    _ls_inputs(A, b)
    d, n = A.shape
    _need(R0, "R0", dtype=torch.float64, rows=n, cols=n, device=A.device)
    C = torch.zeros((n + 1, n + 1), dtype=torch.float64, device=A.device).t()
    pA, lda = _colmajor(A, "A")
    pb, _ = _colmajor(b, "b")
    pR, ldr0 = _colmajor(R0, "R0")
    _check(lib().rc_gram(d, n, pA, lda, pb, pR, ldr0, ctypes.c_void_p(C.data_ptr()), n + 1,
                         _stream(stream, A.device)), "rc_gram")
    return C


def rc_finish(C, R0, want_R: bool = False, stream=None):
    """x (and R = R1 R0) from the (all-reduced) C and R0."""
    torch = _torch()
    n = R0.shape[0]
    _need(R0, "R0", dtype=torch.float64, rows=n, cols=n)
    _need(C, "C", dtype=torch.float64, rows=n + 1, min_cols=n + 1, device=R0.device)
    x = torch.empty(n, dtype=torch.float64, device=C.device)
    R = torch.empty((n, n), dtype=torch.float64, device=C.device).t() if want_R else None
    pC, ldc = _colmajor(C, "C")
    pR0, ldr0 = _colmajor(R0, "R0")
    pR, ldr = _colmajor(R, "R") if want_R else (None, n)
    _check(lib().rc_finish(n, pC, ldc, pR0, ldr0, ctypes.c_void_p(x.data_ptr()), pR, ldr, _stream(stream, C.device)),
           "rc_finish")
    return (x, R) if want_R else x
