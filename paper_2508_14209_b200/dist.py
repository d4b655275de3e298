"""Row-partitioned multi-GPU driver (section 7).

A is distributed block-row over p ranks.  Rank g owns global rows
[row0_g, row0_g + d_g) and builds its plan with ``row0 = row0_g``, so its codes are
the slice of the ONE global CountSketch (globally indexed hash, R3):
C = [C^(1) ... C^(p)] and CA = sum_g C^(g) A^(g).  G is drawn from the
same seed on every rank -- the "cast it to each process" of P:L377 without a
broadcast -- so G_ms C A = sum_g G_ms C^(g) A^(g).  The only exchange
is one SUM all-reduce of the k2 x (n+1) partial Z (NCCL over NVLink), after which
every rank solves the small problem redundantly (no broadcast of x).

``local_apply`` / ``local_solve`` default to the CUDA library; they are injectable
so the host-side logic (partitioning, reduction, solve placement) is testable with
the gloo backend on CPU.  There is no CPU default.
"""
from __future__ import annotations


def row_block(d_global: int, world: int, rank: int):
    """(row0, rows) of rank's contiguous block; the last blocks absorb the remainder."""
    if not (0 <= rank < world) or d_global < world:
        raise ValueError(f"cannot split {d_global} rows over {world} ranks")
    r0 = rank * d_global // world
    r1 = (rank + 1) * d_global // world
    return r0, r1 - r0


def _cuda_apply(A_local, b_local, row0, k1, k2, seed):
    from . import csk
    plan = csk.cs_plan(A_local.shape[0], k1, seed, row0=row0)
    return csk.ms_apply(plan, k2, A_local, b=b_local)


def _cuda_solve(Z, n):
    from . import csk
    return csk.ms_solve(Z, n)


def ms_lstsq_distributed(A_local, b_local, row0: int, k1: int, k2: int, seed: int, group=None,
                         local_apply=None, local_solve=None):
    """Multisketch sketch-and-solve on a row-partitioned [A b]; returns (x, sketched residual)
    on every rank.  Collective over ``group`` (all ranks must call it)."""
    import torch.distributed as dist
    apply_ = local_apply or _cuda_apply
    solve_ = local_solve or _cuda_solve
    Z = apply_(A_local, b_local, row0, k1, k2, seed)       # k2 x (n+1) partial: G C^(g) [A^(g) b^(g)]
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        if Z.t().is_contiguous():                          # column-major: reduce the storage in place
            dist.all_reduce(Z.t(), op=dist.ReduceOp.SUM, group=group)
        else:
            Z = Z.contiguous()
            dist.all_reduce(Z, op=dist.ReduceOp.SUM, group=group)
    return solve_(Z, A_local.shape[1])


def _all_reduce_colmajor(M, group):
    """SUM all-reduce of a column-major (m, k) tensor in place (or of a contiguous copy)."""
    import torch.distributed as dist
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return M
    if M.t().is_contiguous():
        dist.all_reduce(M.t(), op=dist.ReduceOp.SUM, group=group)
        return M
    M = M.contiguous()
    dist.all_reduce(M, op=dist.ReduceOp.SUM, group=group)
    return M


def _cuda_rc_r0(Z, n):
    from . import csk
    return csk.rc_r0(Z, n)


def _cuda_rc_gram(A_local, b_local, R0):
    from . import csk
    return csk.rc_gram(A_local, b_local, R0)


def _cuda_rc_finish(C, R0):
    from . import csk
    return csk.rc_finish(C, R0)


def rc_lstsq_distributed(A_local, b_local, row0: int, k1: int, k2: int, seed: int, group=None,
                         local_apply=None, local_r0=None, local_gram=None, local_finish=None):
    """rand_cholQR least squares (Alg 5) on a row-partitioned [A b]: the exact LS
    solution x on every rank.  Two SUM all-reduces: the k2 x (n+1) sketch Z (as in
    ms_lstsq_distributed) and the (n+1) x (n+1) Gram [Q0^T Q0 | Q0^T b] of the preconditioned
    blocks Q0^(g) = A^(g) R0^-1 (every rank holds the same R0).  Collective over ``group``."""
    apply_ = local_apply or _cuda_apply
    r0_ = local_r0 or _cuda_rc_r0
    gram_ = local_gram or _cuda_rc_gram
    finish_ = local_finish or _cuda_rc_finish
    n = A_local.shape[1]
    Z = _all_reduce_colmajor(apply_(A_local, b_local, row0, k1, k2, seed), group)   # lines 1: G S [A b]
    R0 = r0_(Z, n)                                                                  # line 2 (redundant per rank)
    C = _all_reduce_colmajor(gram_(A_local, b_local, R0), group)                    # lines 3-4
    return finish_(C, R0)                                                           # lines 5-8
