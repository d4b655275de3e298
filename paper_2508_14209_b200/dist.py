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
