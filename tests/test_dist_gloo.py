"""Host logic of the row-partitioned multi-GPU path, world_size 2 on CPU (gloo).

The per-rank compute is injected (the oracle's row0-offset multisketch), so this
checks the partitioning, the SUM all-reduce of the k2 x (n+1) partial and the
redundant solve placement against the single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
import scipy.linalg

from paper_2508_14209_b200.dist import ms_lstsq_distributed, rc_lstsq_distributed, row_block

D, N, K1, K2, SEED = 9001, 6, 72, 14, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_apply(A_local, b_local, row0, k1, k2, seed):
    Z = oracle.ms_apply(A_local.numpy(), k1, k2, seed, b=b_local.numpy(), row0=row0)
    return torch.from_numpy(np.ascontiguousarray(Z.T)).t()       # column-major like the CUDA path


def _oracle_solve(Z, n):
    return oracle.sketch_solve(Z.numpy(), n)


def _worker(rank, world, port, integer, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A = synth.integer_matrix(D, N, seed=5) if integer else synth.gaussian_matrix(D, N, seed=5)
    b = synth.rhs(A, "hard", seed=5)
    r0, rows = row_block(D, world, rank)
    A_local = torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows].T)).t()
    b_local = torch.from_numpy(b[r0:r0 + rows].copy())
    x, r = ms_lstsq_distributed(A_local, b_local, r0, K1, K2, SEED, local_apply=_oracle_apply,
                                local_solve=_oracle_solve)
    q.put((rank, np.asarray(x), r))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_distributed_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, False, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = synth.gaussian_matrix(D, N, seed=5)
    b = synth.rhs(A, "hard", seed=5)
    x1, r1 = oracle.ms_lstsq(A, b, K1, K2, SEED)
    nb = np.linalg.norm(b)
    for _, x, r in res:
        # the reduction changes only the summation order: fitted values agree to 1e-12
        assert np.linalg.norm(A @ (x - x1)) / nb <= 1e-12
        assert abs(r - r1) <= 1e-12 * nb
    # every rank holds the same solution
    assert np.array_equal(res[0][1], res[1][1])


def test_row_block_partition():
    for d, p in [(10, 1), (10, 3), (9001, 7), (1 << 27, 8)]:
        blocks = [row_block(d, p, g) for g in range(p)]
        assert blocks[0][0] == 0
        for (r0, n0), (r1, _) in zip(blocks, blocks[1:]):
            assert r0 + n0 == r1
        assert blocks[-1][0] + blocks[-1][1] == d
        assert max(n for _, n in blocks) - min(n for _, n in blocks) <= 1
    with pytest.raises(ValueError):
        row_block(3, 4, 0)


# ---------------------------------------------------------------- rand_cholQR over ranks
# Injected per-rank phases (numpy/scipy on CPU, written here from Alg 5's lines); the reference
# is the single-process oracle rand_cholqr_lstsq on the whole matrix.
def _np_r0(Z, n):
    R = oracle.householder_qr(Z.numpy())          # line 2: qr of [Y | z]; R[:n,:n] is Y's R
    return torch.from_numpy(np.asfortranarray(R[:n, :n]))


def _np_gram(A_local, b_local, R0):
    A = A_local.numpy()
    Q0 = scipy.linalg.solve_triangular(R0.numpy(), A.T, trans="T", lower=False).T   # line 3: Q0 R0 = A
    n = A.shape[1]
    C = np.zeros((n + 1, n + 1))
    C[:n, :n] = Q0.T @ Q0                                                           # line 4
    C[:n, n] = Q0.T @ b_local.numpy()
    return torch.from_numpy(np.asfortranarray(C))


def _np_finish(C, R0):
    C, R0 = C.numpy(), R0.numpy()
    n = R0.shape[0]
    R1 = np.linalg.cholesky(C[:n, :n]).T                                            # line 5 (upper)
    y = scipy.linalg.solve_triangular(R1, C[:n, n], trans="T", lower=False)         # line 7
    return scipy.linalg.solve_triangular(R1 @ R0, y, lower=False)                   # lines 6, 8


def _rc_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A = synth.ill_conditioned(D, N, 1e6, seed=6)
    b = synth.rhs(A, "hard", seed=6)
    r0, rows = row_block(D, world, rank)
    A_local = torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows].T)).t()
    b_local = torch.from_numpy(b[r0:r0 + rows].copy())
    x = rc_lstsq_distributed(A_local, b_local, r0, K1, K2, SEED, local_apply=_oracle_apply, local_r0=_np_r0,
                             local_gram=_np_gram, local_finish=_np_finish)
    q.put((rank, np.asarray(x)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_rc_distributed_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = synth.ill_conditioned(D, N, 1e6, seed=6)
    b = synth.rhs(A, "hard", seed=6)
    xo = oracle.rand_cholqr_lstsq(A, b, oracle.ms_apply(A, K1, K2, SEED))
    xs, *_ = np.linalg.lstsq(A, b, rcond=None)
    nb = np.linalg.norm(b)
    r = np.linalg.norm(b - A @ xs)
    for _, x in res:
        # the exact LS solution (no distortion), within the LS perturbation bound of the oracle's
        assert np.linalg.norm(A @ (x - xo)) <= 64 * 2.2e-16 * (nb + 1e6 * r)
        assert np.linalg.norm(A @ (x - xs)) <= 64 * 2.2e-16 * (nb + 1e6 * r)
    assert all(np.array_equal(res[0][1], x) for _, x in res)
