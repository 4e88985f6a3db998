"""Row-sharded RGS-GMRES / Arnoldi (gmres(comm=...)) on two ranks sharing cuda:0.

gloo on CUDA tensors (host-staged, no kernel waits on another process) runs
the same code path the NCCL multi-GPU run does: per-rank row blocks of the
operator, all-gathered SpMV inputs, sharded sketches with one k-vector
all-reduce each, replicated LS and Givens, all-reduced norms."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N = 24


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    import paper_2011_05090_b200 as sg
    from paper_2011_05090_b200.workloads import convdiff3d, rhs_gaussian
    rp, ci, va = convdiff3d(N)
    A = sg.SparseMatrix(n=N ** 3, row_ptr=rp, col_idx=ci, values=va)
    return A, rhs_gaussian(A.n, 2), sg.make_sketch(sg.SketchKind.PSRHT, 200, A.n, 0)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2011_05090_b200 as sg
    from paper_2011_05090_b200.distributed import TorchComm
    comm = TorchComm()
    A, b, th = _problem()
    r64 = sg.gmres(A, b, m=60, theta=th, policy=sg.UNIFIED64, tol=1e-9, comm=comm)
    rmx = sg.gmres(A, b, m=60, theta=th, policy=sg.MIXED32_64, tol=1e-6, comm=comm)
    rr = sg.gmres_restarted(A, b, th, sg.UNIFIED64, restart=25, max_iters=200, tol=1e-8,
                            comm=comm)
    dec = sg.arnoldi(A, b, 20, theta=th, policy=sg.UNIFIED64, comm=comm)
    # the halo window (default) and the all-gather give the SpMV the same x:
    # bit-identical solves
    import paper_2011_05090_b200.krylov as kr
    assert kr._HALO
    kr._HALO = False
    g64 = sg.gmres(A, b, m=60, theta=th, policy=sg.UNIFIED64, tol=1e-9, comm=comm)
    glg = sg.gmres(A, b, m=40, theta=th, policy=sg.MIXED32_64, tol=1e-6, comm=comm, lagged=True)
    kr._HALO = True
    hlg = sg.gmres(A, b, m=40, theta=th, policy=sg.MIXED32_64, tol=1e-6, comm=comm, lagged=True)
    assert np.array_equal(g64.x, r64.x) and np.array_equal(g64.residual_history,
                                                          r64.residual_history)
    assert np.array_equal(glg.x, hlg.x)
    out[rank] = (r64.x, r64.iterations, r64.residual_history, r64.final_residual,
                 rmx.iterations, rmx.final_residual, rr.x, rr.iterations, rr.cycles,
                 dec.Q, dec.H)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_gmres_matches_single(cuda):
    import paper_2011_05090_b200 as sg
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    A, b, th = _problem()
    s64 = sg.gmres(A, b, m=60, theta=th, policy=sg.UNIFIED64, tol=1e-9)
    smx = sg.gmres(A, b, m=60, theta=th, policy=sg.MIXED32_64, tol=1e-6)
    srr = sg.gmres_restarted(A, b, th, sg.UNIFIED64, restart=25, max_iters=200, tol=1e-8)
    sdec = sg.arnoldi(A, b, 20, theta=th, policy=sg.UNIFIED64)
    o0, o1 = out[0], out[1]
    # replicated quantities agree across ranks bit for bit
    assert np.array_equal(o0[0], o1[0]) and np.array_equal(o0[2], o1[2])
    assert np.array_equal(o0[10], o1[10])
    # and with the single-GPU solve to rounding (summation order of the sketches)
    assert abs(o0[1] - s64.iterations) <= 1
    assert np.linalg.norm(o0[0] - s64.x) <= 1e-8 * np.linalg.norm(s64.x)
    assert o0[3] <= 10 * s64.final_residual + 1e-14
    assert abs(o0[4] - smx.iterations) <= max(1, round(0.02 * smx.iterations))
    assert o0[5] <= 10 * smx.final_residual
    assert abs(o0[7] - srr.iterations) <= max(1, round(0.02 * srr.iterations))
    assert np.linalg.norm(o0[6] - srr.x) <= 1e-7 * np.linalg.norm(srr.x)
    # Arnoldi: rank-local rows of Q stacked = the single-GPU basis; H replicated
    from paper_2011_05090_b200.workloads import shard_rows
    Q = np.concatenate([out[r][9] for r in range(world)], axis=0)
    assert Q.shape == sdec.Q.shape
    assert np.linalg.norm(Q - sdec.Q) <= 1e-10 * np.linalg.norm(sdec.Q)
    assert np.linalg.norm(o0[10] - sdec.H) <= 1e-10 * np.linalg.norm(sdec.H)
    assert shard_rows(A.n, 2, 1, 4096) == (8192, A.n - 8192)
