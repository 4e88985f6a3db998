"""One-synchronisation (lagged) RGS-Arnoldi / RGS-GMRES on
the GPU against the oracle's restatement of the same algorithm
(oracle_gmres_lagged) and against the reference's standard RGS-GMRES
(oracle_gmres): the lag only reorders Steps 5-7, so iteration counts must stay
within the north_star's +-2 % of the reference's."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2011_05090_b200 as sg
from oracle import (OracleIlu0, OracleSketch, csr_matvec, oracle_gmres, oracle_gmres_lagged,
                    oracle_gmres_restarted)
from paper_2011_05090_b200.workloads import convdiff3d, rhs_gaussian

pytestmark = pytest.mark.gpu

POL = {"f64": sg.UNIFIED64, "mixed": sg.MIXED32_64, "f32": sg.UNIFIED32}


def _its_ok(a, b):
    return abs(a - b) <= max(1, round(0.02 * b))


def _cd(N):
    rp, ci, va = convdiff3d(N)
    A = sg.SparseMatrix(n=N ** 3, row_ptr=rp, col_idx=ci, values=va)
    return A, (lambda x: csr_matvec(rp, ci, va, A.n, x))


@pytest.mark.parametrize("pol", ["f64", "mixed", "f32"])
@pytest.mark.parametrize("kind", ["psrht", "gaussian"])
def test_lagged_gmres_matches_oracle(cuda, pol, kind):
    A, mv = _cd(16)  # n = 4096: one 4096-row tile, the fused column kernel for P-SRHT
    b = rhs_gaussian(A.n, 3)
    k = 200
    th = sg.make_sketch(getattr(sg.SketchKind, kind.upper()), k, A.n, 0)
    oth = OracleSketch(kind, k, A.n, 0)
    tol = {"f64": 1e-9, "mixed": 1e-6, "f32": 1e-5}[pol]
    res = sg.gmres(A, b, m=120, theta=th, policy=POL[pol], tol=tol, lagged=True)
    lag = oracle_gmres_lagged(mv, A.n, b, 120, oth, pol, tol=tol)
    std = oracle_gmres(mv, A.n, b, 120, oth, pol, tol=tol)
    assert _its_ok(res.iterations, lag["iterations"])
    assert _its_ok(res.iterations, std["iterations"])
    assert res.final_residual <= 10 * max(lag["final_residual"], 1e-15)
    if pol == "f64":
        assert np.linalg.norm(res.x - lag["x"]) <= 1e-8 * np.linalg.norm(lag["x"])
        R = res.factors.R
        nr = min(R.shape[0], lag["R"].shape[0])
        assert np.linalg.norm(R[:nr, :nr] - lag["R"][:nr, :nr]) <= 1e-10 * np.linalg.norm(lag["R"])


@pytest.mark.parametrize("n_side", [12, 16])  # n = 1728 (non-fused P-SRHT path), 4096 (fused)
def test_lagged_arnoldi_factors(cuda, n_side):
    A, mv = _cd(n_side)
    b = rhs_gaussian(A.n, 5)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 120, A.n, 1)
    dec = sg.arnoldi(A, b, 40, theta=th, policy=sg.UNIFIED64, lagged=True)
    ref = oracle_gmres_lagged(mv, A.n, b, 40, OracleSketch("psrht", 120, A.n, 1), "f64",
                              scale_by_norm=False)
    assert dec.Q.shape == ref["Q"].shape == (A.n, 41)
    assert np.linalg.norm(dec.Q - ref["Q"]) <= 1e-10 * np.linalg.norm(ref["Q"])
    assert np.linalg.norm(dec.R - ref["R"]) <= 1e-10 * np.linalg.norm(ref["R"])
    AQ = np.column_stack([mv(dec.Q[:, j]) for j in range(40)])
    assert np.linalg.norm(AQ - dec.Q @ dec.H) <= 1e-12 * np.linalg.norm(AQ)
    # same basis as the standard RGS-Arnoldi to rounding
    std = sg.arnoldi(A, b, 40, theta=th, policy=sg.UNIFIED64)
    assert np.linalg.norm(dec.Q - std.Q) <= 1e-10 * np.linalg.norm(std.Q)


def test_lagged_arnoldi_lucky_breakdown(cuda):
    # b in a 3-dimensional invariant subspace: column 4 breaks down
    n = 4096
    d = np.concatenate([[1.0, 2.0, 3.0], np.linspace(4.0, 9.0, n - 3)])
    A = sg.SparseMatrix(n=n, row_ptr=np.arange(n + 1, dtype=np.int32),
                        col_idx=np.arange(n, dtype=np.int32), values=d)
    b = np.zeros(n)
    b[:3] = [1.0, -1.0, 0.5]
    th = sg.make_sketch(sg.SketchKind.PSRHT, 64, n, 0)
    std = sg.arnoldi(A, b, 10, theta=th, policy=sg.UNIFIED64)
    dec = sg.arnoldi(A, b, 10, theta=th, policy=sg.UNIFIED64, lagged=True)
    assert std.breakdown and dec.breakdown
    assert dec.Q.shape == std.Q.shape
    assert np.linalg.norm(dec.Q - std.Q) <= 1e-10 * np.linalg.norm(std.Q)
    # every returned column normalised exactly once
    assert np.allclose(np.linalg.norm(th.apply_block(dec.Q), axis=0), 1.0, atol=1e-12)


@pytest.mark.parametrize("pol", ["f64", "mixed"])
def test_lagged_restarted_matches_reference_iterations(cuda, pol):
    A, mv = _cd(32)  # n = 32768 = 8 tiles, c3's operator family
    b = rhs_gaussian(A.n, 0)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 300, A.n, 0)
    out = sg.gmres_restarted(A, b, th, POL[pol], restart=100, max_iters=800, tol=1e-8,
                             lagged=True)
    ref = oracle_gmres_restarted(mv, A.n, b, OracleSketch("psrht", 300, A.n, 0), pol,
                                 restart=100, max_iters=800, tol=1e-8)
    assert _its_ok(out.iterations, ref["iterations"])
    assert out.final_residual <= 1e-8 * 1.0000001


def test_lagged_ilu_preconditioned(cuda):
    A, mv = _cd(16)
    b = rhs_gaussian(A.n, 1)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 160, A.n, 0)
    M = sg.ilu0(A)
    res = sg.gmres(A, b, m=80, theta=th, policy=sg.UNIFIED64, tol=1e-10, preconditioner=M,
                   lagged=True)
    pre = OracleIlu0(A.row_ptr, A.col_idx, A.values, A.n)
    ref = oracle_gmres(mv, A.n, b, 80, OracleSketch("psrht", 160, A.n, 0), "f64", tol=1e-10,
                       precond=pre)
    assert _its_ok(res.iterations, ref["iterations"])
    assert np.linalg.norm(res.x - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"])


def test_lagged_streaming_is_deterministic(cuda):
    A, _ = _cd(16)
    b = rhs_gaussian(A.n, 9)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 200, A.n, 0)
    r1 = sg.gmres(A, b, m=60, theta=th, policy=sg.MIXED32_64, tol=1e-6, lagged=True)
    r2 = sg.gmres(A, b, m=60, theta=th, policy=sg.MIXED32_64, tol=1e-6, lagged=True)
    assert np.array_equal(r1.x, r2.x) and np.array_equal(r1.residual_history,
                                                          r2.residual_history)


# ---- two ranks sharing cuda:0 (gloo on CUDA tensors), as test_gpu_sharded_krylov ----

N = 24


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    rp, ci, va = convdiff3d(N)
    A = sg.SparseMatrix(n=N ** 3, row_ptr=rp, col_idx=ci, values=va)
    return A, rhs_gaussian(A.n, 2), sg.make_sketch(sg.SketchKind.PSRHT, 200, A.n, 0)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2011_05090_b200.distributed import TorchComm
    comm = TorchComm()
    A, b, th = _problem()
    r64 = sg.gmres(A, b, m=60, theta=th, policy=sg.UNIFIED64, tol=1e-9, comm=comm, lagged=True)
    dec = sg.arnoldi(A, b, 20, theta=th, policy=sg.UNIFIED64, comm=comm, lagged=True)
    out[rank] = (r64.x, r64.iterations, r64.final_residual, dec.Q, dec.H)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_lagged_matches_single(cuda):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    A, b, th = _problem()
    s64 = sg.gmres(A, b, m=60, theta=th, policy=sg.UNIFIED64, tol=1e-9, lagged=True)
    sdec = sg.arnoldi(A, b, 20, theta=th, policy=sg.UNIFIED64, lagged=True)
    o0, o1 = out[0], out[1]
    assert np.array_equal(o0[0], o1[0]) and np.array_equal(o0[4], o1[4])
    assert abs(o0[1] - s64.iterations) <= 1
    assert np.linalg.norm(o0[0] - s64.x) <= 1e-8 * np.linalg.norm(s64.x)
    Q = np.concatenate([out[r][3] for r in range(world)], axis=0)
    assert np.linalg.norm(Q - sdec.Q) <= 1e-10 * np.linalg.norm(sdec.Q)
    assert np.linalg.norm(o0[4] - sdec.H) <= 1e-10 * np.linalg.norm(sdec.H)
