"""RGS-GMRES / Arnoldi across sketch kinds (fused P-SRHT path and the generic
path: dense Rademacher/Gaussian, small-block block-SRHT) and precision
policies, against the oracle (krylov.py:176-319)."""

import numpy as np
import pytest
import torch

import paper_2011_05090_b200 as sg
from oracle import OracleSketch, csr_matvec, oracle_arnoldi, oracle_gmres
from paper_2011_05090_b200.workloads import convdiff3d, rhs_gaussian

pytestmark = pytest.mark.gpu

N = 16
RP, CI, VA = convdiff3d(N)
NN = N ** 3
KINDS = {
    "psrht": (sg.SketchKind.PSRHT, {}, "psrht", {}),
    "rademacher": (sg.SketchKind.RADEMACHER, {}, "rademacher", {}),
    "gaussian": (sg.SketchKind.GAUSSIAN, {}, "gaussian", {}),
    "block_srht": (sg.SketchKind.BLOCK_SRHT, {"block_log2": 10}, "block_srht", {"block_log2": 10}),
}
POL = {"f64": sg.UNIFIED64, "mixed": sg.MIXED32_64, "f32": sg.UNIFIED32}


def _mv(x):
    return csr_matvec(RP, CI, VA, NN, x)


@pytest.mark.parametrize("kind", list(KINDS))
@pytest.mark.parametrize("policy", ["f64", "mixed", "f32"])
def test_gmres_kinds_policies_vs_oracle(cuda, kind, policy):
    sk, kw, ok, okw = KINDS[kind]
    k = 160
    A = sg.SparseMatrix(n=NN, row_ptr=RP, col_idx=CI, values=VA)
    b = rhs_gaussian(NN, 1)
    th = sg.make_sketch(sk, k, NN, 2, **kw)
    tol = 1e-8 if policy != "f32" else 1e-5
    res = sg.gmres(A, b, m=60, theta=th, policy=POL[policy], tol=tol)
    ref = oracle_gmres(_mv, NN, b, 60, OracleSketch(ok, k, NN, 2, **okw), policy, tol=tol)
    its = ref["iterations"]
    assert abs(res.iterations - its) <= max(1, round(0.02 * its)), (res.iterations, its)
    assert res.final_residual <= 10 * ref["final_residual"] + 1e-14
    scale = 1e-6 if policy != "f32" else 1e-2
    assert np.linalg.norm(res.x - ref["x"]) <= scale * np.linalg.norm(ref["x"])


@pytest.mark.parametrize("kind", ["psrht", "gaussian"])
def test_arnoldi_mixed_vs_oracle(cuda, kind):
    sk, kw, ok, okw = KINDS[kind]
    A = sg.SparseMatrix(n=NN, row_ptr=RP, col_idx=CI, values=VA)
    b = rhs_gaussian(NN, 5)
    th = sg.make_sketch(sk, 120, NN, 4, **kw)
    dec = sg.arnoldi(A, b, 30, theta=th, policy=sg.MIXED32_64)
    ref = oracle_arnoldi(_mv, NN, b, 30, OracleSketch(ok, 120, NN, 4, **okw), "mixed")
    assert dec.Q.dtype == np.float32 and dec.Q.shape == ref["Q"].shape
    assert np.linalg.norm(dec.H - ref["H"]) <= 1e-5 * np.linalg.norm(ref["H"])
    assert np.linalg.norm(dec.Q - ref["Q"]) <= 1e-5 * np.linalg.norm(ref["Q"])
    # Arnoldi relation A Q = Q H up to the coarse (fp32) rounding of the basis
    Q = dec.Q.astype(np.float64)
    AQ = np.column_stack([_mv(Q[:, j]) for j in range(30)])
    assert np.linalg.norm(AQ - Q @ dec.H) <= 1e-5 * np.linalg.norm(AQ)


def test_gmres_cuda_tensor_in_out(cuda):
    A = sg.SparseMatrix(n=NN, row_ptr=RP, col_idx=CI, values=VA)
    b = rhs_gaussian(NN, 3)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 160, NN, 0)
    r_np = sg.gmres(A, b, m=50, theta=th, policy=sg.UNIFIED64, tol=1e-10)
    r_cu = sg.gmres(A, torch.from_numpy(b).cuda(), m=50, theta=th, policy=sg.UNIFIED64, tol=1e-10)
    assert isinstance(r_cu.x, torch.Tensor) and r_cu.x.is_cuda
    assert np.array_equal(r_cu.x.cpu().numpy(), r_np.x)
    assert r_cu.iterations == r_np.iterations


def test_gmres_phi_certification_sketches(cuda):
    A = sg.SparseMatrix(n=NN, row_ptr=RP, col_idx=CI, values=VA)
    b = rhs_gaussian(NN, 3)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 160, NN, 0)
    phi = sg.make_sketch(sg.SketchKind.RADEMACHER, 300, NN, 7)
    res = sg.gmres(A, b, m=30, theta=th, policy=sg.UNIFIED64, phi=phi)
    f = res.factors
    Q = np.asarray(f.Q, dtype=np.float64)
    Sphi = np.asarray(f.S_phi)
    assert Sphi.shape == (300, Q.shape[1])
    assert np.linalg.norm(Sphi - phi.apply_block(Q)) <= 1e-12 * np.linalg.norm(Sphi)
    cert = sg.certify_factorization(f, eps_star=0.25, u_crs=sg.UNIFIED64.u_crs)
    assert cert.omega_bar_q >= sg.epsilon_of(th, Q)


def test_restarted_gmres_with_ilu(cuda):
    A = sg.SparseMatrix(n=NN, row_ptr=RP, col_idx=CI, values=VA)
    b = rhs_gaussian(NN, 0)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 160, NN, 0)
    plain = sg.gmres_restarted(A, b, th, sg.UNIFIED64, restart=40, max_iters=400, tol=1e-8)
    pre = sg.gmres_restarted(A, b, th, sg.UNIFIED64, restart=40, max_iters=400, tol=1e-8,
                             preconditioner=sg.ilu0(A))
    assert pre.converged and pre.final_residual <= 1e-8
    assert pre.iterations < plain.iterations
