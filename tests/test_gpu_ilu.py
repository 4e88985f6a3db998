"""ILU(0) right preconditioning on the device vs the reference (krylov.py:86-151,
:229-319) through golden fixtures and the pinned oracle."""

import numpy as np
import pytest
import scipy.sparse

import paper_2011_05090_b200 as sg
from conftest import golden
from oracle import OracleIlu0, OracleSketch, csr_matvec, oracle_gmres
from paper_2011_05090_b200.workloads import convdiff3d, rhs_gaussian

pytestmark = pytest.mark.gpu

ILU_MATS = ("lap6", "rs60", "rs300", "lap40")


def _mat(g, name):
    n = len(g[f"{name}_sv"])
    return sg.SparseMatrix(n=n, row_ptr=g[f"{name}_rp"], col_idx=g[f"{name}_ci"],
                           values=g[f"{name}_v"])


@pytest.mark.parametrize("name", ILU_MATS)
def test_ilu0_factors_bit_identical_to_reference(cuda, name):
    g = golden("ilu.npz")
    pre = sg.ilu0(_mat(g, name))
    for f in ("L", "U"):
        M = getattr(pre, f)
        assert np.array_equal(M.indptr, g[f"{name}_{f}rp"])
        assert np.array_equal(M.indices, g[f"{name}_{f}ci"])
        assert np.array_equal(M.data, g[f"{name}_{f}v"])


@pytest.mark.parametrize("name", ILU_MATS)
def test_ilu0_solve_matches_reference(cuda, name):
    # the sweeps sum in CSR order, scipy's SuperLU gstrs in its own: tolerance 1e-12
    g = golden("ilu.npz")
    pre = sg.ilu0(_mat(g, name))
    ref = g[f"{name}_solve"]
    y = pre.solve(g[f"{name}_sv"])
    assert np.linalg.norm(y - ref) <= 1e-12 * np.linalg.norm(ref)
    # repeated solves reuse the flag array through the epoch counter
    for _ in range(3):
        assert np.array_equal(pre.solve(g[f"{name}_sv"]), y)


def test_ilu0_errors_match_reference(cuda):
    g = golden("ilu.npz")
    Z = sg.SparseMatrix.from_scipy(scipy.sparse.csr_matrix(
        np.array([[1.0, 1, 0], [1, 1, 0], [0, 0, 1]])))
    with pytest.raises(ZeroDivisionError) as e:
        sg.ilu0(Z)
    assert str(e.value) == str(g["zero_pivot_msg"])
    # reference test_ilu0_rejects_zero_diagonal (tests/test_krylov.py:75-78)
    S = sg.SparseMatrix.from_coo(2, [0, 1], [1, 0], [1.0, 1.0])
    with pytest.raises(ValueError, match="structural zero diagonal at row 0"):
        sg.ilu0(S)
    # row 0's pivot used by a later row
    P = sg.SparseMatrix.from_scipy(scipy.sparse.csr_matrix(
        np.array([[0.0, 1, 0], [1, 1, 0], [0, 0, 1]]) + np.diag([1e-40, 0, 0])))
    with pytest.raises(ZeroDivisionError, match="at row 0"):
        sg.ilu0(P)


def test_ilu0_from_host_factors(cuda):
    g = golden("ilu.npz")
    A = _mat(g, "rs300")
    ref = OracleIlu0(A.row_ptr, A.col_idx, A.values, A.n)
    pre = sg.Ilu0Preconditioner(ref.L, ref.U)
    y = pre.solve(g["rs300_sv"])
    assert np.linalg.norm(y - g["rs300_solve"]) <= 1e-12 * np.linalg.norm(y)


def test_preconditioned_gmres_matches_reference(cuda):
    g = golden("ilu.npz")
    A = _mat(g, "lap40")
    th = sg.make_sketch(sg.SketchKind.PSRHT, 200, A.n, 0)
    res = sg.gmres(A, g["pg_b"], m=60, theta=th, policy=sg.UNIFIED64,
                   preconditioner=sg.ilu0(A), tol=1e-12)
    its = int(g["pg_its"])
    assert abs(res.iterations - its) <= max(1, int(0.02 * its))
    assert res.final_residual <= 10 * float(g["pg_res"]) + 1e-14
    assert np.linalg.norm(res.x - g["pg_x"]) <= 1e-9 * np.linalg.norm(g["pg_x"])
    B = _mat(g, "rs300")
    th2 = sg.make_sketch(sg.SketchKind.PSRHT, 200, 300, 0)
    r2 = sg.gmres(B, g["pr_b"], m=40, theta=th2, policy=sg.MIXED32_64,
                  preconditioner=sg.ilu0(B))
    assert r2.iterations == int(g["pr_its"])
    assert r2.final_residual <= 10 * float(g["pr_res"])
    # the reference's own check (tests/test_krylov.py:141-148)
    plain = sg.gmres(B, g["pr_b"], m=40, theta=th2, policy=sg.MIXED32_64)
    assert r2.final_residual < plain.final_residual


def test_criterion6_preconditioned_laplacian(cuda):
    """Acceptance criterion 6's preconditioned half (tests/test_acceptance.py:205-215):
    2D Laplacian, 1e4 unknowns, ILU(0), m=80, tol 1e-12."""
    A = sg.SparseMatrix.from_scipy(_laplacian_2d(100))
    x_star = np.random.default_rng(0).standard_normal(A.n)
    b = A.matvec(x_star)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 200, A.n, seed=0)
    res = sg.gmres(A, b, m=80, theta=th, policy=sg.UNIFIED64, preconditioner=sg.ilu0(A),
                   tol=1e-12)
    err = np.linalg.norm(res.x - x_star) / np.linalg.norm(x_star)
    assert res.final_residual <= 1e-8 and err <= 1e-6
    ref = oracle_gmres(lambda v: csr_matvec(A.row_ptr, A.col_idx, A.values, A.n, v), A.n, b, 80,
                       OracleSketch("psrht", 200, A.n, 0), "f64", tol=1e-12,
                       precond=OracleIlu0(A.row_ptr, A.col_idx, A.values, A.n))
    assert abs(res.iterations - ref["iterations"]) <= max(1, int(0.02 * ref["iterations"]))


def test_ilu0_convdiff_factor_bitwise_and_solve(cuda):
    rp, ci, va = convdiff3d(24)
    A = sg.SparseMatrix(n=24 ** 3, row_ptr=rp, col_idx=ci, values=va)
    pre = sg.ilu0(A)
    ref = OracleIlu0(rp, ci, va, A.n)
    assert np.array_equal(pre.L.data, ref.L.data) and np.array_equal(pre.U.data, ref.U.data)
    v = rhs_gaussian(A.n, 3)
    y = pre.solve(v)
    yr = ref.solve(v)
    assert np.linalg.norm(y - yr) <= 1e-12 * np.linalg.norm(yr)


def test_ilu0_full_size_c3_properties(cuda):
    """At c3's 128^3: L U y == v through the device factors (residual of the
    two sweeps), and preconditioned RGMRES beats the unpreconditioned one."""
    import torch
    rp, ci, va = convdiff3d(128)
    A = sg.SparseMatrix(n=128 ** 3, row_ptr=rp, col_idx=ci, values=va)
    pre = sg.ilu0(A)
    v = torch.from_numpy(rhs_gaussian(A.n, 0)).cuda()
    y = pre.solve(v)
    L, U = pre.L, pre.U
    yh = y.cpu().numpy()
    back = L @ (U @ yh)
    assert np.linalg.norm(back - v.cpu().numpy()) <= 1e-12 * np.linalg.norm(v.cpu().numpy())
    th = sg.make_sketch(sg.SketchKind.PSRHT, 200, A.n, 0)
    b = rhs_gaussian(A.n, 0)
    r_pre = sg.gmres(A, b, m=40, theta=th, policy=sg.UNIFIED64, preconditioner=pre)
    r_plain = sg.gmres(A, b, m=40, theta=th, policy=sg.UNIFIED64)
    assert r_pre.final_residual < r_plain.final_residual


def _laplacian_2d(grid):
    """5-point Laplacian (the reference's generate_laplacian_2d, io.py:102-115)."""
    T = scipy.sparse.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(grid, grid))
    I = scipy.sparse.eye(grid)
    return (scipy.sparse.kron(I, T) + scipy.sparse.kron(T, I)).tocsr()
