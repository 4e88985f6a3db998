"""Edge cases the reference handles (gram_schmidt.py:293-339, krylov.py:176-199)."""

import numpy as np
import pytest
import scipy.sparse

import paper_2011_05090_b200 as sg
from oracle import OracleSketch, oracle_gmres, oracle_rgs_factorize, rel_diff

pytestmark = pytest.mark.gpu


def test_single_column(cuda, rng):
    n, k = 5000, 40
    w = rng.standard_normal((n, 1))
    th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 3)
    f, cert = sg.rgs_factorize(w, th, sg.UNIFIED64)
    ref = oracle_rgs_factorize(w, OracleSketch("psrht", k, n, 3), "f64")
    assert f.Q.shape == (n, 1) and f.R.shape == (1, 1)
    assert rel_diff(f.Q, ref["Q"]) < 1e-13 and rel_diff(f.R, ref["R"]) < 1e-13
    assert abs(np.linalg.norm(f.S) - 1.0) < 1e-13


def test_tiny_dimensions(cuda):
    th = sg.make_sketch(sg.SketchKind.PSRHT, 1, 1, 0)
    f, _ = sg.rgs_factorize(np.array([[3.0]]), th, sg.UNIFIED64)
    ref = oracle_rgs_factorize(np.array([[3.0]]), OracleSketch("psrht", 1, 1, 0), "f64")
    assert np.allclose(f.R, ref["R"]) and np.allclose(f.Q, ref["Q"])
    th = sg.make_sketch(sg.SketchKind.PSRHT, 3, 5, 1)
    W = np.arange(15, dtype=np.float64).reshape(5, 3) + np.eye(5, 3)
    f, _ = sg.rgs_factorize(W, th, sg.UNIFIED64)
    ref = oracle_rgs_factorize(W, OracleSketch("psrht", 3, 5, 1), "f64")
    assert rel_diff(f.R, ref["R"]) < 1e-12


@pytest.mark.parametrize("bf", [10.0, 0.0])
def test_zero_first_column_breaks_down_at_column_one(cuda, rng, bf):
    W = rng.standard_normal((2000, 3))
    W[:, 0] = 0.0
    th = sg.make_sketch(sg.SketchKind.PSRHT, 20, 2000, 0)
    with pytest.raises(sg.BreakdownError) as e:
        sg.rgs_factorize(W, th, sg.UNIFIED64, breakdown_factor=bf)
    assert e.value.column == 1 and e.value.r_ii == 0.0


def test_nan_propagates_like_numpy(cuda, rng):
    W = rng.standard_normal((3000, 4))
    W[7, 2] = np.nan
    th = sg.make_sketch(sg.SketchKind.PSRHT, 30, 3000, 0)
    f, _ = sg.rgs_factorize(W, th, sg.UNIFIED64, with_certificate=False)
    assert np.isfinite(f.R[:2, :2]).all() and np.isnan(f.R[2, 2])


def test_arnoldi_lucky_breakdown(cuda):
    A = sg.SparseMatrix.from_scipy(scipy.sparse.eye(30, format="csr") * 2.0)
    b = np.zeros(30)
    b[0] = 1.0
    th = sg.make_sketch(sg.SketchKind.PSRHT, 16, 30, 0)
    dec = sg.arnoldi(A, b, 5, theta=th, policy=sg.UNIFIED64)
    assert dec.breakdown and dec.Q.shape[1] < 6


def test_gmres_breakdown_on_first_step_matches_reference(cuda):
    # krylov.py:288-318: a breakdown before any Hessenberg column leaves k = 0,
    # x = 0, final residual 1 and converged = breakdown = True.
    A = sg.SparseMatrix.from_scipy(scipy.sparse.eye(5000, format="csr") * 4.0)
    b = np.random.default_rng(0).standard_normal(5000)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 64, 5000, 0)
    res = sg.gmres(A, b, m=10, theta=th, policy=sg.UNIFIED64, tol=1e-10)
    assert res.iterations == 0 and res.breakdown and res.converged
    assert not res.x.any() and res.final_residual == pytest.approx(1.0)


def test_gmres_breakdown_after_two_steps(cuda, rng):
    # A with two distinct eigenvalues: the Krylov space of b has dimension 2,
    # so the third push breaks down and GMRES returns the exact solution.
    n = 6000
    d = np.where(np.arange(n) % 2 == 0, 2.0, 5.0)
    As = scipy.sparse.diags(d, format="csr")
    A = sg.SparseMatrix.from_scipy(As)
    b = rng.standard_normal(n)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 64, n, 0)
    res = sg.gmres(A, b, m=10, theta=th, policy=sg.UNIFIED64)
    ref = oracle_gmres(lambda v: As @ v, n, b, 10, OracleSketch("psrht", 64, n, 0), "f64")
    assert res.breakdown == ref["breakdown"] and res.iterations == ref["iterations"]
    assert abs(res.final_residual - ref["final_residual"]) < 1e-8


@pytest.mark.parametrize("policy", ["f64", "mixed"])
def test_push_after_breakdown_is_unaffected(cuda, rng, policy):
    # gram_schmidt.py:323-326: the failed push leaves the state unchanged, so
    # the next columns factorise exactly as if it had never been pushed
    n, k = 5000, 64
    W = rng.standard_normal((n, 6))
    th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 1)
    pol = sg.policy_from_name(policy)
    a = sg.RgsState(th, pol)
    b = sg.RgsState(th, pol)
    for j in range(3):
        a.push(W[:, j])
        b.push(W[:, j])
    bad = W[:, 0] + 2.0 * W[:, 1]  # in the span: r_ii ~ rounding level
    with pytest.raises(sg.BreakdownError) as e:
        a.push(bad)
    assert e.value.column == 4
    for j in range(3, 6):
        a.push(W[:, j])
        b.push(W[:, j])
    for name in ("Q", "R", "S", "P"):
        assert np.array_equal(getattr(a, name), getattr(b, name)), name
