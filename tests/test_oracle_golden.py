"""The CPU oracle reproduces the reference bit for bit on the golden vectors
produced by running the reference itself (oracle/make_golden.py)."""

import numpy as np
import pytest

from conftest import golden
from oracle import (OracleIlu0, OracleSketch, csr_matvec, fwht_ref, oracle_arnoldi, oracle_certificates,
                    oracle_gmres, oracle_rgs_factorize, psrht_setup)
from oracle.ref_rgs import OracleBreakdown


def test_fwht_kat_and_golden():
    g = golden("fwht.npz")
    assert np.array_equal(fwht_ref(g["kat_in"]), np.array([10.0, -2.0, -4.0, 0.0]))
    assert np.array_equal(g["kat_out"], np.array([10.0, -2.0, -4.0, 0.0]))
    for s in (1, 2, 8, 64, 1024, 4096, 16384):
        assert np.array_equal(fwht_ref(g[f"x_{s}"]), g[f"y_{s}"]), s
    assert np.array_equal(fwht_ref(g["X_mat"]), g["Y_mat"])


def test_fwht_rejects_non_pow2():
    with pytest.raises(ValueError):
        fwht_ref(np.zeros(6))


def test_psrht_construction_and_apply_match_reference():
    g = golden("psrht.npz")
    for (k, n, seed) in g["cases"]:
        tag = f"{k}_{n}_{seed}"
        s, signs, samples = psrht_setup(int(k), int(n), int(seed))
        assert s == 1 << (int(n) - 1).bit_length()
        assert np.array_equal(signs, g[f"signs_{tag}"])
        assert np.array_equal(samples, g[f"samples_{tag}"])
        op = OracleSketch("psrht", int(k), int(n), int(seed))
        assert np.array_equal(op.apply(g[f"x_{tag}"]), g[f"y_{tag}"]), tag
        assert np.array_equal(op.apply_block(g[f"X_{tag}"]), g[f"Y_{tag}"]), tag


def test_rademacher_materialize_matches_reference():
    g = golden("psrht.npz")
    op = OracleSketch("rademacher", 20, 50, 5)
    assert np.allclose(op.apply_block(np.eye(50)), g["rad_materialize_20_50_5"], atol=1e-15)


@pytest.mark.parametrize("name", ["psrht_f64", "psrht_mixed", "rad_f64", "psrht_f32",
                                  "psrht_mixed_wide", "c1shape_mixed"])
def test_oracle_rgs_bit_identical_to_reference(name):
    g = golden(f"rgs_{name}.npz")
    n, m, k, seed = (int(v) for v in g["meta"])
    op = OracleSketch(str(g["kind"]), k, n, seed)
    out = oracle_rgs_factorize(g["W"], op, str(g["policy"]), float(g["bf"]))
    for key in ("Q", "R", "S", "P"):
        assert out[key].dtype == g[key].dtype
        assert np.array_equal(out[key], g[key]), (name, key)
    cert = oracle_certificates(out["S"], out["P"], out["R"])
    assert np.allclose(cert, g["cert"], rtol=1e-12)


def test_oracle_breakdown_column():
    g = golden("rgs_breakdown.npz")
    op = OracleSketch("psrht", 64, 200, 5)
    with pytest.raises(OracleBreakdown) as e:
        oracle_rgs_factorize(g["W"], op, "f64", 10.0)
    assert e.value.column == int(g["column"]) == 5


def test_oracle_krylov_matches_reference():
    g = golden("krylov.npz")
    n = len(g["lap_b"])
    mv = lambda x: csr_matvec(g["lap_rp"], g["lap_ci"], g["lap_v"], n, x)
    op = OracleSketch("psrht", 200, n, 0)
    out = oracle_gmres(mv, n, g["lap_b"], 150, op, "f64", tol=1e-12)
    assert out["iterations"] == int(g["lap_its"])
    assert np.array_equal(out["x"], g["lap_x"])
    assert np.array_equal(out["history"], g["lap_hist"])
    nb = len(g["rs_b"])
    mv2 = lambda x: csr_matvec(g["rs_rp"], g["rs_ci"], g["rs_v"], nb, x)
    dec = oracle_arnoldi(mv2, nb, g["rs_b"], 15, OracleSketch("psrht", 64, nb, 0), "f64")
    assert np.array_equal(dec["Q"], g["rs_Q"])
    assert np.array_equal(dec["H"], g["rs_H"])
    n12 = len(g["l12_b"])
    mv3 = lambda x: csr_matvec(g["l12_rp"], g["l12_ci"], g["l12_v"], n12, x)
    r12 = oracle_gmres(mv3, n12, g["l12_b"], 120, OracleSketch("psrht", 140, n12, 0), "mixed")
    assert r12["iterations"] == int(g["l12_its"])
    assert r12["final_residual"] == float(g["l12_res"])


ILU_MATS = ("lap6", "rs60", "rs300", "lap40")


@pytest.mark.parametrize("name", ILU_MATS)
def test_oracle_ilu0_bit_identical_to_reference(name):
    g = golden("ilu.npz")
    n = len(g[f"{name}_sv"])
    pre = OracleIlu0(g[f"{name}_rp"], g[f"{name}_ci"], g[f"{name}_v"], n)
    for f in ("L", "U"):
        M = getattr(pre, f)
        assert np.array_equal(M.indptr, g[f"{name}_{f}rp"])
        assert np.array_equal(M.indices, g[f"{name}_{f}ci"])
        assert np.array_equal(M.data, g[f"{name}_{f}v"])
    assert np.array_equal(pre.solve(g[f"{name}_sv"]), g[f"{name}_solve"])


def test_oracle_ilu0_errors_match_reference():
    import scipy.sparse
    g = golden("ilu.npz")
    Z = scipy.sparse.csr_matrix(np.array([[1.0, 1, 0], [1, 1, 0], [0, 0, 1]]))
    with pytest.raises(ZeroDivisionError) as e:
        OracleIlu0(Z.indptr, Z.indices, Z.data, 3)
    assert str(e.value) == str(g["zero_pivot_msg"])
    S = scipy.sparse.csr_matrix(np.array([[0.0, 1.0], [1.0, 0.0]]))
    with pytest.raises(ValueError, match="structural zero diagonal at row 0"):
        OracleIlu0(S.indptr, S.indices, S.data, 2)


def test_oracle_preconditioned_gmres_matches_reference():
    g = golden("ilu.npz")
    n = len(g["lap40_sv"])
    mv = lambda x: csr_matvec(g["lap40_rp"], g["lap40_ci"], g["lap40_v"], n, x)
    pre = OracleIlu0(g["lap40_rp"], g["lap40_ci"], g["lap40_v"], n)
    out = oracle_gmres(mv, n, g["pg_b"], 60, OracleSketch("psrht", 200, n, 0), "f64",
                       tol=1e-12, precond=pre)
    assert out["iterations"] == int(g["pg_its"])
    assert np.array_equal(out["history"], g["pg_hist"])
    assert np.array_equal(out["x"], g["pg_x"])
    assert out["final_residual"] == float(g["pg_res"])
    mv2 = lambda x: csr_matvec(g["rs300_rp"], g["rs300_ci"], g["rs300_v"], 300, x)
    pre2 = OracleIlu0(g["rs300_rp"], g["rs300_ci"], g["rs300_v"], 300)
    out2 = oracle_gmres(mv2, 300, g["pr_b"], 40, OracleSketch("psrht", 200, 300, 0), "mixed",
                        precond=pre2)
    assert out2["iterations"] == int(g["pr_its"])
    assert np.array_equal(out2["x"], g["pr_x"])


def test_oracle_certification_matches_reference():
    from oracle import oracle_certify, oracle_epsilon_of, oracle_omega_bar
    g = golden("cert.npz")
    th = OracleSketch("psrht", 96, 1024, 3)
    for t in range(3):
        assert oracle_omega_bar(g[f"Vt{t}"], g[f"Vp{t}"], 0.25) == float(g[f"ob{t}"])
        assert oracle_epsilon_of(th, g[f"V{t}"]) == float(g[f"om{t}"])
    r = oracle_certify(g["cf_S"], g["cf_Sphi"], g["cf_P"], g["cf_Pphi"], 0.25, 2.0 ** -53)
    assert r["omega_bar_q"] == float(g["cf_obq"]) and r["omega_bar_w"] == float(g["cf_obw"])
    assert r["margin_q"] == float(g["cf_mq"]) and r["margin_w"] == float(g["cf_mw"])


def test_sizing_helpers_match_reference():
    # host arithmetic of the package (no device work)
    import paper_2011_05090_b200 as sg
    g = golden("cert.npz")
    got = [sg.eps_star_for_dim(sg.vector_certificate_dim(e, 1e-3), 1e-3)
           for e in (0.05, 0.1, 0.25, 0.5)]
    assert np.array_equal(np.array(got), g["eps_inv"])
    assert sg.vector_certificate_dim(0.25, 1e-3) == 584  # reference test_certification.py:13
    assert sg.CertificationParams(k_phi=100).dimension() == 100
    with pytest.raises(ValueError):
        sg.eps_star_for_dim(1, 1e-3)
    with pytest.raises(ValueError):
        sg.EmbeddingParams(1.5, 0.1, 3)


def test_rademacher_philox_restatement_matches_numpy():
    """The device generator's algorithm (oracle.rademacher_column_bits) is numpy's
    Philox(key=(seed << 64) | j).integers(0, 2, size=k) bit for bit."""
    from oracle.ref_sketch import _gen, rademacher_column_bits
    for seed, j, k in ((0, 0, 1), (5, 3, 20), (5, 49, 33), (7, 2**40 + 5, 600), (123, 99999, 1500)):
        assert np.array_equal(rademacher_column_bits(seed, j, k), _gen(seed, j).integers(0, 2, size=k))


def test_problem_generators_match_reference():
    """oracle.ref_io restates the reference's generators (io.py:84-141) bit for
    bit: tests/golden/io_gen.npz, and test_io.py's W[99, 49] golden value."""
    from oracle.ref_io import laplacian_2d, random_sparse, synthetic_matrix
    g = golden("io_gen.npz")
    W = synthetic_matrix(100, 50)
    assert np.array_equal(W, g["synth"])
    assert W[99, 49] == 0.43473583367982266 or abs(W[99, 49] - 0.43473583367982266) <= 1e-15
    for name, (n, rp, ci, v) in (("lap6", laplacian_2d(6)), ("rs30", random_sparse(30, 3, 9)),
                                 ("rs200", random_sparse(200, 8, 4))):
        assert np.array_equal(rp, g[f"{name}_rp"]) and np.array_equal(ci, g[f"{name}_ci"])
        assert np.array_equal(v, g[f"{name}_v"])
