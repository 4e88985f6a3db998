"""Host-side logic of the package, checked on the CPU (no kernels launched)."""

import numpy as np
import pytest
import scipy.sparse
import torch

import paper_2011_05090_b200 as sg
from paper_2011_05090_b200 import _lib
from paper_2011_05090_b200.sketch import _pack_signs
from paper_2011_05090_b200.workloads import (convdiff3d, make_w, make_w_rows, rhs_gaussian,
                                             shard_rows)
from conftest import golden
from oracle import OracleSketch, psrht_setup


def test_exports_cover_reference_hot_path_names():
    for name in ("SketchKind", "SketchOperator", "make_sketch", "fwht", "RgsState",
                 "rgs_factorize", "QrFactors", "StabilityCertificate", "certificates",
                 "BreakdownError", "LsqSolver", "HOUSEHOLDER_QR", "PrecisionPolicy", "UNIFIED64",
                 "MIXED32_64", "UNIFIED32", "policy_from_name", "GsVariant", "SparseMatrix",
                 "arnoldi", "gmres", "GmresResult", "ArnoldiDecomposition"):
        assert hasattr(sg, name), name


def test_policies():
    assert sg.policy_from_name("mixed") is sg.MIXED32_64
    assert sg.MIXED32_64.coarse_dtype == np.float32 and sg.MIXED32_64.fine_dtype == np.float64
    with pytest.raises(ValueError):
        sg.policy_from_name("f16")
    with pytest.raises(ValueError):
        sg.LsqSolver("qr")


def test_psrht_host_construction_matches_reference_draws():
    g = golden("psrht.npz")
    for (k, n, seed) in g["cases"]:
        op = sg.make_sketch(sg.SketchKind.PSRHT, int(k), int(n), int(seed))
        tag = f"{k}_{n}_{seed}"
        assert op.s == 1 << (int(n) - 1).bit_length()
        assert np.array_equal(op.signs, g[f"signs_{tag}"])
        assert np.array_equal(op.sample_indices, g[f"samples_{tag}"])


def test_sketch_validation_like_reference():
    with pytest.raises(ValueError):
        sg.SketchOperator(sg.SketchKind.PSRHT, 0, 10, seed=0)
    with pytest.warns(UserWarning):
        sg.SketchOperator(sg.SketchKind.PSRHT, 20, 10, seed=0)
    with pytest.raises(ValueError):
        sg.SketchOperator(sg.SketchKind.BLOCK_SRHT, 8, 3000, seed=0, block_log2=10)
    assert sg.make_sketch(sg.SketchKind.PSRHT, 4, 24, 0).frobenius_norm() == pytest.approx(24**0.5)


def test_sign_bit_packing_layout():
    rng = np.random.default_rng(0)
    signs = np.where(rng.integers(0, 2, 77) == 1, 1.0, -1.0)
    words = _pack_signs(signs)
    assert words.dtype == np.uint32 and words.size == 3
    for r in range(77):
        bit = (int(words[r >> 5]) >> (r & 31)) & 1
        assert bit == (1 if signs[r] > 0 else 0)


def test_block_srht_blocks_are_reference_psrht():
    op = sg.make_sketch(sg.SketchKind.BLOCK_SRHT, 16, 4 * 1024, 3, block_log2=10)
    assert op.nblocks == 4 and op.sample_indices.shape == (4, 16)
    for j in range(4):
        _, sg_j, sm_j = psrht_setup(16, 1024, sg.block_seed(3, j))
        assert np.array_equal(op.signs[j * 1024:(j + 1) * 1024], sg_j)
        assert np.array_equal(op.sample_indices[j], sm_j)
    assert op.scale == pytest.approx(1.0 / 4.0 / 2.0)


def test_shard_rows_partition():
    for n, world, align in ((1_000_000, 8, 4096), (1 << 23, 3, 4096), (5000, 2, 32), (10, 4, 4)):
        got = [shard_rows(n, world, r, align) for r in range(world)]
        pos = 0
        for r0, nl in got:
            assert r0 == pos and (r0 % align == 0 or nl == 0)
            pos += nl
        assert pos == n


def test_convdiff3d_matches_kron_construction():
    N = 6
    rp, ci, va = convdiff3d(N, (20.0, 20.0, 20.0))
    h = 1.0 / (N + 1)
    T = scipy.sparse.diags([-1, 2, -1], [-1, 0, 1], shape=(N, N)) / h**2
    C = scipy.sparse.diags([-1, 0, 1], [-1, 0, 1], shape=(N, N)) / (2 * h)
    Ax = T + 20.0 * C
    I = scipy.sparse.identity(N)
    A = (scipy.sparse.kron(I, scipy.sparse.kron(I, Ax)) + scipy.sparse.kron(I, scipy.sparse.kron(Ax, I))
         + scipy.sparse.kron(Ax, scipy.sparse.kron(I, I))).tocsr()
    A.sum_duplicates()
    ours = scipy.sparse.csr_matrix((va, ci, rp), shape=(N**3, N**3))
    assert abs(ours - A).max() < 1e-9 * abs(A).max()
    assert len(va) == 7 * N**3 - 6 * N**2
    assert np.all(np.diff(ci[rp[0]:rp[1]]) > 0)


def test_convdiff_128_nnz():
    rp, ci, va = convdiff3d(128)
    assert rp[-1] == 14_581_760 and len(rp) == 2_097_153


def test_make_w_spectrum_and_row_blocks():
    W = make_w(3000, 20, 1e-6, 5)
    sv = np.linalg.svd(W, compute_uv=False)
    target = np.logspace(0, -6, 20)
    # G is N(0, 1/n): W's singular values track sigma within sampling noise
    assert np.all(np.abs(np.log10(sv / target)) < 0.2)
    assert np.array_equal(make_w_rows(3000, 20, 1e-6, 5, 1000, 2500), W[1000:2500])


def test_rhs_is_default_rng():
    assert np.array_equal(rhs_gaussian(10, 0), np.random.default_rng(0).standard_normal(10))


def test_compute_paths_fail_loudly_without_cuda():
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    op = sg.make_sketch(sg.SketchKind.PSRHT, 8, 64, 0)
    with pytest.raises(RuntimeError):
        op.apply(np.zeros(64))
    with pytest.raises(RuntimeError):
        sg.RgsState(op, sg.UNIFIED64)
    with pytest.raises(RuntimeError):
        sg.rgs_factorize(np.ones((64, 2)), op, sg.UNIFIED64)


def test_oracle_sketch_agrees_with_package_construction():
    op = sg.make_sketch(sg.SketchKind.PSRHT, 12, 100, 4)
    orc = OracleSketch("psrht", 12, 100, 4)
    assert np.array_equal(op.signs, orc.signs) and np.array_equal(op.sample_indices, orc.samples)


def test_srht_rows_limit_is_explicit():
    import paper_2011_05090_b200 as sg
    from paper_2011_05090_b200.sketch import MAX_SRHT_ROWS
    with pytest.raises(ValueError, match="k <= 8192"):
        sg.make_sketch(sg.SketchKind.PSRHT, MAX_SRHT_ROWS + 1, 1 << 20, 0)


def test_oracle_lagged_gmres_restatement_cpu():
    """The one-synchronisation restatement against the
    reference's standard RGS-GMRES in the oracle: same Krylov space, so the
    same iteration count to +-2 % and x to the stated tolerances."""
    import numpy as np
    from oracle import OracleSketch, csr_matvec, oracle_gmres, oracle_gmres_lagged
    from paper_2011_05090_b200.workloads import convdiff3d, rhs_gaussian
    N = 10
    rp, ci, va = convdiff3d(N)
    n = N ** 3
    mv = lambda x: csr_matvec(rp, ci, va, n, x)  # noqa: E731
    b = rhs_gaussian(n, 0)
    th = OracleSketch("psrht", 120, n, 0)
    for pol, tol in (("f64", 1e-9), ("mixed", 1e-6)):
        a = oracle_gmres(mv, n, b, 80, th, pol, tol=tol)
        lg = oracle_gmres_lagged(mv, n, b, 80, th, pol, tol=tol)
        assert abs(a["iterations"] - lg["iterations"]) <= max(1, round(0.02 * a["iterations"]))
        assert lg["final_residual"] <= 10 * a["final_residual"]
    dec = oracle_gmres_lagged(mv, n, b, 25, th, "f64", scale_by_norm=False)
    Q, H = dec["Q"], dec["H"]
    AQ = np.column_stack([mv(Q[:, j]) for j in range(25)])
    assert np.linalg.norm(AQ - Q @ H) <= 1e-12 * np.linalg.norm(AQ)
