"""BASELINE-size checks on the GPU, through size-independent properties and
the oracle-pinned RGMRES iteration counts (tests/golden/c3_oracle_128.json,
produced by oracle/run_c3_oracle.py)."""

import json
import os

import numpy as np
import pytest
import torch

import paper_2011_05090_b200 as sg
from conftest import GOLDEN
from paper_2011_05090_b200.workloads import CONFIGS, convdiff3d, make_w_device, rhs_gaussian

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("lagged", [False, True])
@pytest.mark.parametrize("policy", ["f64", "mixed"])
def test_c3_rgmres_iterations_match_oracle(cuda, policy, lagged):
    ref = json.load(open(os.path.join(GOLDEN, "c3_oracle_128.json")))[policy]
    cfg = CONFIGS["c3"]
    N = cfg["grid"]
    rp, ci, va = convdiff3d(N, (cfg["beta"],) * 3)
    A = sg.SparseMatrix(n=N ** 3, row_ptr=rp, col_idx=ci, values=va)
    b = torch.from_numpy(rhs_gaussian(A.n, 0)).cuda()
    th = sg.make_sketch(sg.SketchKind.PSRHT, cfg["k"], A.n, 0)
    res = sg.gmres_restarted(A, b, th, sg.policy_from_name(policy), cfg["restart"],
                             cfg["max_iters"], cfg["tol"], lagged=lagged)
    its = ref["iterations"]
    assert abs(res.iterations - its) <= round(0.02 * its), (res.iterations, its)
    assert res.final_residual <= cfg["tol"]
    assert res.cycles[0] == ref["cycles"][0]


def test_c1_size_factorization_properties(cuda):
    # c1 shape (n = 1e6, k = 1500 P-SRHT, mixed, breakdown_factor 0) with m = 96
    n, m, k = 1_000_000, 96, 1500
    W = make_w_device(n, m, 1e-10, 0, torch.float32, "cuda")
    th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
    st = sg.RgsState(th, sg.MIXED32_64, capacity=m + 1, breakdown_factor=0.0)
    st.factorize_columns(W, W.shape[1], m)
    f = st.device_factors()
    Q64, R = f.Q.double(), f.R
    Wm = W[:, :n].t().double()
    # S = Theta Q and P = Theta W for the computed factors (fine-dtype sketches)
    cols = [0, 1, m // 2, m - 1]
    SQ = th.apply_block(f.Q[:, cols])
    assert float(torch.linalg.norm(SQ - f.S[:, cols]) / torch.linalg.norm(f.S[:, cols])) < 1e-6
    PW = th.apply_block(Wm[:, cols])
    assert float(torch.linalg.norm(PW - f.P[:, cols]) / torch.linalg.norm(f.P[:, cols])) < 1e-12
    # W = Q R to the coarse roundoff, S nearly orthonormal, R upper triangular
    rel = float(torch.linalg.norm(Wm - Q64 @ R) / torch.linalg.norm(Wm))
    assert rel < 1e-5
    eye = torch.eye(m, dtype=torch.float64, device="cuda")
    assert float(torch.linalg.norm(eye - f.S.t() @ f.S, 2)) < 0.5
    assert float(torch.linalg.norm(torch.tril(R, -1))) == 0.0
    # bit-identical rerun of the whole factorisation
    st2 = sg.RgsState(th, sg.MIXED32_64, capacity=m + 1, breakdown_factor=0.0)
    st2.factorize_columns(W, W.shape[1], m)
    g = st2.device_factors()
    assert torch.equal(f.Q, g.Q) and torch.equal(f.R, g.R) and torch.equal(f.S, g.S)


def test_c0_shape_device_rademacher_factorization(cuda):
    """c0 shapes (n = 1e5, k = 600, fp64) with the reference's Rademacher
    sketch generated on the device: W = QR to fp64 roundoff, S = Theta Q
    nearly orthonormal (the sketch of the fp64 basis), streaming == batch."""
    cfg = CONFIGS["c0r"]
    n, m, k = cfg["n"], 120, cfg["k"]
    W = make_w_device(n, m, 1e-4, 0, torch.float64, "cuda")
    th = sg.make_sketch(sg.SketchKind.RADEMACHER, k, n, 0)
    st = sg.RgsState(th, sg.UNIFIED64, capacity=m + 1)
    st.factorize_columns(W, W.shape[1], m)
    f = st.device_factors()
    Wm = W[:, :n].t()
    assert float(torch.linalg.norm(Wm - f.Q @ f.R) / torch.linalg.norm(Wm)) < 1e-14
    eye = torch.eye(m, dtype=torch.float64, device="cuda")
    assert float(torch.linalg.norm(eye - f.S.t() @ f.S, 2)) < 1e-12
    cols = [0, m // 2, m - 1]
    SQ = th.apply_block(f.Q[:, cols])
    assert float(torch.linalg.norm(SQ - f.S[:, cols]) / torch.linalg.norm(f.S[:, cols])) < 1e-13
    # streaming pushes give the batch factorisation bit for bit
    st2 = sg.RgsState(th, sg.UNIFIED64, capacity=m + 1)
    for j in range(12):
        st2.push(Wm[:, j])
    assert torch.equal(st2.device_factors().R, f.R[:12, :12])
    assert torch.equal(st2.device_factors().Q, f.Q[:, :12])


def _metrics_dev(W, f):
    """factor_metrics (oracle/metrics.py) on the GPU in fp64: ||I - S^T S||_2,
    ||I - Q^T Q||_2, ||W - QR||_F / ||W||_F."""
    Q, R, S = f.Q.double(), f.R.double(), f.S.double()
    Wd = W.double()
    eye = torch.eye(Q.shape[1], dtype=torch.float64, device=Q.device)
    return {"orth_S_2": float(torch.linalg.matrix_norm(eye - S.t() @ S, ord=2)),
            "orth_Q_2": float(torch.linalg.matrix_norm(eye - Q.t() @ Q, ord=2)),
            "relres_F": float(torch.linalg.norm(Wd - Q @ R) / torch.linalg.norm(Wd))}


def _golden_fullsize():
    return np.load(os.path.join(GOLDEN, "fullsize.npz"))


def test_c0_full_size_metrics_within_10x_of_oracle(cuda):
    """BASELINE c0 at full size (n = 1e5, m = 300, k = 600 Gaussian, fp64,
    sigma_min = 1e-8): the 2-norm metrics within 10x of the oracle's
    (tests/golden/fullsize.npz, oracle/make_fullsize_golden.py)."""
    from paper_2011_05090_b200.workloads import make_w
    g = _golden_fullsize()
    n, m, k = 100_000, 300, 600
    W = torch.from_numpy(make_w(n, m, 1e-8, 0)).cuda()
    th = sg.make_sketch(sg.SketchKind.GAUSSIAN, k, n, 0)
    f, _ = sg.rgs_factorize(W, th, sg.UNIFIED64, device_factors=True)
    ours = _metrics_dev(W, f)
    for key, v in ours.items():
        assert v <= 10.0 * max(float(g[f"c0_{key}"]), 1e-15), (key, v, float(g[f"c0_{key}"]))


def test_c0_twin_full_size_q_r_s_within_1e10(cuda):
    """c0's well-conditioned twin (sigma_min = 1e-2) at full size: R, S and
    sampled rows of Q within 1e-10 of the oracle (the north_star fp64 gate)."""
    from paper_2011_05090_b200.workloads import make_w
    g = _golden_fullsize()
    n, m, k = 100_000, 300, 600
    W = torch.from_numpy(make_w(n, m, 1e-2, 0)).cuda()
    th = sg.make_sketch(sg.SketchKind.GAUSSIAN, k, n, 0)
    f, _ = sg.rgs_factorize(W, th, sg.UNIFIED64, device_factors=True)
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
    assert rel(f.R.cpu().numpy(), g["c0twin_R"]) <= 1e-10
    assert rel(f.S.cpu().numpy(), g["c0twin_S"]) <= 1e-10
    rows = torch.from_numpy(g["c0twin_rows"]).cuda()
    assert rel(f.Q[rows].cpu().numpy(), g["c0twin_Qrows"]) <= 1e-10


def test_c1_full_size_metrics_within_10x_of_oracle(cuda):
    """BASELINE c1 at full size (n = 1e6, m = 500, k = 1500 P-SRHT,
    MIXED32_64, breakdown_factor 0, W fp32): the 2-norm metrics within 10x of
    the oracle's, and diag(R) close to the oracle's."""
    from paper_2011_05090_b200.workloads import make_w
    g = _golden_fullsize()
    n, m, k = 1_000_000, 500, 1500
    W = torch.from_numpy(make_w(n, m, 1e-10, 0, dtype=np.float32)).cuda()
    th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
    f, _ = sg.rgs_factorize(W, th, sg.MIXED32_64, breakdown_factor=0.0, device_factors=True)
    ours = _metrics_dev(W, f)
    for key, v in ours.items():
        assert v <= 10.0 * max(float(g[f"c1_{key}"]), 1e-15), (key, v, float(g[f"c1_{key}"]))
    d = torch.diagonal(f.R).cpu().numpy()
    assert np.linalg.norm(d - g["c1_Rdiag"]) <= 1e-3 * np.linalg.norm(g["c1_Rdiag"])


def test_c2_shape_q_r_s_vs_oracle(cuda):
    """BASELINE c2's shape (n = 2^23, k = 2000 block-SRHT over 8 seeded 2^20-row
    blocks, fp64, breakdown_factor 0) with 200 of its 1000 columns (the oracle
    host cannot hold the full W): R, S and sampled rows of Q within 1e-10 of the
    oracle (tests/golden/c2m200.npz, oracle/make_c2_golden.py), metrics within 10x."""
    from paper_2011_05090_b200.workloads import make_w
    g = np.load(os.path.join(GOLDEN, "c2m200.npz"))
    n, m, k = 1 << 23, 200, 2000
    W = torch.from_numpy(make_w(n, m, 1e-6, 0)).cuda()
    th = sg.make_sketch(sg.SketchKind.BLOCK_SRHT, k, n, 0, block_log2=20)
    f, _ = sg.rgs_factorize(W, th, sg.UNIFIED64, breakdown_factor=0.0, device_factors=True)
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
    assert rel(f.R.cpu().numpy(), g["c2_R"]) <= 1e-10
    assert rel(f.S.cpu().numpy(), g["c2_S"]) <= 1e-10
    rows = torch.from_numpy(g["c2_rows"]).cuda()
    assert rel(f.Q[rows].cpu().numpy(), g["c2_Qrows"]) <= 1e-10
    ours = _metrics_dev(W, f)
    for key, v in ours.items():
        assert v <= 10.0 * max(float(g[f"c2_{key}"]), 1e-15), (key, v, float(g[f"c2_{key}"]))


def test_c4_shape_metrics_vs_oracle(cuda):
    """BASELINE c4's shape on one GPU (n = 2^25, k = 3000 block-SRHT over 32
    seeded 2^20-row blocks, W fp32, MIXED32_64, breakdown_factor 0) with 64 of
    its 1500 columns (c4 itself needs 4 GPUs): the 2-norm metrics within 10x of
    the oracle's (tests/golden/c4m64.npz, oracle/make_c4_golden.py) and R close
    to the oracle's at the fp32 level."""
    from paper_2011_05090_b200.workloads import make_w
    g = np.load(os.path.join(GOLDEN, "c4m64.npz"))
    n, m, k = 1 << 25, 64, 3000
    W = torch.from_numpy(make_w(n, m, 1e-10, 0, dtype=np.float32)).cuda()
    th = sg.make_sketch(sg.SketchKind.BLOCK_SRHT, k, n, 0, block_log2=20)
    f, _ = sg.rgs_factorize(W, th, sg.MIXED32_64, breakdown_factor=0.0, device_factors=True)
    ours = _metrics_dev(W, f)
    for key, v in ours.items():
        assert v <= 10.0 * max(float(g[f"c4_{key}"]), 1e-15), (key, v, float(g[f"c4_{key}"]))
    R = f.R.cpu().numpy()
    assert np.linalg.norm(R - g["c4_R"]) <= 1e-5 * np.linalg.norm(g["c4_R"])
