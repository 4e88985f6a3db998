"""The reference's acceptance criteria (pkg/tests/test_acceptance.py), the
parts that concern the randomized path, run on the GPU classes with the
reference's own sizes, seeds and thresholds: criteria 1, 2, 4, 5, 6, 7, 8
and 9.  The classical CGS/MGS/CGS2 comparisons are out of scope (SURVEY.md
section 2) and are left out; criterion 3 fails in the reference itself (its
k = 1500 clause "cannot hold", pkg/test_output.txt) and is not ported."""

import hashlib

import numpy as np
import pytest
import scipy.sparse.linalg

import paper_2011_05090_b200 as sg
from oracle.ref_io import laplacian_2d, random_sparse, synthetic_matrix

pytestmark = pytest.mark.gpu

N, M, K = 100_000, 300, 5000  # test_acceptance.py:30
SEED = 1


def _A(t):
    n, rp, ci, v = t
    return sg.SparseMatrix(n=n, row_ptr=rp, col_idx=ci, values=v)


@pytest.fixture(scope="module")
def big_run():
    """test_acceptance.py:52-72 (the randomized factorizations)."""
    W = synthetic_matrix(N, M)
    theta = sg.make_sketch(sg.SketchKind.PSRHT, K, N, SEED)
    rgs, _ = sg.rgs_factorize(W, theta, sg.MIXED32_64, with_certificate=False,
                              breakdown_factor=0.0)
    rgs32, _ = sg.rgs_factorize(W, theta, sg.UNIFIED32, with_certificate=False,
                                breakdown_factor=0.0)
    return {"W": W, "rgs": rgs, "rgs32": rgs32}


def test_criterion_1_conditioning_randomized(big_run):
    """test_acceptance.py:83-110: cond(Q_rgs) <= 2, 10 <= cond(Q_rgs32) <= 1e4."""
    c = float(np.linalg.cond(big_run["rgs"].Q.astype(np.float64)))
    c32 = float(np.linalg.cond(big_run["rgs32"].Q.astype(np.float64)))
    assert c <= 2.0, c
    assert 10.0 <= c32 <= 1e4, c32


def test_criterion_2_factorization_error_randomized(big_run):
    """test_acceptance.py:113-129: ||W - QR||_F / ||W||_F <= 50 u_crs m^1.5."""
    W, f = big_run["W"], big_run["rgs"]
    rel = float(np.linalg.norm(W - f.Q.astype(np.float64) @ f.R) / np.linalg.norm(W))
    assert rel <= 50.0 * sg.MIXED32_64.u_crs * M ** 1.5, rel


def test_criterion_6_gmres_correctness():
    """test_acceptance.py:205-244 (the preconditioned Laplacian half is also in
    test_gpu_ilu.py): ILU(0)-GMRES on the 100^2 Laplacian, the Arnoldi
    identity, and 20 seeded random sparse systems against a direct solve."""
    A = _A(laplacian_2d(100))
    rng = np.random.default_rng(0)
    x_star = rng.standard_normal(A.n)
    b = A.matvec(x_star)
    theta = sg.make_sketch(sg.SketchKind.PSRHT, 200, A.n, seed=0)
    res = sg.gmres(A, b, m=80, theta=theta, policy=sg.UNIFIED64,
                   preconditioner=sg.ilu0(A), tol=1e-12)
    err = float(np.linalg.norm(res.x - x_star) / np.linalg.norm(x_star))
    dec = sg.arnoldi(A, b, 80, theta=theta, policy=sg.UNIFIED64)
    mc = dec.Q.shape[1] - 1
    AQ = np.column_stack([A.matvec(dec.Q[:, j]) for j in range(mc)])
    arn = float(np.linalg.norm(AQ - dec.Q @ dec.H[:mc + 1, :mc]))
    assert res.final_residual <= 1e-8 and err <= 1e-6
    assert arn <= 15.0 * sg.UNIFIED64.u_crs * 80 ** 2 * 10.0
    worst_res = worst_err = 0.0
    for trial in range(20):
        B = _A(random_sparse(2000, 8, seed=trial))
        xs = np.random.default_rng(trial).standard_normal(2000)
        th = sg.make_sketch(sg.SketchKind.PSRHT, 160, 2000, seed=trial)
        r = sg.gmres(B, B.matvec(xs), m=80, theta=th, policy=sg.UNIFIED64, tol=1e-12)
        x_ref = scipy.sparse.linalg.spsolve(B.to_scipy().tocsc(), B.matvec(xs))
        worst_res = max(worst_res, r.final_residual)
        worst_err = max(worst_err, float(np.linalg.norm(r.x - x_ref) / np.linalg.norm(x_ref)))
    assert worst_res <= 1e-8 and worst_err <= 1e-6, (worst_res, worst_err)


@pytest.mark.parametrize("lagged", [False, True])
def test_criterion_7_mixed_precision_plateau(lagged):
    """test_acceptance.py:247-268, the RGS clause: unpreconditioned
    mixed-precision RGMRES(400) on the 100^2 Laplacian stagnates at a residual
    in [1e-8, 1e-5] (the fp32 basis), not at the classical CGS level."""
    A = _A(laplacian_2d(100))
    y = np.ones(A.n)
    ay = A.matvec(y)
    b = ay / float(np.linalg.norm(ay))
    theta = sg.make_sketch(sg.SketchKind.PSRHT, 800, A.n, seed=0)
    r = sg.gmres(A, b, m=400, theta=theta, policy=sg.MIXED32_64, lagged=lagged)
    assert 1e-8 <= r.final_residual <= 1e-5, r.final_residual


def test_criterion_9_determinism():
    """test_acceptance.py:305-323: bit-identical reruns (sha256 of the
    factors of two independent runs)."""
    W = synthetic_matrix(20_000, 60)
    digests = []
    for _ in range(2):
        th = sg.make_sketch(sg.SketchKind.PSRHT, 400, 20_000, SEED)
        f, _ = sg.rgs_factorize(W, th, sg.MIXED32_64, breakdown_factor=0.0)
        h = hashlib.sha256()
        for a in (f.Q, f.R, f.S, f.P):
            h.update(np.ascontiguousarray(a).tobytes())
        digests.append(h.hexdigest())
    assert digests[0] == digests[1]


def test_criterion_4_certification_bound():
    """test_acceptance.py:150-176: the certified bound omega_bar (from S and
    S_phi) never falls below the exact omega of Theta on the computed basis,
    over 20 trials x 20 columns, and is sharp (median ratio in [1.3, 3.5])."""
    n, m, k = 1024, 20, 128
    eps_star = 0.25
    k_phi = sg.vector_certificate_dim(eps_star, 1e-3)
    violations, ratios = 0, []
    for trial in range(20):
        rng = np.random.default_rng(1000 + trial)
        W = rng.standard_normal((n, m))
        theta = sg.make_sketch(sg.SketchKind.PSRHT, k, n, seed=trial)
        phi = sg.make_sketch(sg.SketchKind.RADEMACHER, k_phi, n, seed=5000 + trial)
        f, _ = sg.rgs_factorize(W, theta, sg.UNIFIED64, phi=phi)
        for i in range(m):
            om = sg.epsilon_of(theta, f.Q[:, :i + 1])
            ob = sg.omega_bar(f.S[:, :i + 1], f.S_phi[:, :i + 1], eps_star)
            violations += ob < om
            ratios.append(ob / om)
    assert violations == 0
    assert 1.3 <= float(np.median(ratios)) <= 3.5, float(np.median(ratios))


def test_criterion_5_certificate_bounds():
    """test_acceptance.py:179-202: whenever Theta embeds range(W) with
    epsilon <= 1/2, Delta_m <= 20 u m^2 cond(W) and Delta~_m <= 6 u m^1.5."""
    m, k = 20, 256
    u = sg.UNIFIED64.u_crs
    fails = eligible = 0
    for trial in range(200):
        rng = np.random.default_rng(trial)
        U, _ = np.linalg.qr(rng.standard_normal((500, m)))
        V, _ = np.linalg.qr(rng.standard_normal((m, m)))
        cond = 10.0 ** rng.uniform(1, 4)
        W = (U * np.logspace(0, -np.log10(cond), m)) @ V.T
        theta = sg.make_sketch(sg.SketchKind.RADEMACHER, k, 500, seed=trial)
        f, cert = sg.rgs_factorize(W, theta, sg.UNIFIED64)
        if sg.epsilon_of(theta, W) > 0.5:
            continue
        eligible += 1
        cond_w = float(np.linalg.cond(W))
        if cert.delta_m > 20.0 * u * m ** 2 * cond_w or cert.delta_tilde_m > 6.0 * u * m ** 1.5:
            fails += 1
    assert eligible > 0 and fails == 0, (eligible, fails)


def test_criterion_8_oblivious_embedding_statistics():
    """test_acceptance.py:271-302 with the device-generated Rademacher sketch:
    k = 2318 for (0.5, 0.01, 10), epsilon <= 0.5 in >= 190 of 200 trials, the
    rounding-trial failure rate <= 0.01, and the FWHT against the dense
    Sylvester Hadamard matrix at n = 4096."""
    import warnings
    params = sg.EmbeddingParams(epsilon=0.5, delta=0.01, d=10)
    k = sg.required_sketch_dim(sg.SketchKind.RADEMACHER, params)
    assert k == 2318
    good = 0
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)  # k > n is intended here
        for trial in range(200):
            V = np.random.default_rng(trial).standard_normal((1024, 10))
            theta = sg.make_sketch(sg.SketchKind.RADEMACHER, k, 1024, seed=trial)
            good += sg.epsilon_of(theta, V) <= 0.5
        theta = sg.make_sketch(sg.SketchKind.RADEMACHER, k, 1024, seed=0)
        fail_rate = sg.rounding_sketch_trial(theta, np.ones(1024), trials=200, seed=0, eps=0.5)
    H = np.array([[1.0]])
    while H.shape[0] < 4096:
        H = np.block([[H, H], [H, -H]])
    x = np.random.default_rng(42).standard_normal(4096)
    fwht_err = float(np.max(np.abs(sg.fwht(x) - H @ x)))
    assert good >= 190, good
    assert fail_rate <= 0.01, fail_rate
    assert fwht_err <= 1e-12 * 4096, fwht_err
