"""GPU randomized Gram-Schmidt vs the reference's golden factorizations and the
oracle.  Tolerances (BASELINE.json north_star): fp64 well-conditioned
relative ||Q - Q_ref||_F, ||R - R_ref||_F <= 1e-10; every case
||I - S^T S||_2, ||I - Q^T Q||_2, ||W - QR||_F / ||W||_F within 10x of the
oracle's value."""

import numpy as np
import pytest
import torch

import paper_2011_05090_b200 as sg
from conftest import golden
from oracle import OracleRgs, OracleSketch, factor_metrics, oracle_rgs_factorize, rel_diff
from paper_2011_05090_b200.workloads import make_w

pytestmark = pytest.mark.gpu

POL = {"f64": sg.UNIFIED64, "mixed": sg.MIXED32_64, "f32": sg.UNIFIED32}


def _problem(rng, n=400, m=12, cond=1e4):
    U, _ = np.linalg.qr(rng.standard_normal((n, m)))
    V, _ = np.linalg.qr(rng.standard_normal((m, m)))
    return (U * np.logspace(0, -np.log10(cond), m)) @ V.T


def _within_10x(ours, ref, floor=1e-15):
    return ours <= 10.0 * max(ref, floor)


@pytest.mark.parametrize("name", ["psrht_f64", "rad_f64"])
def test_rgs_f64_matches_reference_golden(cuda, name):
    g = golden(f"rgs_{name}.npz")
    n, m, k, seed = (int(v) for v in g["meta"])
    kind = sg.SketchKind.PSRHT if str(g["kind"]) == "psrht" else sg.SketchKind.RADEMACHER
    th = sg.make_sketch(kind, k, n, seed)
    f, cert = sg.rgs_factorize(g["W"], th, sg.UNIFIED64, breakdown_factor=float(g["bf"]))
    assert f.Q.dtype == np.float64 and f.R.dtype == np.float64 and f.S.dtype == np.float64
    assert rel_diff(f.Q, g["Q"]) <= 1e-10
    assert rel_diff(f.R, g["R"]) <= 1e-10
    assert rel_diff(f.S, g["S"]) <= 1e-10
    assert rel_diff(f.P, g["P"]) <= 1e-13
    assert np.linalg.norm(g["W"] - f.Q @ f.R) / np.linalg.norm(g["W"]) < 1e-13
    assert np.allclose(f.R, np.triu(f.R))
    assert cert.delta_m < 1e-12 and cert.delta_tilde_m < 1e-12
    assert np.linalg.cond(f.Q) < 5.0


@pytest.mark.parametrize("name", ["psrht_mixed", "psrht_f32", "psrht_mixed_wide", "c1shape_mixed"])
def test_rgs_multiprecision_metrics_within_10x(cuda, name):
    g = golden(f"rgs_{name}.npz")
    n, m, k, seed = (int(v) for v in g["meta"])
    pol = POL[str(g["policy"])]
    th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, seed)
    f, _ = sg.rgs_factorize(g["W"], th, pol, breakdown_factor=float(g["bf"]))
    assert f.Q.dtype == pol.coarse_dtype and f.S.dtype == pol.fine_dtype
    assert f.R.dtype == np.float64
    ours = factor_metrics(g["W"], f.Q, f.R, f.S)
    ref = factor_metrics(g["W"], g["Q"], g["R"], g["S"])
    for key in ours:
        assert _within_10x(ours[key], ref[key]), (name, key, ours[key], ref[key])
    assert rel_diff(f.P, g["P"]) <= 1e-6  # P = Theta W: fine dtype sketch of the same W


def test_rgs_well_conditioned_baseline_w_f64(cuda):
    # c0-shaped twin at reduced n with sigma_min = 1e-2 (well-conditioned gate)
    n, m, k = 20000, 60, 120
    W = make_w(n, m, 1e-2, 3)
    for kind in ("gaussian", "psrht"):
        th = sg.make_sketch(sg.SketchKind(kind), k, n, 3)
        f, _ = sg.rgs_factorize(W, th, sg.UNIFIED64)
        ref = oracle_rgs_factorize(W, OracleSketch(kind, k, n, 3), "f64")
        assert rel_diff(f.Q, ref["Q"]) <= 1e-10, kind
        assert rel_diff(f.R, ref["R"]) <= 1e-10, kind
        assert rel_diff(f.S, ref["S"]) <= 1e-10, kind


def test_rgs_ill_conditioned_c0_shape_metrics(cuda):
    n, m, k = 20000, 60, 120
    W = make_w(n, m, 1e-8, 4)
    th = sg.make_sketch(sg.SketchKind.GAUSSIAN, k, n, 4)
    f, _ = sg.rgs_factorize(W, th, sg.UNIFIED64)
    ref = oracle_rgs_factorize(W, OracleSketch("gaussian", k, n, 4), "f64")
    ours = factor_metrics(W, f.Q, f.R, f.S)
    theirs = factor_metrics(W, ref["Q"], ref["R"], ref["S"])
    for key in ours:
        assert _within_10x(ours[key], theirs[key]), (key, ours[key], theirs[key])


def test_rgs_sketch_consistency(cuda, rng):
    W = _problem(rng, cond=10.0)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 96, 400, seed=3)
    f, _ = sg.rgs_factorize(W, th, sg.UNIFIED64)
    assert np.allclose(f.P, th.apply_block(W), atol=1e-12)
    assert np.allclose(f.S, th.apply_block(f.Q), atol=1e-10)


def test_rgs_streaming_matches_batch_bit_exact(cuda, rng):
    W = _problem(rng, n=300, m=10)
    for kind, pol in ((sg.SketchKind.RADEMACHER, sg.MIXED32_64), (sg.SketchKind.PSRHT, sg.UNIFIED64),
                      (sg.SketchKind.GAUSSIAN, sg.MIXED32_64)):
        th = sg.make_sketch(kind, 80, 300, seed=2)
        batch, _ = sg.rgs_factorize(W, th, pol, with_certificate=False)
        st = sg.RgsState(th, pol)
        for j in range(10):
            st.push(W[:, j])
        f = st.factors()
        assert np.array_equal(batch.Q, f.Q), kind
        assert np.array_equal(batch.R, f.R), kind
        assert np.array_equal(batch.S, f.S), kind
        assert np.array_equal(batch.P, f.P), kind


def test_rgs_rerun_bit_identical(cuda):
    W = make_w(50000, 40, 1e-10, 9, dtype=np.float32)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 200, 50000, 9)
    a, _ = sg.rgs_factorize(W, th, sg.MIXED32_64, breakdown_factor=0.0)
    b, _ = sg.rgs_factorize(W, th, sg.MIXED32_64, breakdown_factor=0.0)
    for key in ("Q", "R", "S", "P"):
        assert np.array_equal(getattr(a, key), getattr(b, key))


def test_rgs_breakdown_on_dependent_columns(cuda):
    g = golden("rgs_breakdown.npz")
    th = sg.make_sketch(sg.SketchKind.PSRHT, 64, 200, 5)
    with pytest.raises(sg.BreakdownError) as exc:
        sg.rgs_factorize(g["W"], th, sg.UNIFIED64)
    assert exc.value.column == int(g["column"]) == 5
    # streaming: state keeps the 4 good columns and m is unchanged
    st = sg.RgsState(th, sg.UNIFIED64)
    for j in range(4):
        st.push(g["W"][:, j])
    with pytest.raises(sg.BreakdownError) as exc:
        st.push(g["W"][:, 4])
    assert exc.value.column == 5 and st.m == 4 and st.Q.shape == (200, 4)


def test_rgs_breakdown_factor_zero_pushes_through(cuda, rng):
    W = _problem(rng, n=200, m=4).astype(np.float32).astype(np.float64)
    W = np.concatenate([W, W[:, :1] * (1 + 1e-7)], axis=1)
    th = sg.make_sketch(sg.SketchKind.RADEMACHER, 64, 200, seed=5)
    with pytest.raises(sg.BreakdownError):
        sg.rgs_factorize(W, th, sg.UNIFIED32)
    f, _ = sg.rgs_factorize(W, th, sg.UNIFIED32, breakdown_factor=0.0)
    assert f.Q.shape == (200, 5)


def test_rgs_input_validation(cuda, rng):
    th = sg.make_sketch(sg.SketchKind.PSRHT, 8, 100, seed=0)
    with pytest.raises(ValueError):
        sg.rgs_factorize(rng.standard_normal((100, 12)), th)  # k < m
    with pytest.raises(ValueError):
        sg.rgs_factorize(rng.standard_normal(100), th)  # not a matrix
    st = sg.RgsState(th, sg.UNIFIED64)
    with pytest.raises(ValueError):
        st.push(np.zeros(99))


def test_gpu_sketch_in_oracle_state_duck_typing(cuda, rng):
    # minimum slice: the GPU operator plugged into the CPU state through the
    # duck-typed interface (.n, .k, .apply -> ndarray) reproduces the oracle
    W = _problem(rng, n=400, m=12, cond=100.0)
    gpu_op = sg.make_sketch(sg.SketchKind.PSRHT, 96, 400, 3)
    a = OracleRgs(gpu_op, "f64")
    b = OracleRgs(OracleSketch("psrht", 96, 400, 3), "f64")
    for j in range(12):
        a.push(W[:, j])
        b.push(W[:, j])
    assert rel_diff(a.Q, b.Q) <= 1e-12 and rel_diff(a.R, b.R) <= 1e-12


def test_capacity_growth_in_streaming(cuda, rng):
    W = _problem(rng, n=500, m=40, cond=100.0)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 100, 500, 1)
    st = sg.RgsState(th, sg.UNIFIED64, capacity=4)
    for j in range(40):
        st.push(W[:, j])
    batch, _ = sg.rgs_factorize(W, th, sg.UNIFIED64)
    assert rel_diff(st.Q, batch.Q) <= 1e-12


def test_device_factors_and_certificates(cuda):
    n, m, k = 100_000, 50, 200
    W = make_w(n, m, 1e-4, 2)
    Wd = torch.from_numpy(W).cuda()
    th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 2)
    f, cert = sg.rgs_factorize(Wd, th, sg.UNIFIED64, device_factors=True)
    assert isinstance(f.Q, torch.Tensor) and f.Q.shape == (n, m)
    fh, certh = sg.rgs_factorize(W, th, sg.UNIFIED64)
    assert np.array_equal(f.Q.cpu().numpy(), fh.Q)
    assert cert.delta_m == pytest.approx(certh.delta_m, rel=1e-10, abs=1e-15)
    assert cert.passes_gate()


@pytest.mark.parametrize("knobs", [
    {},
    # every schedule branch at m = 80: late chunks doubling, Q copies from
    # column 40, far copies, the two-column tail; and the in-stream sketches
    {"_e2e_late": (24, 32), "_e2e_ship_from": 40, "_e2e_ship_far": 12, "_e2e_tail": 10,
     "_e2e_ahead": 2},
    {"_e2e_side": False, "_e2e_late": (24, 32)},
])
def test_pinned_host_pipeline_matches_device_path(cuda, monkeypatch, knobs):
    # the end-to-end path (chunked H2D / compute / D2H overlap) gives the same bits
    for key, val in knobs.items():
        monkeypatch.setattr(sg.RgsState, key, val)
    n, m, k = 200_000, 80, 300
    W = make_w(n, m, 1e-8, 21, dtype=np.float32)
    pin = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
    pin.copy_(torch.from_numpy(np.ascontiguousarray(W.T)))
    Wh = pin.numpy().T
    assert Wh.flags.f_contiguous
    th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 21)
    a, _ = sg.rgs_factorize(Wh, th, sg.MIXED32_64, breakdown_factor=0.0)
    b, _ = sg.rgs_factorize(W, th, sg.MIXED32_64, breakdown_factor=0.0)
    for key in ("Q", "R", "S", "P"):
        assert np.array_equal(getattr(a, key), getattr(b, key)), key


@pytest.mark.parametrize("kind,k,n,pol,blog", [
    ("psrht", 300, 20_000, "f32", None),          # UNIFIED32 through the fused column kernel
    ("block_srht", 3000, 4 * 16384, "mixed", 14),  # c4-like: k = 3000 (> 128 rows per LS CTA)
    ("block_srht", 2000, 8 * 8192, "f64", 13),     # c2-like block structure
])
def test_rgs_larger_k_and_policies_vs_oracle(cuda, kind, k, n, pol, blog):
    m = 40
    W = make_w(n, m, 1e-6, 5, dtype=np.float32 if pol != "f64" else np.float64)
    kw = {"block_log2": blog} if blog else {}
    th = sg.make_sketch(sg.SketchKind(kind), k, n, 5, **kw)
    f, _ = sg.rgs_factorize(W, th, POL[pol], breakdown_factor=0.0)
    ref = oracle_rgs_factorize(W, OracleSketch(kind, k, n, 5, **kw), pol, 0.0)
    ours = factor_metrics(W, f.Q, f.R, f.S)
    theirs = factor_metrics(W, ref["Q"], ref["R"], ref["S"])
    for key in ours:
        assert _within_10x(ours[key], theirs[key]), (key, ours[key], theirs[key])
    if pol == "f64":
        assert rel_diff(f.Q, ref["Q"]) <= 1e-10 and rel_diff(f.R, ref["R"]) <= 1e-10
    # streaming == batch holds on these paths too
    st = sg.RgsState(th, POL[pol], breakdown_factor=0.0)
    for j in range(8):
        st.push(W[:, j])
    assert np.array_equal(st.R, f.R[:8, :8])


@pytest.mark.parametrize("phikind,n", [("rademacher", 3000), ("psrht", 20000)])
def test_certification_sketches_phi(cuda, phikind, n):
    # S_phi = Phi q'_i / r_ii and P_phi = Phi w_i (gram_schmidt.py:304-305, 333-335)
    m, k, kphi = 20, 120, 60
    W = make_w(n, m, 1e-4, 8)
    th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 8)
    phi = sg.make_sketch(sg.SketchKind(phikind), kphi, n, 99)
    f, _ = sg.rgs_factorize(W, th, sg.UNIFIED64, phi=phi)
    ref = oracle_rgs_factorize(W, OracleSketch("psrht", k, n, 8), "f64",
                               phi=OracleSketch(phikind, kphi, n, 99))
    assert f.S_phi.shape == (kphi, m) and f.P_phi.shape == (kphi, m)
    assert rel_diff(f.P_phi, ref["P_phi"]) <= 1e-13
    assert rel_diff(f.S_phi, ref["S_phi"]) <= 1e-10
    # streaming carries them too
    st = sg.RgsState(th, sg.UNIFIED64, phi=phi)
    for j in range(m):
        st.push(W[:, j])
    g = st.factors()
    assert np.array_equal(g.S_phi, f.S_phi) and np.array_equal(g.P_phi, f.P_phi)
    with pytest.raises(ValueError):
        sg.RgsState(th, sg.UNIFIED64, phi=sg.make_sketch(sg.SketchKind.PSRHT, 10, n + 1, 0))


@pytest.mark.parametrize("thkind,phikind,pol,n", [
    ("psrht", "psrht", "f64", 20000), ("psrht", "psrht", "mixed", 3 * 4096 + 517),
    ("block_srht", "block_srht", "mixed", 4 * 4096), ("psrht", "block_srht", "f64", 8 * 4096)])
def test_phi_fused_epilogue_bit_identical(cuda, thkind, phikind, pol, n):
    """Phi q' from the column kernel's epilogue and Phi W from the pair tile
    kernel (no re-read of q' / W) equal the stand-alone Phi launches bit for
    bit (SGS_PHI_FUSED=0 path), batch and streaming."""
    from paper_2011_05090_b200 import gram_schmidt as gsm
    m, k, kphi = 24, 160, 72
    W = make_w(n, m, 1e-4, 3, dtype=np.float32 if pol == "mixed" else np.float64)
    kw = lambda kind: {"block_log2": 12} if kind == "block_srht" else {}  # noqa: E731
    th = sg.make_sketch(sg.SketchKind(thkind), k, n, 4, **kw(thkind))
    phi = sg.make_sketch(sg.SketchKind(phikind), kphi, n, 77, **kw(phikind))
    f, _ = sg.rgs_factorize(W, th, POL[pol], phi=phi, breakdown_factor=0.0)
    assert sg.RgsState(th, POL[pol], phi=phi).phi_fused
    old = gsm._PHI_FUSED
    try:
        gsm._PHI_FUSED = False
        g, _ = sg.rgs_factorize(W, th, POL[pol], phi=phi, breakdown_factor=0.0)
        assert not sg.RgsState(th, POL[pol], phi=phi).phi_fused
    finally:
        gsm._PHI_FUSED = old
    for a, b in ((f.S_phi, g.S_phi), (f.P_phi, g.P_phi), (f.R, g.R), (f.S, g.S), (f.Q, g.Q)):
        assert np.array_equal(a, b)
    st = sg.RgsState(th, POL[pol], phi=phi, breakdown_factor=0.0)
    for j in range(m):
        st.push(W[:, j])
    h = st.factors()
    assert np.array_equal(h.S_phi, f.S_phi) and np.array_equal(h.P_phi, f.P_phi)
