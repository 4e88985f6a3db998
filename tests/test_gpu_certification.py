"""A-posteriori certification on the device vs the reference (certification.py,
sketch.py:213-228) and the reference's own checks (tests/test_certification.py)."""

import numpy as np
import pytest

import paper_2011_05090_b200 as sg
from conftest import golden

pytestmark = pytest.mark.gpu


def test_omega_bar_and_epsilon_match_reference(cuda):
    g = golden("cert.npz")
    theta = sg.make_sketch(sg.SketchKind.PSRHT, 96, 1024, seed=3)
    for t in range(3):
        ob = sg.omega_bar(g[f"Vt{t}"], g[f"Vp{t}"], 0.25)
        assert ob == pytest.approx(float(g[f"ob{t}"]), rel=1e-10)
        assert sg.epsilon_of(theta, g[f"V{t}"]) == pytest.approx(float(g[f"om{t}"]), rel=1e-10)
        # the certification sketch itself is the reference's (seeded Rademacher)
        phi = sg.make_certification_sketch(
            sg.CertificationParams(eps_star=0.25, delta_star=1e-3, phi_seed=t), 1024)
        Vp = phi.apply_block(g[f"V{t}"])
        assert np.linalg.norm(Vp - g[f"Vp{t}"]) <= 1e-13 * np.linalg.norm(g[f"Vp{t}"])


def test_certify_factorization_matches_reference(cuda):
    g = golden("cert.npz")
    theta = sg.make_sketch(sg.SketchKind.PSRHT, 128, 1024, seed=0)
    phi = sg.make_certification_sketch(sg.CertificationParams(eps_star=0.25), 1024)
    f, _ = sg.rgs_factorize(g["cf_W"], theta, sg.UNIFIED64, phi=phi)
    res = sg.certify_factorization(f, eps_star=0.25, u_crs=sg.UNIFIED64.u_crs)
    assert res.omega_bar_q == pytest.approx(float(g["cf_obq"]), rel=1e-9)
    assert res.omega_bar_w == pytest.approx(float(g["cf_obw"]), rel=1e-9)
    assert res.margin_q == pytest.approx(float(g["cf_mq"]), rel=1e-6)
    assert res.margin_ok_q and res.margin_ok_w
    assert res.omega_bar_q_halved == pytest.approx(0.5 * res.omega_bar_q)
    # device factors (CUDA tensors) take the same path
    fd, _ = sg.rgs_factorize(g["cf_W"], theta, sg.UNIFIED64, phi=phi, device_factors=True)
    rd = sg.certify_factorization(fd, eps_star=0.25, u_crs=sg.UNIFIED64.u_crs)
    assert rd.omega_bar_q == pytest.approx(res.omega_bar_q, rel=1e-12)
    # reference test_certification.py:98-110: the bounds hold
    assert res.omega_bar_q >= sg.epsilon_of(theta, f.Q)
    assert res.omega_bar_w >= sg.epsilon_of(theta, g["cf_W"])


def test_omega_bar_upper_bounds_omega_across_seeds(cuda, rng):
    # reference tests/test_certification.py:25-40 and :43-56
    n, d = 1024, 8
    theta = sg.make_sketch(sg.SketchKind.PSRHT, 96, n, seed=3)
    ratios = []
    for trial in range(20):
        V = rng.standard_normal((n, d))
        phi = sg.make_certification_sketch(
            sg.CertificationParams(eps_star=0.25, delta_star=1e-3, phi_seed=trial), n)
        ob = sg.omega_bar(theta.apply_block(V), phi.apply_block(V), 0.25)
        om = sg.epsilon_of(theta, V)
        assert ob >= om
        ratios.append(ob / om)
    assert 1.0 <= float(np.median(ratios)) <= 5.0


def test_omega_bar_sharpness_identity_and_errors(cuda, rng):
    # reference tests/test_certification.py:59-85
    n, d = 512, 6
    theta = sg.make_sketch(sg.SketchKind.PSRHT, 64, n, seed=1)
    phi = sg.make_sketch(sg.SketchKind.RADEMACHER, 400, n, seed=99)
    V = rng.standard_normal((n, d))
    om = sg.epsilon_of(theta, V)
    eps_prime = sg.epsilon_of(phi, V)
    assert eps_prime < 0.5
    ob = sg.omega_bar(theta.apply_block(V), phi.apply_block(V), eps_star=0.25)
    assert ob <= sg.omega_bar_sharpness(om, 0.25, eps_prime) + 1e-12
    V2 = rng.standard_normal((64, 5))
    assert sg.omega_bar(V2, V2, eps_star=0.1) == pytest.approx(0.1, abs=1e-10)
    Z = np.zeros((30, 2))
    Z[:, 0] = Z[:, 1] = np.arange(30, dtype=np.float64)
    with pytest.raises(np.linalg.LinAlgError):
        sg.omega_bar(Z, Z, 0.1)
    with pytest.raises(ValueError):
        sg.omega_bar(np.ones((30, 2)), np.ones((30, 3)), 0.1)


def test_certify_requires_phi(cuda, rng):
    W = rng.standard_normal((256, 5))
    theta = sg.make_sketch(sg.SketchKind.PSRHT, 64, 256, seed=0)
    f, _ = sg.rgs_factorize(W, theta, sg.UNIFIED64)
    with pytest.raises(ValueError):
        sg.certify_factorization(f, eps_star=0.25, u_crs=sg.UNIFIED64.u_crs)


def test_rounding_sketch_trial(cuda):
    theta = sg.make_sketch(sg.SketchKind.PSRHT, 256, 2048, seed=0)
    gamma = np.full(2048, 1e-3)
    rate = sg.rounding_sketch_trial(theta, gamma, trials=50, seed=1, eps=0.5)
    assert 0.0 <= rate <= 0.1
