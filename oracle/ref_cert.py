"""Oracle a-posteriori certification (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Restates reference certification.py omega_bar (:57-79), certify_factorization
(:120-144) and sketch.py epsilon_of (:213-228) with the same numpy/scipy calls.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg


def oracle_omega_bar(V_theta, V_phi, eps_star):
    Vt = np.asarray(V_theta, dtype=np.float64)
    Vp = np.asarray(V_phi, dtype=np.float64)
    if Vt.ndim == 1:
        Vt = Vt[:, None]
    if Vp.ndim == 1:
        Vp = Vp[:, None]
    if Vt.shape[1] != Vp.shape[1]:
        raise ValueError("sketches have different column counts")
    R = np.linalg.qr(Vt, mode="r")
    d = np.abs(np.diag(R))
    if d.min() <= 1e-14 * max(d.max(), 1.0):
        raise np.linalg.LinAlgError("Theta-sketch is numerically rank deficient")
    B = scipy.linalg.solve_triangular(R.T, Vp.T, lower=True).T
    sv = np.linalg.svd(B, compute_uv=False)
    return max(1.0 - (1.0 - eps_star) * sv[-1] ** 2, (1.0 + eps_star) * sv[0] ** 2 - 1.0)


def oracle_epsilon_of(theta, V):
    V = np.asarray(V, dtype=np.float64)
    if V.ndim == 1:
        V = V[:, None]
    sv_v = np.linalg.svd(V, compute_uv=False)
    if sv_v[-1] <= 1e-12 * sv_v[0]:
        raise np.linalg.LinAlgError("V is numerically rank deficient")
    U, _ = np.linalg.qr(V)
    sv = np.linalg.svd(theta.apply_block(U), compute_uv=False)
    return max(1.0 - sv[-1] ** 2, sv[0] ** 2 - 1.0)


def _cond(M):
    sv = np.linalg.svd(np.asarray(M, dtype=np.float64), compute_uv=False)
    return float(sv[0] / sv[-1]) if sv[-1] > 0 else np.inf


def oracle_certify(S, S_phi, P, P_phi, eps_star, u_crs):
    ob_q = oracle_omega_bar(S, S_phi, eps_star)
    ob_w = oracle_omega_bar(P, P_phi, eps_star)
    mq, mw = u_crs * _cond(S_phi), u_crs * _cond(P_phi)
    return {"omega_bar_q": ob_q, "omega_bar_w": ob_w, "margin_q": mq, "margin_w": mw,
            "margin_ok_q": mq <= 0.1 * max(abs(ob_q), eps_star),
            "margin_ok_w": mw <= 0.1 * max(abs(ob_w), eps_star)}
