"""A-posteriori certification of the embedding (reference certification.py,
sketch.py:45-87, :213-251).

The certified bound omega_bar (certification.py:57-79) needs only the two
small sketches of a basis - S = Theta Q and S_phi = Phi Q (or P, P_phi for W),
which the device factorisation already produces in the same pass as the
column (RgsState(phi=...)).  The k x m linear algebra (QR, triangular solve,
singular values) runs on the GPU in binary64 through cuSOLVER/cuBLAS; scalar
bounds (dimension formulas, the eps* bisection) are plain arithmetic.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .gram_schmidt import QrFactors
from .sketch import SketchKind, SketchOperator, make_sketch

__all__ = ["CertificationParams", "CertificationResult", "omega_bar", "omega_bar_sharpness",
           "eps_star_for_dim", "certify_factorization", "make_certification_sketch",
           "EmbeddingParams", "required_sketch_dim", "vector_certificate_dim", "epsilon_of",
           "rounding_sketch_trial"]


# ---- sketch sizing (sketch.py:45-87) ---------------------------------------------
@dataclass(frozen=True)
class EmbeddingParams:
    """(epsilon, delta, d) of an oblivious subspace embedding (sketch.py:45-58)."""

    epsilon: float
    delta: float
    d: int

    def __post_init__(self):
        if not 0.0 < self.epsilon < 1.0:
            raise ValueError("epsilon must lie in (0, 1)")
        if not 0.0 < self.delta < 1.0:
            raise ValueError("delta must lie in (0, 1)")
        if self.d < 1:
            raise ValueError("d must be a positive integer")


def required_sketch_dim(kind: SketchKind, p: EmbeddingParams, n: int | None = None) -> int:
    """Rows for an (epsilon, delta, d) embedding (sketch.py:61-73): Rademacher
    7.87 eps^-2 (6.9 d + ln 1/delta); P-SRHT 2/(eps^2 - eps^3/3) (sqrt d +
    sqrt(8 ln(6n/delta)))^2 ln(3d/delta)."""
    eps, delta, d = p.epsilon, p.delta, p.d
    if kind is SketchKind.RADEMACHER:
        return math.ceil(7.87 / (eps * eps) * (6.9 * d + math.log(1.0 / delta)))
    if kind is SketchKind.PSRHT:
        if n is None:
            raise ValueError("P-SRHT bound depends on the ambient dimension n")
        root = math.sqrt(d) + math.sqrt(8.0 * math.log(6.0 * n / delta))
        return math.ceil(2.0 / (eps ** 2 - eps ** 3 / 3.0) * root * root
                         * math.log(3.0 * d / delta))
    raise TypeError(f"unknown sketch kind {kind!r}")


def vector_certificate_dim(eps_star: float, delta_star: float) -> int:
    """Rows for a Rademacher (eps*, delta*, 1) embedding (sketch.py:76-87)."""
    if not 0.0 < eps_star < 1.0:
        raise ValueError("eps_star must lie in (0, 1)")
    if not 0.0 < delta_star < 1.0:
        raise ValueError("delta_star must lie in (0, 1)")
    return math.ceil(2.0 / (eps_star ** 2 / 2.0 - eps_star ** 3 / 3.0)
                     * math.log(2.0 / delta_star))


# ---- device helpers ---------------------------------------------------------------
def _dev64(M) -> torch.Tensor:
    _lib.require_cuda()
    if isinstance(M, torch.Tensor):
        t = M.to(device="cuda" if not M.is_cuda else M.device, dtype=torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(M, dtype=np.float64))).cuda()
    return t[:, None] if t.dim() == 1 else t


def epsilon_of(theta: SketchOperator, V) -> float:
    """Exact embedding error of theta on range(V) (sketch.py:213-228):
    max{1 - s_min(Theta U)^2, s_max(Theta U)^2 - 1} for an orthonormal basis U."""
    Vd = _dev64(V)
    sv = torch.linalg.svdvals(Vd)
    if float(sv[-1]) <= 1e-12 * float(sv[0]):
        raise np.linalg.LinAlgError("V is numerically rank deficient")
    U = torch.linalg.qr(Vd, mode="reduced").Q
    s = torch.linalg.svdvals(_dev64(theta.apply_block(U.contiguous())))
    return max(1.0 - float(s[-1]) ** 2, float(s[0]) ** 2 - 1.0)


def rounding_sketch_trial(theta: SketchOperator, gamma, trials: int, seed: int,
                          eps: float = 0.5) -> float:
    """Failure rate of | ||phi||^2 - ||Theta phi||^2 | > eps ||gamma||^2 for phi
    uniform in [-gamma, gamma] (sketch.py:231-251; same Philox stream 0x7B1A)."""
    gamma = np.asarray(gamma, dtype=np.float64)
    if np.any(gamma < 0):
        raise ValueError("gamma entries must be nonnegative")
    bound = eps * float(gamma @ gamma)
    rng = np.random.Generator(np.random.Philox(key=(int(seed) << 64) | 0x7B1A))
    phis = np.stack([rng.uniform(-gamma, gamma) for _ in range(trials)], axis=1)
    Pd = _dev64(phis)
    sk = _dev64(theta.apply_block(Pd.contiguous()))
    diff = (Pd * Pd).sum(0) - (sk * sk).sum(0)
    return float((diff.abs() > bound).sum()) / trials


# ---- certification (certification.py) ----------------------------------------------
@dataclass(frozen=True)
class CertificationParams:
    """Accuracy/failure levels and seeding of Phi (certification.py:34-46)."""

    eps_star: float = 0.05
    delta_star: float = 1e-3
    phi_seed: int = 0x0F1A
    k_phi: int | None = None

    def dimension(self) -> int:
        if self.k_phi is not None:
            return self.k_phi
        return vector_certificate_dim(self.eps_star, self.delta_star)


def make_certification_sketch(params: CertificationParams, n: int,
                              kind: SketchKind = SketchKind.RADEMACHER) -> SketchOperator:
    """Phi (certification.py:49-54); PSRHT at large n."""
    return make_sketch(kind, params.dimension(), n, params.phi_seed)


def omega_bar(V_theta, V_phi, eps_star: float) -> float:
    """Certified bound on the embedding error of Theta on range(V) from
    V_theta = Theta V and V_phi = Phi V (certification.py:57-79): with R from
    the QR of V_theta and B = V_phi R^{-1},
    max{1 - (1 - eps*) s_min(B)^2, (1 + eps*) s_max(B)^2 - 1}."""
    Vt, Vp = _dev64(V_theta), _dev64(V_phi)
    if Vt.shape[1] != Vp.shape[1]:
        raise ValueError("sketches have different column counts")
    R = torch.linalg.qr(Vt, mode="r").R
    diag = R.diagonal().abs()
    if float(diag.min()) <= 1e-14 * max(float(diag.max()), 1.0):
        raise np.linalg.LinAlgError("Theta-sketch is numerically rank deficient")
    B = torch.linalg.solve_triangular(R.t(), Vp.t(), upper=False).t()
    sv = torch.linalg.svdvals(B)
    return max(1.0 - (1.0 - eps_star) * float(sv[-1]) ** 2,
               (1.0 + eps_star) * float(sv[0]) ** 2 - 1.0)


def omega_bar_sharpness(omega: float, eps_star: float, eps_prime: float) -> float:
    """Ceiling on omega_bar when Phi embeds range(V) with eps' (certification.py:82-84)."""
    return (1.0 + eps_star) / (1.0 - eps_prime) * (1.0 + omega) - 1.0


def eps_star_for_dim(k_phi: int, delta_star: float) -> float:
    """Smallest eps* a k_phi-row Rademacher sketch certifies (certification.py:87-103)."""
    if k_phi < 1:
        raise ValueError("k_phi must be positive")
    lo, hi = 1e-8, 1.0 - 1e-12
    if vector_certificate_dim(hi, delta_star) > k_phi:
        raise ValueError(f"k_phi={k_phi} too small for any eps* < 1 at delta*={delta_star}")
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if vector_certificate_dim(mid, delta_star) <= k_phi:
            hi = mid
        else:
            lo = mid
    return hi


@dataclass
class CertificationResult:
    eps_star: float
    omega_bar_q: float
    omega_bar_w: float
    margin_q: float
    margin_w: float
    margin_ok_q: bool
    margin_ok_w: bool
    omega_bar_q_halved: float
    omega_bar_w_halved: float


def _cond(M) -> float:
    sv = torch.linalg.svdvals(_dev64(M))
    return float(sv[0] / sv[-1]) if float(sv[-1]) > 0 else math.inf


def certify_factorization(factors: QrFactors, eps_star: float,
                          u_crs: float) -> CertificationResult:
    """Certify Theta on range(Q) and range(W) from S, S_phi, P, P_phi
    (certification.py:120-144); factors from RgsState / rgs_factorize(phi=...)."""
    if getattr(factors, "S_phi", None) is None or getattr(factors, "P_phi", None) is None:
        raise ValueError("factors lack the certification sketches "
                         "(factorize with a phi operator)")
    ob_q = omega_bar(factors.S, factors.S_phi, eps_star)
    ob_w = omega_bar(factors.P, factors.P_phi, eps_star)
    margin_q = u_crs * _cond(factors.S_phi)
    margin_w = u_crs * _cond(factors.P_phi)
    return CertificationResult(
        eps_star=eps_star, omega_bar_q=ob_q, omega_bar_w=ob_w,
        margin_q=margin_q, margin_w=margin_w,
        margin_ok_q=margin_q <= 0.1 * max(abs(ob_q), eps_star),
        margin_ok_w=margin_w <= 0.1 * max(abs(ob_w), eps_star),
        omega_bar_q_halved=0.5 * ob_q, omega_bar_w_halved=0.5 * ob_w)
