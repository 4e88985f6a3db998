"""Oracle randomized Gram-Schmidt (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Restates reference gram_schmidt.py: the incrementally updated Householder
least-squares solver (_IncrementalHouseholderQR, :122-190), one RGS step
(RgsState.push, :293-339) with the precision policy dtypes (precision.py:37-42),
rgs_factorize (:350-375) and certificates (:474-487).  Same numpy/BLAS/LAPACK
calls in the same order as the reference.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg

POLICIES = {
    # name: (coarse dtype, fine dtype, u_crs)       precision.py:37-42
    "f32": (np.float32, np.float32, 2.0**-24),
    "f64": (np.float64, np.float64, 2.0**-53),
    "mixed": (np.float32, np.float64, 2.0**-24),
}


class OracleBreakdown(RuntimeError):
    def __init__(self, column, r_ii, tol):
        super().__init__(f"breakdown at column {column}")
        self.column, self.r_ii, self.tol = column, r_ii, tol


class householder_lsq:
    """Householder QR of S grown column by column (gram_schmidt.py:122-190)."""

    def __init__(self, k: int, dtype):
        self.k, self.dt = k, np.dtype(dtype)
        self.V, self.nrm2, self.Rc = [], [], []

    def _reflect(self, z):
        # gram_schmidt.py:141-146, reflectors in append order
        for v, vn2 in zip(self.V, self.nrm2):
            off = self.k - v.shape[0]
            t = z[off:]
            t -= (self.dt.type(2.0) * (v @ t) / vn2) * v
        return z

    def add(self, col):
        # gram_schmidt.py:148-171
        i = len(self.V)
        z = self._reflect(np.asarray(col, dtype=self.dt).copy())
        x = z[i:].copy()
        nx = np.linalg.norm(x)
        alpha = -np.copysign(nx, x[0]) if x[0] != 0 else -nx
        v = x
        v[0] -= alpha
        vn2 = float(v @ v)
        if vn2 == 0.0:
            v = np.zeros_like(x)
            v[0] = 1.0
            vn2 = 1.0
        r = np.empty(i + 1, dtype=self.dt)
        r[:i] = z[:i]
        r[i] = alpha
        self.V.append(v)
        self.nrm2.append(vn2)
        self.Rc.append(r)

    def solve(self, p):
        # gram_schmidt.py:180-190
        i = len(self.V)
        if i == 0:
            return np.zeros(0, dtype=self.dt)
        z = self._reflect(np.asarray(p, dtype=self.dt).copy())
        R = np.zeros((i, i), dtype=self.dt)
        for j, c in enumerate(self.Rc):
            R[:j + 1, j] = c
        d = np.abs(np.diag(R))
        if np.min(d) < 1e-8 * max(np.max(d), 1.0):
            raise np.linalg.LinAlgError("sketched basis numerically rank deficient")
        return scipy.linalg.solve_triangular(R, z[:i], lower=False)


class OracleRgs:
    """Streaming RGS state (gram_schmidt.py:228-347) with preallocated storage."""

    def __init__(self, theta, policy: str = "mixed", breakdown_factor: float = 10.0,
                 capacity: int = 16, phi=None):
        self.theta = theta
        self.phi = phi
        self.crs, self.fine, self.u_crs = POLICIES[policy]
        self.bf = float(breakdown_factor)
        n, k = theta.n, theta.k
        self.m = 0
        self._Q = np.zeros((n, capacity), dtype=self.crs)
        self._R = np.zeros((capacity, capacity))
        self._S = np.zeros((k, capacity), dtype=self.fine)
        self._P = np.zeros((k, capacity), dtype=self.fine)
        self.ls = householder_lsq(k, self.fine)
        if phi is not None:
            self._S_phi = np.zeros((phi.k, capacity), dtype=self.fine)
            self._P_phi = np.zeros((phi.k, capacity), dtype=self.fine)

    def _ensure(self):
        cap = self._Q.shape[1]
        if self.m < cap:
            return
        grow = lambda a: np.concatenate([a, np.zeros((a.shape[0], cap), a.dtype)], axis=1)
        self._Q, self._S, self._P = grow(self._Q), grow(self._S), grow(self._P)
        if self.phi is not None:
            self._S_phi, self._P_phi = grow(self._S_phi), grow(self._P_phi)
        R = np.zeros((2 * cap, 2 * cap))
        R[:cap, :cap] = self._R
        self._R = R

    def push(self, w) -> float:
        # gram_schmidt.py:293-339
        self._ensure()
        i = self.m
        fine = np.dtype(self.fine)
        w64 = np.asarray(w, dtype=np.float64)
        p = self.theta.apply(w64).astype(fine)                      # step 1
        if self.phi is not None:                                    # gram_schmidt.py:304-305
            self._P_phi[:, i] = self.phi.apply(w64).astype(fine)
        if i == 0:
            r = np.zeros(0, dtype=fine)
            qp = w64.astype(self.crs)
            sp = p.copy()
        else:
            r = self.ls.solve(p)                                    # step 2
            qp = w64.astype(self.crs) - self._Q[:, :i] @ r.astype(self.crs)   # step 3
            sp = self.theta.apply(qp.astype(np.float64)).astype(fine)       # step 4
        r_ii = float(np.sqrt(np.sum(sp.astype(fine) * sp)))         # step 5
        tol = self.bf * self.u_crs * float(np.linalg.norm(p))
        if r_ii <= tol:
            raise OracleBreakdown(i + 1, r_ii, tol)
        self._S[:, i] = sp / fine.type(r_ii)                        # step 6
        self._Q[:, i] = (qp.astype(np.float64) / r_ii).astype(self.crs)
        self._P[:, i] = p
        self._R[:i, i] = r.astype(np.float64)
        self._R[i, i] = r_ii
        if self.phi is not None:                                    # gram_schmidt.py:333-335
            self._S_phi[:, i] = (self.phi.apply(qp.astype(np.float64)) / r_ii).astype(fine)
        self.ls.add(self._S[:, i])
        self.m += 1
        return r_ii

    @property
    def Q(self):
        return self._Q[:, :self.m]

    @property
    def R(self):
        return self._R[:self.m, :self.m]

    @property
    def S(self):
        return self._S[:, :self.m]

    @property
    def P(self):
        return self._P[:, :self.m]


def oracle_rgs_factorize(W, theta, policy: str = "mixed", breakdown_factor: float = 10.0,
                         phi=None, capacity: int = 16, progress=None):
    """Returns dict Q, R, S, P (+ S_phi, P_phi) (gram_schmidt.py:350-375).

    `capacity` only sizes the first allocation (the reference starts at 16 and
    doubles, which changes storage, not arithmetic); the full-size golden runs
    preallocate m columns so the doubling copy of a 67 GB Q never happens.
    `progress(j)` is called after column j (logging of long runs)."""
    W = np.asarray(W)
    n, m = W.shape
    if not (theta.k >= m and n >= m >= 1):
        raise ValueError("need k >= m and n >= m >= 1")
    st = OracleRgs(theta, policy, breakdown_factor, capacity=capacity, phi=phi)
    for j in range(m):
        st.push(W[:, j])
        if progress is not None:
            progress(j)
    out = {"Q": st.Q.copy(), "R": st.R.copy(), "S": st.S.copy(), "P": st.P.copy()}
    if phi is not None:
        out["S_phi"] = st._S_phi[:, :st.m].copy()
        out["P_phi"] = st._P_phi[:, :st.m].copy()
    return out


def oracle_certificates(S, P, R):
    """(delta_m, delta_tilde_m, cond_S) as gram_schmidt.py:474-487."""
    S = np.asarray(S, dtype=np.float64)
    P = np.asarray(P, dtype=np.float64)
    m = S.shape[1]
    dm = float(np.linalg.norm(np.eye(m) - S.T @ S))
    dt = float(np.linalg.norm(P - S @ R) / np.linalg.norm(P))
    sv = np.linalg.svd(S, compute_uv=False)
    return dm, dt, float(sv[0] / sv[-1]) if sv[-1] > 0 else np.inf
