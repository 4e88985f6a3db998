"""Oracle RGS-Arnoldi / RGS-GMRES (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Restates reference krylov.py: SparseMatrix.matvec (:81-83, scipy CSR),
_operator_norm_estimate (:213-226), arnoldi (:176-199), gmres (:229-319,
with the ILU(0) right preconditioner of :86-151), and the restart wrapper BASELINE config 3 needs
(identical definition to paper_2011_05090_b200.gmres_restarted).
"""

from __future__ import annotations

import numpy as np
import scipy.linalg
import scipy.sparse

from .ref_rgs import OracleBreakdown, OracleRgs


def csr_matvec(row_ptr, col_idx, values, n, x):
    A = scipy.sparse.csr_matrix((values, col_idx, row_ptr), shape=(n, n))
    return A @ np.asarray(x, dtype=np.float64)


class OracleIlu0:
    """ILU(0) factors (krylov.py:86-151): F holds L (strict lower, unit
    diagonal implied) and U (upper incl. diagonal) on A's pattern."""

    def __init__(self, row_ptr, col_idx, values, n, pivot_tol=1e-30):
        self.n = n
        indptr = np.asarray(row_ptr, dtype=np.int64)
        indices = np.asarray(col_idx, dtype=np.int64)
        data = np.asarray(values, dtype=np.float64).copy()
        # krylov.py:114-124: {col: pos} per row (last one wins), structural check
        diag = np.full(n, -1, dtype=np.int64)
        maps = []
        for i in range(n):
            cm = {}
            for p in range(indptr[i], indptr[i + 1]):
                cm[int(indices[p])] = p
            maps.append(cm)
            diag[i] = cm.get(i, -1)
        if np.any(diag < 0):
            raise ValueError(f"structural zero diagonal at row {int(np.argmin(diag))}")
        # krylov.py:125-145: row-oriented IKJ elimination in storage order
        for i in range(1, n):
            lo, hi = int(indptr[i]), int(indptr[i + 1])
            for p in range(lo, hi):
                k = int(indices[p])
                if k >= i:
                    break
                pivot = data[diag[k]]
                if abs(pivot) < pivot_tol:
                    raise ZeroDivisionError(f"ILU(0) pivot too small at row {k}")
                lik = data[p] / pivot
                data[p] = lik
                cmk = maps[k]
                for q in range(p + 1, hi):
                    pos = cmk.get(int(indices[q]))
                    if pos is not None:
                        data[q] -= lik * data[pos]
            if abs(data[diag[i]]) < pivot_tol:
                raise ZeroDivisionError(f"ILU(0) pivot too small at row {i}")
        self.F = data
        full = scipy.sparse.csr_matrix((data, indices.copy(), indptr.copy()), shape=(n, n))
        # krylov.py:146-151
        self.L = (scipy.sparse.tril(full, k=-1, format="csr")
                  + scipy.sparse.eye(n, format="csr")).tocsr()
        self.U = scipy.sparse.triu(full, k=0, format="csr")

    def solve(self, v):
        """M^{-1} v = U^{-1} L^{-1} v with scipy's triangular solves (krylov.py:95-99)."""
        import scipy.sparse.linalg as spla
        v = np.asarray(v, dtype=np.float64)
        y = spla.spsolve_triangular(self.L, v, lower=True, unit_diagonal=True)
        return spla.spsolve_triangular(self.U, y, lower=False)


def power_norm_estimate(matvec, n: int, iters: int = 20) -> float:
    v = np.cos(np.arange(n, dtype=np.float64) + 1.0)
    v /= np.linalg.norm(v)
    sigma = 1.0
    for _ in range(iters):
        w = matvec(v)
        nw = np.linalg.norm(w)
        if nw == 0.0:
            return 0.0
        sigma = nw
        v = w / nw
    return float(sigma)


def oracle_arnoldi(matvec, n, b, m, theta, policy="mixed"):
    st = OracleRgs(theta, policy, capacity=16)
    st.push(np.asarray(b, dtype=np.float64))
    broke = False
    for i in range(m):
        w = matvec(st.Q[:, i].astype(np.float64))
        try:
            st.push(w)
        except OracleBreakdown:
            broke = True
            break
    R = st.R.copy()
    return {"Q": st.Q.copy(), "H": R[:, 1:].copy(), "R": R, "beta": float(R[0, 0]),
            "breakdown": broke}


def oracle_gmres(matvec, n, b, m, theta, policy="mixed", tol=None, precond=None):
    """krylov.py:229-319; `precond` is an OracleIlu0 (right preconditioning:
    the Arnoldi operator is A M^{-1}, x = M^{-1} x_tilde, residual on A)."""
    b = np.asarray(b, dtype=np.float64)
    a_matvec = matvec
    if precond is not None:
        def matvec(v):  # noqa: F811 - effective operator A M^{-1}
            return a_matvec(precond.solve(v))
    b_norm = float(np.linalg.norm(b))
    if b_norm == 0.0:
        return {"x": np.zeros(n), "history": np.zeros(0), "final_residual": 0.0,
                "iterations": 0, "converged": True, "breakdown": False}
    alpha = power_norm_estimate(matvec, n)
    if alpha == 0.0:
        raise np.linalg.LinAlgError("operator norm estimate is zero")
    st = OracleRgs(theta, policy, capacity=16)
    st.push(b / b_norm)
    beta = float(st.R[0, 0])
    g = np.zeros(m + 1)
    g[0] = beta
    T = np.zeros((m + 1, m))
    cs, sn = np.zeros(m), np.zeros(m)
    hist, broke, iters = [], False, 0
    for i in range(m):
        w = matvec(st.Q[:, i].astype(np.float64)) / alpha
        try:
            st.push(w)
        except OracleBreakdown:
            broke = True
            break
        iters = i + 1
        h = st.R[:i + 2, i + 1].copy()
        for j in range(i):
            t = cs[j] * h[j] + sn[j] * h[j + 1]
            h[j + 1] = -sn[j] * h[j] + cs[j] * h[j + 1]
            h[j] = t
        rr = np.hypot(h[i], h[i + 1])
        if rr == 0.0:
            cs[i], sn[i] = 1.0, 0.0
        else:
            cs[i], sn[i] = h[i] / rr, h[i + 1] / rr
        h[i], h[i + 1] = rr, 0.0
        T[:i + 2, i] = h
        g[i + 1] = -sn[i] * g[i]
        g[i] = cs[i] * g[i]
        est = abs(g[i + 1]) / beta
        hist.append(est)
        if tol is not None and est <= tol:
            break
    k = iters
    if k == 0:
        x = np.zeros(n)
    else:
        y = scipy.linalg.solve_triangular(T[:k, :k], g[:k], lower=False)
        x = (b_norm / alpha) * (st.Q[:, :k].astype(np.float64) @ y)
        if precond is not None:
            x = precond.solve(x)
    res = float(np.linalg.norm(b - a_matvec(x)) / b_norm)
    conv = (res <= max(tol, 0.0)) if tol is not None else False
    return {"x": x, "history": np.asarray(hist), "final_residual": res, "iterations": k,
            "converged": conv or broke, "breakdown": broke, "R": st.R.copy(),
            "Q": st.Q.copy(), "alpha": alpha}


def oracle_gmres_lagged(matvec, n, b, m, theta, policy="mixed", tol=None, scale_by_norm=True):
    """One-synchronisation RGS-Arnoldi / RGS-GMRES (not in the
    reference package): Steps 5-7 of column c lag behind the next matvec, so the
    sketches s'_c = Theta q'_c and p'_{c+1} = Theta A q'_c are formed together
    from the *unnormalised* q'_c, then r_cc = ||s'_c||, s_c = s'_c / r_cc,
    q_c = q'_c / r_cc, p_{c+1} = p'_{c+1} / r_cc and w_{c+1} = A q'_c / r_cc.
    Everything else is krylov.py:229-319 (power estimate, Givens, stop test,
    x = (||b|| / alpha) Q y, true residual) and gram_schmidt.py:293-339 (step 2
    LS solve, step 3 in the coarse dtype, breakdown test against ||p||).
    ``scale_by_norm=False`` is arnoldi (krylov.py:176-199): b pushed as is, no
    1/alpha, no Givens."""
    from .ref_rgs import POLICIES, householder_lsq
    crs, fine_t, u_crs = POLICIES[policy]
    fine = np.dtype(fine_t)
    b = np.asarray(b, dtype=np.float64)
    b_norm = float(np.linalg.norm(b))
    alpha = 1.0
    if scale_by_norm:
        if b_norm == 0.0:
            return {"x": np.zeros(n), "history": np.zeros(0), "final_residual": 0.0,
                    "iterations": 0, "converged": True, "breakdown": False}
        alpha = power_norm_estimate(matvec, n)
        w = b / b_norm
    else:
        w = b
    k = theta.k
    Q = np.zeros((n, m + 1), dtype=crs)
    R = np.zeros((m + 1, m + 1))
    S = np.zeros((k, m + 1), dtype=fine)
    P = np.zeros((k, m + 1), dtype=fine)
    ls = householder_lsq(k, fine)
    bf = 10.0
    # column 0: q'_0 = w, s'_0 = p_0 (gram_schmidt.py:307-310)
    p = theta.apply(w).astype(fine)
    P[:, 0] = p
    qp = w.astype(crs)
    sp = p.copy()
    g = np.zeros(m + 1)
    T = np.zeros((m + 1, m))
    cs, sn = np.zeros(m), np.zeros(m)
    hist, broke, iters, ncols = [], False, 0, 0
    beta, unnormalised = None, -1
    for c in range(m + 1):
        # ---- finalize column c (steps 5-6; step 7 waits for the next update) ----
        r_cc = float(np.sqrt(np.sum(sp.astype(fine) * sp)))
        tol_b = bf * u_crs * float(np.linalg.norm(P[:, c]))
        if r_cc <= tol_b:
            broke = True
            break
        S[:, c] = sp / fine.type(r_cc)
        R[c, c] = r_cc
        ls.add(S[:, c])
        ncols = c + 1
        Q[:, c] = qp  # still q'_c
        unnormalised = c
        if c == 0:
            beta = r_cc
            g[0] = beta
        else:  # Givens of step c-1 on H[:, c-1] = R[:c+1, c] (krylov.py:281-300)
            i = c - 1
            iters = c
            if scale_by_norm:
                h = R[:i + 2, i + 1].copy()
                for j in range(i):
                    t = cs[j] * h[j] + sn[j] * h[j + 1]
                    h[j + 1] = -sn[j] * h[j] + cs[j] * h[j + 1]
                    h[j] = t
                rr = np.hypot(h[i], h[i + 1])
                if rr == 0.0:
                    cs[i], sn[i] = 1.0, 0.0
                else:
                    cs[i], sn[i] = h[i] / rr, h[i + 1] / rr
                h[i], h[i + 1] = rr, 0.0
                T[:i + 2, i] = h
                g[i + 1] = -sn[i] * g[i]
                g[i] = cs[i] * g[i]
                est = abs(g[i + 1]) / beta
                hist.append(est)
                if tol is not None and est <= tol:
                    break
        if c == m:
            break
        # ---- the lagged matvec and its sketch, from the unnormalised q'_c ----
        wp = matvec(qp.astype(np.float64))
        if scale_by_norm:
            wp = wp / alpha
        pp = theta.apply(wp)
        p = (pp / r_cc).astype(fine)
        P[:, c + 1] = p
        w = wp / r_cc
        Q[:, c] = (qp.astype(np.float64) / r_cc).astype(crs)  # step 7 of column c
        unnormalised = -1
        r = ls.solve(p)                                       # step 2
        qp = w.astype(crs) - Q[:, :c + 1] @ r.astype(crs)     # step 3
        sp = theta.apply(qp.astype(np.float64)).astype(fine)  # step 4
        R[:c + 1, c + 1] = r.astype(np.float64)
    # the newest committed column is still q' (its step 7 had no successor)
    if unnormalised >= 0:
        j = unnormalised
        Q[:, j] = (Q[:, j].astype(np.float64) / R[j, j]).astype(crs)
    Qm, Rm = Q[:, :ncols], R[:ncols, :ncols]
    out = {"Q": Qm.copy(), "R": Rm.copy(), "S": S[:, :ncols].copy(), "P": P[:, :ncols].copy(),
           "breakdown": broke, "iterations": iters}
    if not scale_by_norm:
        out["H"] = Rm[:, 1:].copy()
        return out
    kk = iters
    if kk == 0:
        x = np.zeros(n)
    else:
        y = scipy.linalg.solve_triangular(T[:kk, :kk], g[:kk], lower=False)
        x = (b_norm / alpha) * (Q[:, :kk].astype(np.float64) @ y)
    res = float(np.linalg.norm(b - matvec(x)) / b_norm)
    conv = (res <= max(tol, 0.0)) if tol is not None else False
    out.update({"x": x, "history": np.asarray(hist), "final_residual": res,
                "converged": conv or broke, "alpha": alpha})
    return out


def oracle_gmres_restarted(matvec, n, b, theta, policy="mixed", restart=300,
                           max_iters=3000, tol=1e-8, max_cycles=None, lagged=False):
    b = np.asarray(b, dtype=np.float64)
    b_norm = float(np.linalg.norm(b))
    x = np.zeros(n)
    r = b.copy()
    r_norm = b_norm
    its, cycles = 0, []
    while not (b_norm == 0.0 or r_norm / b_norm <= tol or its >= max_iters):
        if max_cycles is not None and len(cycles) >= max_cycles:
            break
        if lagged:
            out = oracle_gmres_lagged(matvec, n, r, min(restart, max_iters - its), theta, policy,
                                      tol=tol * b_norm / r_norm)
        else:
            out = oracle_gmres(matvec, n, r, min(restart, max_iters - its), theta, policy,
                               tol=tol * b_norm / r_norm)
        cycles.append(out["iterations"])
        its += out["iterations"]
        x = x + out["x"]
        r = b - matvec(x)
        r_norm = float(np.linalg.norm(r))
        if out["iterations"] == 0:
            break
    rel = r_norm / b_norm if b_norm else 0.0
    return {"x": x, "iterations": its, "cycles": cycles, "final_residual": rel}
