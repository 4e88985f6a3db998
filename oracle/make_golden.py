"""Generate tests/golden/*.npz by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):
    python oracle/make_golden.py
The reference is imported unmodified from /root/reference/pkg/src with
single-threaded BLAS (as its tests/conftest.py:8-12 pins).  The fixtures pin
the oracle (tests/test_oracle_golden.py) and serve as golden vectors for the
GPU parity tests (tests/test_gpu_parity.py), which run where the reference
does not exist.
"""

import os
import sys

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMEXPR_NUM_THREADS"):
    os.environ[_v] = "1"

import numpy as np  # noqa: E402

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _problem(rng, n, m, cond):
    U, _ = np.linalg.qr(rng.standard_normal((n, m)))
    V, _ = np.linalg.qr(rng.standard_normal((m, m)))
    sv = np.logspace(0, -np.log10(cond), m)
    return (U * sv) @ V.T


def ilu_fixtures(sg):
    """ILU(0) factors, M^{-1} v and a preconditioned GMRES (krylov.py:86-151, :229-319)."""
    d = {}
    mats = {"lap6": sg.generate_laplacian_2d(6), "rs60": sg.generate_random_sparse(60, 4, seed=3),
            "rs300": sg.generate_random_sparse(300, 8, seed=2, diag_shift=0.1),
            "lap40": sg.generate_laplacian_2d(40)}
    for name, A in mats.items():
        pre = sg.ilu0(A)
        v = np.random.default_rng(A.n).standard_normal(A.n)
        full = (pre.L - sg.krylov.scipy.sparse.eye(A.n, format="csr") + pre.U).tocsr()
        full.sort_indices()
        d.update({f"{name}_rp": A.row_ptr, f"{name}_ci": A.col_idx, f"{name}_v": A.values,
                  f"{name}_Lrp": pre.L.indptr, f"{name}_Lci": pre.L.indices,
                  f"{name}_Lv": pre.L.data, f"{name}_Urp": pre.U.indptr,
                  f"{name}_Uci": pre.U.indices, f"{name}_Uv": pre.U.data,
                  f"{name}_sv": v, f"{name}_solve": pre.solve(v)})
    A = mats["lap40"]
    b = np.random.default_rng(0).standard_normal(A.n)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 200, A.n, seed=0)
    res = sg.gmres(A, b, m=60, theta=th, policy=sg.UNIFIED64, preconditioner=sg.ilu0(A),
                   tol=1e-12)
    d.update({"pg_b": b, "pg_x": res.x, "pg_its": res.iterations, "pg_res": res.final_residual,
              "pg_hist": res.residual_history})
    B = mats["rs300"]
    bb = np.random.default_rng(1).standard_normal(300)
    th2 = sg.make_sketch(sg.SketchKind.PSRHT, 200, 300, seed=0)
    r2 = sg.gmres(B, bb, m=40, theta=th2, policy=sg.MIXED32_64, preconditioner=sg.ilu0(B))
    d.update({"pr_b": bb, "pr_x": r2.x, "pr_its": r2.iterations, "pr_res": r2.final_residual,
              "pr_hist": r2.residual_history})
    # ZeroDivisionError / ValueError messages
    Z = sg.SparseMatrix.from_coo(3, [0, 0, 1, 1, 2], [0, 1, 0, 1, 2], [1.0, 1.0, 1.0, 1.0, 1.0])
    try:
        sg.ilu0(Z)
        d["zero_pivot_msg"] = np.array("")
    except ZeroDivisionError as e:
        d["zero_pivot_msg"] = np.array(str(e))
    np.savez_compressed(os.path.join(OUT, "ilu.npz"), **d)


def cert_fixtures(sg):
    """omega_bar / epsilon_of / certify_factorization (certification.py, sketch.py:213-228)."""
    d = {}
    n, dcols = 1024, 8
    theta = sg.make_sketch(sg.SketchKind.PSRHT, 96, n, seed=3)
    rng = np.random.default_rng(2024)
    for t in range(3):
        V = rng.standard_normal((n, dcols))
        phi = sg.make_certification_sketch(
            sg.CertificationParams(eps_star=0.25, delta_star=1e-3, phi_seed=t), n)
        Vt, Vp = theta.apply_block(V), phi.apply_block(V)
        d[f"V{t}"], d[f"Vt{t}"], d[f"Vp{t}"] = V, Vt, Vp
        d[f"ob{t}"] = sg.omega_bar(Vt, Vp, 0.25)
        d[f"om{t}"] = sg.epsilon_of(theta, V)
    W = rng.standard_normal((n, 10))
    th = sg.make_sketch(sg.SketchKind.PSRHT, 128, n, seed=0)
    phi = sg.make_certification_sketch(sg.CertificationParams(eps_star=0.25), n)
    f, _ = sg.rgs_factorize(W, th, sg.UNIFIED64, phi=phi)
    res = sg.certify_factorization(f, eps_star=0.25, u_crs=sg.UNIFIED64.u_crs)
    d.update({"cf_W": W, "cf_S": f.S, "cf_Sphi": f.S_phi, "cf_P": f.P, "cf_Pphi": f.P_phi,
              "cf_Q": f.Q, "cf_obq": res.omega_bar_q, "cf_obw": res.omega_bar_w,
              "cf_mq": res.margin_q, "cf_mw": res.margin_w})
    d["eps_inv"] = np.array([sg.eps_star_for_dim(sg.vector_certificate_dim(e, 1e-3), 1e-3)
                             for e in (0.05, 0.1, 0.25, 0.5)])
    np.savez_compressed(os.path.join(OUT, "cert.npz"), **d)


def main(only=None):
    sys.path.insert(0, REF)
    import sketchgs as sg
    if only in ("ilu", "cert"):
        os.makedirs(OUT, exist_ok=True)
        (ilu_fixtures if only == "ilu" else cert_fixtures)(sg)
        print(only, "fixtures written to", os.path.abspath(OUT))
        return
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
    from paper_2011_05090_b200.workloads import make_w, convdiff3d, rhs_gaussian
    os.makedirs(OUT, exist_ok=True)

    # ---- FWHT (sketch.py:90-109) -------------------------------------------------
    rng = np.random.default_rng(7)
    d = {"kat_in": np.array([1.0, 2.0, 3.0, 4.0]),
         "kat_out": sg.fwht(np.array([1.0, 2.0, 3.0, 4.0]))}
    for s in (1, 2, 8, 64, 1024, 4096, 16384):
        x = rng.standard_normal(s)
        d[f"x_{s}"] = x
        d[f"y_{s}"] = sg.fwht(x)
    X = rng.standard_normal((64, 3))
    d["X_mat"] = X
    d["Y_mat"] = sg.fwht(X)
    np.savez_compressed(os.path.join(OUT, "fwht.npz"), **d)

    # ---- P-SRHT construction + apply (sketch.py:123-198) --------------------------
    d = {}
    cases = [(10, 24, 9), (40, 100, 11), (16, 24, 0), (96, 400, 3), (200, 256, 0),
             (600, 5000, 1), (64, 4096, 5), (300, 20000, 2)]
    d["cases"] = np.array(cases)
    for (k, n, seed) in cases:
        th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, seed)
        r = np.random.default_rng(k * 7 + n)
        x = r.standard_normal(n)
        Xb = r.standard_normal((n, 3))
        tag = f"{k}_{n}_{seed}"
        d[f"signs_{tag}"] = th.signs
        d[f"samples_{tag}"] = th.sample_indices
        d[f"x_{tag}"] = x
        d[f"y_{tag}"] = th.apply(x)
        d[f"X_{tag}"] = Xb
        d[f"Y_{tag}"] = th.apply_block(Xb)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 16, 24, 0)
    d["materialize_16_24_0"] = th.materialize()
    th = sg.make_sketch(sg.SketchKind.RADEMACHER, 20, 50, 5)
    d["rad_materialize_20_50_5"] = th.materialize()
    np.savez_compressed(os.path.join(OUT, "psrht.npz"), **d)

    # ---- rgs_factorize (gram_schmidt.py:350-375) -----------------------------------
    pol = {"f64": sg.UNIFIED64, "mixed": sg.MIXED32_64, "f32": sg.UNIFIED32}
    specs = [
        # name, n, m, cond, kind, k, seed, policy, bf
        ("psrht_f64", 400, 12, 100.0, "psrht", 96, 3, "f64", 10.0),
        ("psrht_mixed", 400, 12, 1e4, "psrht", 128, 0, "mixed", 10.0),
        ("rad_f64", 400, 12, 100.0, "rademacher", 128, 1, "f64", 10.0),
        ("psrht_f32", 400, 12, 1e3, "psrht", 96, 4, "f32", 10.0),
        ("psrht_mixed_wide", 3000, 40, 1e5, "psrht", 200, 8, "mixed", 0.0),
    ]
    for name, n, m, cond, kind, k, seed, pname, bf in specs:
        W = _problem(np.random.default_rng(12345), n, m, cond)
        th = sg.make_sketch(sg.SketchKind.PSRHT if kind == "psrht" else sg.SketchKind.RADEMACHER,
                            k, n, seed)
        f, cert = sg.rgs_factorize(W, th, pol[pname], breakdown_factor=bf)
        np.savez_compressed(os.path.join(OUT, f"rgs_{name}.npz"), W=W, Q=f.Q, R=f.R, S=f.S,
                            P=f.P, meta=np.array([n, m, k, seed]), kind=kind, policy=pname,
                            bf=bf, cert=np.array([cert.delta_m, cert.delta_tilde_m, cert.cond_S]))
    # BASELINE-style W (G diag(sigma) V^T), mixed, SRHT, benchmark protocol bf=0
    n, m, k = 8192, 64, 256
    W = make_w(n, m, 1e-10, 11, dtype=np.float32)
    th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 11)
    f, cert = sg.rgs_factorize(W, th, sg.MIXED32_64, breakdown_factor=0.0)
    np.savez_compressed(os.path.join(OUT, "rgs_c1shape_mixed.npz"), W=W, Q=f.Q, R=f.R, S=f.S,
                        P=f.P, meta=np.array([n, m, k, 11]), kind="psrht", policy="mixed",
                        bf=0.0, cert=np.array([cert.delta_m, cert.delta_tilde_m, cert.cond_S]))
    # breakdown on an exactly repeated column (test_gram_schmidt.py:69-75)
    W = _problem(np.random.default_rng(12345), 200, 4, 1e4)
    W = np.concatenate([W, W[:, :1]], axis=1)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 64, 200, 5)
    try:
        sg.rgs_factorize(W, th, sg.UNIFIED64)
        col = -1
    except sg.BreakdownError as e:
        col = e.column
    np.savez_compressed(os.path.join(OUT, "rgs_breakdown.npz"), W=W, column=col)

    # ---- Krylov (krylov.py:176-319) -------------------------------------------------
    A = sg.generate_laplacian_2d(16)
    xs = np.sin(np.arange(A.n) * 0.1)
    b = A.matvec(xs)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 200, A.n, 0)
    res = sg.gmres(A, b, m=150, theta=th, policy=sg.UNIFIED64, tol=1e-12)
    d = {"lap_rp": A.row_ptr, "lap_ci": A.col_idx, "lap_v": A.values, "lap_b": b,
         "lap_x": res.x, "lap_hist": res.residual_history, "lap_res": res.final_residual,
         "lap_its": res.iterations, "lap_R": res.factors.R}
    B = sg.generate_random_sparse(200, 5, seed=1)
    bb = np.random.default_rng(12345).standard_normal(200)
    th2 = sg.make_sketch(sg.SketchKind.PSRHT, 64, 200, 0)
    dec = sg.arnoldi(B, bb, 15, variant=sg.GsVariant.RGS, theta=th2, policy=sg.UNIFIED64)
    d.update({"rs_rp": B.row_ptr, "rs_ci": B.col_idx, "rs_v": B.values, "rs_b": bb,
              "rs_Q": dec.Q, "rs_H": dec.H, "rs_beta": dec.beta})
    A12 = sg.generate_laplacian_2d(12)
    b12 = np.random.default_rng(12345).standard_normal(A12.n)
    th3 = sg.make_sketch(sg.SketchKind.PSRHT, 140, A12.n, 0)
    r12 = sg.gmres(A12, b12, m=120, theta=th3, policy=sg.MIXED32_64)
    d.update({"l12_rp": A12.row_ptr, "l12_ci": A12.col_idx, "l12_v": A12.values, "l12_b": b12,
              "l12_res": r12.final_residual, "l12_its": r12.iterations,
              "l12_hist": r12.residual_history})
    # 3D conv-diff at 16^3 with the restart wrapper structure (one gmres cycle)
    rp, ci, va = convdiff3d(16)
    A3 = sg.SparseMatrix(n=16 ** 3, row_ptr=rp, col_idx=ci, values=va)
    b3 = rhs_gaussian(A3.n, 0)
    th4 = sg.make_sketch(sg.SketchKind.PSRHT, 200, A3.n, 0)
    r3 = sg.gmres(A3, b3, m=100, theta=th4, policy=sg.UNIFIED64, tol=1e-8)
    d.update({"cd_b": b3, "cd_x": r3.x, "cd_its": r3.iterations, "cd_res": r3.final_residual,
              "cd_hist": r3.residual_history})
    np.savez_compressed(os.path.join(OUT, "krylov.npz"), **d)
    ilu_fixtures(sg)
    cert_fixtures(sg)
    print("golden fixtures written to", os.path.abspath(OUT))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
