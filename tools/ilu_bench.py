"""Timing of the device ILU(0) path at BASELINE c3's 128^3 conv-diff operator:
factorization, one M^{-1} v solve, and preconditioned restarted RGMRES, with
scipy's triangular solves (the reference's Ilu0Preconditioner.solve) beside."""

import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2011_05090_b200 as sg  # noqa: E402
from paper_2011_05090_b200.workloads import convdiff3d, rhs_gaussian  # noqa: E402


def ev_time(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    rp, ci, va = convdiff3d(N)
    A = sg.SparseMatrix(n=N ** 3, row_ptr=rp, col_idx=ci, values=va)
    A.device_arrays()
    out = {"N": N, "n": A.n}
    from paper_2011_05090_b200.krylov import _ilu_analyse
    rpd, cid, _ = A.device_arrays()
    ctl = torch.zeros(2, dtype=torch.int64, device="cuda")
    out["analyse_ms"] = ev_time(lambda: _ilu_analyse(A.n, rpd, cid, ctl), 3)
    out["factor_ms"] = ev_time(lambda: sg.ilu0(A), 3)
    pre = sg.ilu0(A)
    v = torch.from_numpy(rhs_gaussian(A.n, 0)).cuda()
    y = torch.empty_like(v)
    out["solve_ms"] = ev_time(lambda: pre.solve_into(v.data_ptr(), 1, y), 10)
    out["spmv_ms"] = ev_time(lambda: A.spmv_into(v.data_ptr(), 1, y), 10)
    L, U = pre.L, pre.U
    vh = v.cpu().numpy()
    import scipy.sparse.linalg as spla
    t = time.perf_counter()
    spla.spsolve_triangular(U, spla.spsolve_triangular(L, vh, lower=True, unit_diagonal=True),
                            lower=False)
    out["scipy_solve_ms"] = (time.perf_counter() - t) * 1e3
    if len(sys.argv) > 2:
        print(json.dumps(out))
        return
    b = rhs_gaussian(A.n, 0)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 2000 if N == 128 else 200, A.n, 0)
    for pol_name, pol in (("f64", sg.UNIFIED64), ("mixed", sg.MIXED32_64)):
        torch.cuda.synchronize()
        t = time.perf_counter()
        res = sg.gmres_restarted(A, b, th, pol, restart=300, max_iters=3000, tol=1e-8,
                                 preconditioner=pre)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        out[f"pgmres_{pol_name}"] = {"iterations": res.iterations, "cycles": res.cycles,
                                     "residual": res.final_residual, "s": dt,
                                     "steps_per_s": res.iterations / dt}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
