"""Sweep-time scaling of the device ILU(0) solve: depth-bound (~3N) or row-bound (~N^3)?"""
import json
import sys

import numpy as np
import scipy.sparse
import torch

sys.path.insert(0, ".")
import paper_2011_05090_b200 as sg  # noqa: E402
from paper_2011_05090_b200.workloads import convdiff3d  # noqa: E402


def t_solve(pre, n, reps=5):
    v = torch.randn(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(v)
    pre.solve_into(v.data_ptr(), 1, y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        pre.solve_into(v.data_ptr(), 1, y)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


out = {}
for N in (16, 32, 64, 96, 128):
    rp, ci, va = convdiff3d(N)
    A = sg.SparseMatrix(n=N ** 3, row_ptr=rp, col_idx=ci, values=va)
    out[f"cd{N}"] = t_solve(sg.ilu0(A), A.n)
for n in (2 ** 16, 2 ** 21):
    A = sg.SparseMatrix.from_scipy(scipy.sparse.eye(n, format="csr") * 2.0)
    out[f"diag{n}"] = t_solve(sg.ilu0(A), n)
    # 1D chain (bidiagonal): depth n
for n in (2 ** 12, 2 ** 16):
    A = sg.SparseMatrix.from_scipy(scipy.sparse.diags([-1.0, 4.0, -1.0], [-1, 0, 1], shape=(n, n),
                                                      format="csr"))
    out[f"tri{n}"] = t_solve(sg.ilu0(A), n)
print(json.dumps(out))
