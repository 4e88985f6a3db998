"""Factor-kernel timing across structures (diag: no deps, tri: chain, cd: 3D stencil)."""
import json
import sys

import scipy.sparse
import torch

sys.path.insert(0, ".")
import paper_2011_05090_b200 as sg  # noqa: E402
from paper_2011_05090_b200 import _lib  # noqa: E402
from paper_2011_05090_b200.krylov import _ilu_analyse  # noqa: E402
from paper_2011_05090_b200.workloads import convdiff3d  # noqa: E402


def factor_only(A, reps=3):
    rp, ci, va = A.device_arrays()
    n = A.n
    ctl = torch.zeros(2, dtype=torch.int64, device="cuda")
    pl, pu = _ilu_analyse(n, rp, ci, ctl)
    F = torch.empty_like(va)
    diag = torch.empty(n, dtype=torch.int32, device="cuda")
    flags = torch.zeros(n, dtype=torch.int32, device="cuda")
    aux = torch.empty(2, dtype=torch.int64, device="cuda")
    f = lambda: _lib.call("sgs_ilu0_factor", n, rp.data_ptr(), ci.data_ptr(), va.data_ptr(),
                          F.data_ptr(), diag.data_ptr(), pl.data_ptr(), flags.data_ptr(),
                          ctl.data_ptr(), aux.data_ptr(), 1e-30, _lib.stream_ptr())
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


out = {}
n = 2 ** 21
out["diag"] = factor_only(sg.SparseMatrix.from_scipy(scipy.sparse.eye(n, format="csr") * 2.0))
for N in (32, 64, 128):
    rp, ci, va = convdiff3d(N)
    out[f"cd{N}"] = factor_only(sg.SparseMatrix(n=N ** 3, row_ptr=rp, col_idx=ci, values=va))
out["tri4096"] = factor_only(sg.SparseMatrix.from_scipy(
    scipy.sparse.diags([-1.0, 4.0, -1.0], [-1, 0, 1], shape=(4096, 4096), format="csr")))
print(json.dumps(out))
