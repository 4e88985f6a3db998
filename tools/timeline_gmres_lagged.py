"""Per-step timeline of one one-synchronisation RGMRES cycle (config 3,
gmres(lagged=True)) from %globaltimer stamps.  Row c holds: [0..2] column
kernel c (start, after its dependency wait, end), [9,10] SpMV of q'_c,
[12,13] SRHT of w, [6,3,4,5] the LS launch finalizing c / solving c+1 (start,
pre-wait done, wait done, end), [11] Givens."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2011_05090_b200 as sg
from paper_2011_05090_b200 import _lib
from paper_2011_05090_b200 import krylov as kr
from paper_2011_05090_b200.workloads import convdiff3d, rhs_gaussian

pol = sg.policy_from_name(sys.argv[1] if len(sys.argv) > 1 else "f64")
m = 300
rp, ci, va = convdiff3d(128)
A = sg.SparseMatrix(n=128 ** 3, row_ptr=rp, col_idx=ci, values=va)
b = torch.from_numpy(rhs_gaussian(A.n, 0)).cuda()
th = sg.make_sketch(sg.SketchKind.PSRHT, 600, A.n, 0)
sg.gmres(A, b, m=20, theta=th, policy=pol, lagged=True)
tl = torch.zeros((m + 3, 16), dtype=torch.int64, device="cuda")
for c in (0, 1, 9, 12):
    tl[:, c] = 2**62
lib = _lib.load()
orig = kr._ArnoldiEngine._step_lagged


def step(self, i, alpha, tol):
    lib.sgs_debug_timeline_col(i + 1)
    return orig(self, i, alpha, tol)


kr._ArnoldiEngine._step_lagged = step
lib.sgs_debug_timeline(tl.data_ptr())
res = sg.gmres(A, b, m=m, theta=th, policy=pol, lagged=True)
torch.cuda.synchronize()
lib.sgs_debug_timeline(None)
t = tl.cpu().numpy().astype(np.float64) / 1e3
rows = []
for r in range(3, m - 1):
    rows.append((t[r, 1] - t[r, 0], t[r, 2] - t[r, 1], t[r, 10] - t[r, 9], t[r, 13] - t[r, 12],
                 t[r, 3] - t[r, 6], t[r, 5] - t[r, 4],
                 t[r, 9] - t[r, 2], t[r, 12] - t[r, 10], t[r, 4] - t[r, 13],
                 t[r + 1, 1] - t[r, 5], t[r + 1, 9] - t[r, 9]))
names = ["col_prewait", "column", "spmv", "srht", "ls_prewait", "ls_postwait", "col->spmv",
         "spmv->srht", "srht->ls", "ls->next_col(givens)", "period"]
a = np.array(rows)
out = {f"q{q}": dict(zip(names, [round(float(x), 2) for x in p.mean(0)]))
       for q, p in enumerate(np.array_split(a, 4))}
out["mean"] = dict(zip(names, [round(float(x), 2) for x in a.mean(0)]))
out["iterations"] = res.iterations
print(json.dumps(out, indent=1))
