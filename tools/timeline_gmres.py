"""Per-step timeline of one RGMRES cycle (config 3) from %globaltimer stamps.
Row i+1 holds: [0..2] column kernel i+1, [3..5] LS finalize i+1, [6..8] LS
solve i+1, [9,10] SpMV of step i, [11] Givens of step i."""
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
sg.gmres(A, b, m=20, theta=th, policy=pol)
tl = torch.zeros((m + 3, 16), dtype=torch.int64, device="cuda")
tl[:, 0] = 2**62
tl[:, 1] = 2**62
tl[:, 9] = 2**62
tl[:, 12] = 2**62
lib = _lib.load()
orig = kr._ArnoldiEngine.step


def step(self, i, alpha, tol):
    lib.sgs_debug_timeline_col(i + 1)
    return orig(self, i, alpha, tol)


kr._ArnoldiEngine.step = step
lib.sgs_debug_timeline(tl.data_ptr())
res = sg.gmres(A, b, m=m, theta=th, policy=pol)
torch.cuda.synchronize()
lib.sgs_debug_timeline(None)
t = tl.cpu().numpy().astype(np.float64) / 1e3
rows = []
for r in range(3, m - 1):
    spmv = t[r, 10] - t[r, 9]
    solve = t[r, 8] - t[r, 7]
    col = t[r, 2] - t[r, 1]
    fin = t[r, 5] - t[r, 4]
    giv_done = t[r, 11]
    period = t[r + 1, 9] - t[r, 9]
    gaps = period - spmv - solve - col - fin
    srht = t[r, 13] - t[r, 12]
    rows.append((spmv, srht, solve, col, fin, t[r, 12] - t[r, 10], t[r, 7] - t[r, 13],
                 t[r, 1] - t[r, 8], t[r, 4] - t[r, 2], t[r + 1, 9] - t[r, 5], period))
names = ["spmv", "srht", "ls_solve", "column", "ls_fin", "spmv->srht", "srht->solve",
         "solve->col", "col->fin", "fin->next_spmv(givens)", "period"]
a = np.array(rows)
out = {f"q{q}": dict(zip(names, [round(float(x), 2) for x in p.mean(0)]))
       for q, p in enumerate(np.array_split(a, 4))}
out["mean"] = dict(zip(names, [round(float(x), 2) for x in a.mean(0)]))
print(json.dumps(out, indent=1))
