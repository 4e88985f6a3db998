"""Per-phase cycle trace of the cluster LS kernel over one c3 RGMRES cycle
(argv: policy [lagged]).  Lagged launches finalize c and solve c + 1."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2011_05090_b200 as sg
from paper_2011_05090_b200 import krylov as kr
from paper_2011_05090_b200.workloads import convdiff3d, rhs_gaussian

pol = sg.policy_from_name(sys.argv[1] if len(sys.argv) > 1 else "mixed")
lagged = len(sys.argv) > 2 and sys.argv[2] == "lagged"
m = 300
rp, ci, va = convdiff3d(128)
A = sg.SparseMatrix(n=128 ** 3, row_ptr=rp, col_idx=ci, values=va)
b = torch.from_numpy(rhs_gaussian(A.n, 0)).cuda()
th = sg.make_sketch(sg.SketchKind.PSRHT, 600, A.n, 0)
holder = {}
orig = kr._ArnoldiEngine.__init__


def init(self, *a, **kw):
    orig(self, *a, **kw)
    self.state._trace = torch.zeros((self.m + 3, 16), dtype=torch.int64, device="cuda")
    holder["st"] = self.state


kr._ArnoldiEngine.__init__ = init
for _ in range(2):
    sg.gmres(A, b, m=m, theta=th, policy=pol, lagged=lagged)
torch.cuda.synchronize()
tr = holder["st"]._trace[:m].cpu().numpy().astype(np.float64)
names = {1: "prewait(cache,z,y)", 2: "wait", 3: "reduce_parts", 4: "exch1",
         5: "gather+s+matvec", 6: "exch2", 7: "reorth/fast path", 8: "rinv_col",
         9: "solve_prep", 10: "store"}
out = {}
for dec, rows in enumerate(np.array_split(tr[2:-1], 4)):
    d = {}
    for ix in range(1, 11):
        prev = ix - 1
        while prev > 0 and np.all(rows[:, prev] == 0):
            prev -= 1
        ok = (rows[:, ix] > 0) & (rows[:, prev] > 0)
        if ok.any():
            d[names[ix]] = round(float(np.mean(rows[ok, ix] - rows[ok, prev])) / 1.965e3, 2)
    cyc = lambda a, b: round(float(np.mean(rows[:, b] - rows[:, a])) / 1.965e3, 2)  # noqa: E731
    d["pre:cache"] = cyc(0, 11)
    d["pre:deferred"] = cyc(11, 12)
    d["post_wait_us"] = cyc(2, 10)
    out[f"q{dec}"] = d
print(json.dumps(out))
