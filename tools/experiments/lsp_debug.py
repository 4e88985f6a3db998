"""Debug the persistent LS coupling: one small factorisation (eager, or
captured in a CUDA graph and replayed) with the debug timeline on; prints the
status block, the loop's flag and column counter, and per-column stamps (us
from column 0's entry; -1 = never)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2011_05090_b200 as sg
from paper_2011_05090_b200 import _lib, gram_schmidt as gsm
from paper_2011_05090_b200.workloads import make_w
gsm._LS_PERSIST = True
m = int(sys.argv[1]) if len(sys.argv) > 1 else 6
graph = len(sys.argv) > 2 and sys.argv[2] == "graph"
n, k = 5 * 4096 + 333, 200
W = make_w(n, m, 1e-6, 5, dtype=np.float32)
th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 6)
Wd = torch.from_numpy(np.ascontiguousarray(W.T)).cuda()
st = sg.RgsState(th, sg.MIXED32_64, capacity=m + 1, breakdown_factor=0.0)
st._reserve(m + 1)
tl = torch.zeros((m + 1, 16), dtype=torch.int64, device="cuda")
tl[:, 0] = 2**62
_lib.load().sgs_debug_timeline(tl.data_ptr())
if graph:
    g = st.capture_factorization(Wd, n, m)
    g.replay()
else:
    st._enqueue_factorization(Wd, n, m)
torch.cuda.synchronize()
_lib.load().sgs_debug_timeline(None)
print("status", st.status.read(), "flag", int(st._lsp[0]), "done", int(st._lsp[32 * 16]) & 0xffffffff,
      "col_ctas", st._col_ctas, flush=True)
t = tl.cpu().numpy().astype(np.float64)
t0 = t[0, 0]
for i in range(min(m, 12)):
    r = [(x - t0) / 1e3 if 0 < x < 2**61 else -1 for x in t[i, :7]]
    print(i, "col entry/after-wait/exit", [round(v, 1) for v in r[:3]], "ls pre/post/exit/entry",
          [round(v, 1) for v in r[3:7]])
