"""Per-column timeline of one c1 factorisation from %globaltimer stamps:
column kernel (first CTA entry, first CTA past the dependency wait, last CTA
exit) and the LS launch (entry, past the wait, exit)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2011_05090_b200 as sg
from paper_2011_05090_b200 import _lib
from paper_2011_05090_b200.workloads import CONFIGS, make_w_device

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"]
n, m, k = cfg["n"], cfg["m"], cfg["k"]
if len(sys.argv) > 2:  # override n (e.g. grids that fit beside a resident LS cluster)
    n = int(sys.argv[2])
pol = sg.policy_from_name(cfg["policy"])
th = sg.make_sketch(sg.SketchKind(cfg["kind"]), k, n, 0)
W = make_w_device(n, m, cfg["sigma_min"], 0,
                  torch.float32 if pol.coarse_dtype == np.float32 else torch.float64, "cuda")
st = sg.RgsState(th, pol, capacity=m + 1, breakdown_factor=cfg["breakdown_factor"])
st.factorize_columns(W, W.shape[1], m)
tl = torch.zeros((m + 1, 16), dtype=torch.int64, device="cuda")
tl[:, 0] = 2**62
tl[:, 1] = 2**62
_lib.load().sgs_debug_timeline(tl.data_ptr())
st.m = 0
st.factorize_columns(W, W.shape[1], m)
torch.cuda.synchronize()
_lib.load().sgs_debug_timeline(None)
t = tl.cpu().numpy().astype(np.float64) / 1e3  # us
# columns 1..m-1: col kernel i: [0]=entry [1]=after wait [2]=exit ; LS i: [3] entry [4] after wait [5] exit
t = t[:, :8]
rows = []
for i in range(2, m - 1):
    col_run = t[i, 2] - t[i, 1]
    ls_post = t[i, 5] - t[i, 4]
    gap_col_to_ls = t[i, 4] - t[i, 2]      # LS passes its wait after the column kernel's last exit
    gap_ls_to_col = t[i + 1, 1] - t[i, 5]  # next column kernel passes its wait after the LS exit
    period = t[i + 1, 1] - t[i, 1]
    window = t[i + 1, 1] - t[i + 1, 0]     # next column kernel: entry -> past its wait
    ls_to_entry = t[i + 1, 0] - t[i, 4]    # LS past its wait -> next column kernel entry
    ls_entry = t[i, 6] - t[i, 2]           # LS entry relative to the column kernel's last exit
    ls_pre = t[i, 3] - t[i, 2]             # LS pre-wait work done, relative to that exit
    rows.append((col_run, ls_post, gap_col_to_ls, gap_ls_to_col, period, window, ls_to_entry,
                 ls_entry, ls_pre))
a = np.array(rows)
out = {}
for q, part in enumerate(np.array_split(a, 5)):
    out[f"quintile{q}"] = dict(zip(["col_run", "ls_post", "col_exit->ls_go", "ls_exit->col_go",
                                    "period", "prewait_window", "ls_go->col_entry",
                                    "ls_entry-col_exit", "ls_ready-col_exit"],
                                   [round(float(x), 2) for x in part.mean(0)]))
out["mean"] = dict(zip(["col_run", "ls_post", "col_exit->ls_go", "ls_exit->col_go", "period",
                        "prewait_window", "ls_go->col_entry", "ls_entry-col_exit", "ls_ready-col_exit"],
                       [round(float(x), 2) for x in a.mean(0)]))
print(json.dumps(out, indent=1))
