"""Per-phase cycle trace of the cluster LS kernel over one factorisation."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2011_05090_b200 as sg
from paper_2011_05090_b200.workloads import CONFIGS, make_w_device

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"]
n, m, k = cfg["n"], cfg["m"], cfg["k"]
pol = sg.policy_from_name(cfg["policy"])
th = sg.make_sketch(sg.SketchKind(cfg["kind"]), k, n, 0)
W = make_w_device(n, m, cfg["sigma_min"], 0,
                  torch.float32 if pol.coarse_dtype == np.float32 else torch.float64, "cuda")
for rep in range(2):
    st = sg.RgsState(th, pol, capacity=m + 1, breakdown_factor=cfg["breakdown_factor"])
    st._trace = torch.zeros((m + 1, 16), dtype=torch.int64, device="cuda")
    st.factorize_columns(W, W.shape[1], m)
tr = st._trace[:m].cpu().numpy().astype(np.float64)
names = {1: "prewait(cache,z,y)", 2: "wait", 3: "reduce_parts", 4: "exch1",
         5: "gather+s+matvec", 6: "exch2", 7: "reorth/fast path", 8: "rinv_col",
         9: "solve_prep", 10: "store"}
LAST = max(names)
out = {}
for dec, rows in enumerate(np.array_split(tr[1:-1], 5)):
    d = {}
    for ix in range(1, LAST + 1):
        prev = ix - 1
        while prev > 0 and np.all(rows[:, prev] == 0):
            prev -= 1
        ok = (rows[:, ix] > 0) & (rows[:, prev] > 0)
        if ok.any():
            d[names[ix]] = round(float(np.mean(rows[ok, ix] - rows[ok, prev])) / 1.965e3, 2)
    d["total_us"] = round(float(np.mean(rows[:, LAST] - rows[:, 0])) / 1.965e3, 2)
    d["post_wait_us"] = round(float(np.mean(rows[:, LAST] - rows[:, 2])) / 1.965e3, 2)
    out[f"quintile{dec}"] = d
for dec, rows in enumerate(np.array_split(tr[1:-1], 5)):
    d = out[f"quintile{dec}"]
    cyc = lambda a, b: round(float(np.mean(rows[:, b] - rows[:, a])) / 1.965e3, 2)  # noqa: E731
    d["pre:cache"] = cyc(0, 11)
    d["pre:deferred"] = cyc(11, 12)
    d["pre:coldot"] = cyc(12, 13)
    d["pre:gather+matvec"] = cyc(13, 1)
    d["exch1:norms"] = cyc(3, 14)
    d["exch1:coldot"] = cyc(14, 15)
    d["exch1:xsync"] = cyc(15, 4)
    if np.all(rows[:, 5] > 0) and np.all(rows[:, 6] > 0):  # fast-path launches
        d["fast:gather"] = cyc(4, 5)
        d["fast:s_write+coef"] = cyc(5, 6)
        d["fast:sums"] = cyc(6, 7)
print(json.dumps(out, indent=1))
