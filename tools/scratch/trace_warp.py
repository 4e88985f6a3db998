import json, os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2011_05090_b200 as sg
from paper_2011_05090_b200.workloads import CONFIGS, make_w_device
cfg = CONFIGS["c1"]
n, m, k = cfg["n"], cfg["m"], cfg["k"]
pol = sg.policy_from_name(cfg["policy"])
th = sg.make_sketch(sg.SketchKind(cfg["kind"]), k, n, 0)
W = make_w_device(n, m, cfg["sigma_min"], 0, torch.float32, "cuda")
for rep in range(2):
    st = sg.RgsState(th, pol, capacity=m + 1, breakdown_factor=cfg["breakdown_factor"])
    st._trace = torch.zeros((m + 1, 64), dtype=torch.int64, device="cuda")
    st.factorize_columns(W, W.shape[1], m)
tr = st._trace[:m].cpu().numpy().astype(np.float64)
np.set_printoptions(linewidth=250, precision=2, suppress=True)
for rows in (tr[40:60], tr[400:420]):
    base = rows[:, 3:4]
    print("rep0 start - TR3:", np.mean(rows[:, 16:32] - base, axis=0) / 1.965e3)
    print("rep1 start - TR3:", np.mean(rows[:, 32:48] - base, axis=0) / 1.965e3)
    print("end - TR3:", np.mean(rows[:, 48:64] - base, axis=0) / 1.965e3)
