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
    st._trace = torch.zeros((m + 1, 16), dtype=torch.int64, device="cuda")
    st.factorize_columns(W, W.shape[1], m)
tr = st._trace[:m].cpu().numpy().astype(np.float64)
for dec, rows in enumerate(np.array_split(tr[1:-1], 5)):
    cyc = lambda a, b: round(float(np.mean(rows[:, b] - rows[:, a])) / 1.965e3, 2)
    print(dec, "wait->reduce", cyc(2,3), "loop", cyc(3,11), "bsum2", cyc(11,12), "tr", cyc(12,13), "store", cyc(13,14), "coldot", cyc(14,15), "xsync", cyc(15,4))
