"""Per-column device timeline of the pinned end-to-end factorisation vs the
resident one (c1): where does the end-to-end time go?"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2011_05090_b200 as sg  # noqa: E402
from paper_2011_05090_b200 import _lib  # noqa: E402
from paper_2011_05090_b200.workloads import CONFIGS, make_w_device  # noqa: E402

cfg = CONFIGS["c1"]
n, m, k = cfg["n"], cfg["m"], cfg["k"]
pol = sg.policy_from_name(cfg["policy"])
th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
W = make_w_device(n, m, cfg["sigma_min"], 0, torch.float32, "cuda")
lib = _lib.load()


def run(fn):
    tl = torch.zeros((m + 1, 16), dtype=torch.int64, device="cuda")
    tl[:, 0] = 2**62
    tl[:, 1] = 2**62
    fn()
    torch.cuda.synchronize()
    lib.sgs_debug_timeline(tl.data_ptr())
    fn()
    torch.cuda.synchronize()
    lib.sgs_debug_timeline(None)
    t = tl.cpu().numpy().astype(np.float64) / 1e3
    go = t[:m, 1]  # column kernel past its wait
    return go - go[0]


st = sg.RgsState(th, pol, capacity=m + 1, breakdown_factor=0.0)


def resident():
    st.m = 0
    st.factorize_columns(W, W.shape[1], m)


res = run(resident)
del st
torch.cuda.empty_cache()
pin = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
pin.copy_(W[:, :n])
Wh = pin.numpy().T
e2e = run(lambda: sg.rgs_factorize(Wh, th, pol, with_certificate=False, breakdown_factor=0.0))
out = {c: {"resident_us": round(float(res[c]), 1), "e2e_us": round(float(e2e[c]), 1),
           "lag_us": round(float(e2e[c] - res[c]), 1)}
       for c in (1, 10, 50, 100, 150, 200, 250, 300, 400, 499)}
print(json.dumps(out, indent=1))
