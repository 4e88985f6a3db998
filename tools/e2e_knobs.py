"""Sweep the pipelined end-to-end path's chunk / ship knobs at c1 and report
the per-column lag against the resident factorisation."""
import itertools
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2011_05090_b200 as sg  # noqa: E402
from paper_2011_05090_b200 import _lib  # noqa: E402
from paper_2011_05090_b200.gram_schmidt import RgsState  # noqa: E402
from paper_2011_05090_b200.workloads import CONFIGS, make_w_device  # noqa: E402

cfg = CONFIGS["c1"]
n, m, k = cfg["n"], cfg["m"], cfg["k"]
pol = sg.policy_from_name(cfg["policy"])
th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
W = make_w_device(n, m, cfg["sigma_min"], 0, torch.float32, "cuda")
lib = _lib.load()
tl = torch.zeros((m + 1, 16), dtype=torch.int64, device="cuda")


def timeline(fn):
    tl.zero_()
    tl[:, 0] = 2**62
    tl[:, 1] = 2**62
    lib.sgs_debug_timeline(tl.data_ptr())
    fn()
    torch.cuda.synchronize()
    lib.sgs_debug_timeline(None)
    t = tl.cpu().numpy().astype(np.float64) / 1e3
    go = t[:m, 1]
    return go - go[0]


st = RgsState(th, pol, capacity=m + 1, breakdown_factor=0.0)


def resident():
    st.m = 0
    st.factorize_columns(W, W.shape[1], m)


resident()
res = timeline(resident)
del st
torch.cuda.empty_cache()
pin = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
pin.copy_(W[:, :n])
Wh = pin.numpy().T
cols = (50, 100, 200, 300, 499)
print("resident", [round(res[c]) for c in cols])
for ship, late, early in itertools.product((8, 32, 10**6), ((192, 64), (96, 32), (10**6, 8)), (8, 16)):
    RgsState._e2e_ship = ship
    RgsState._e2e_late = late
    f = lambda: sg.rgs_factorize(Wh, th, pol, with_certificate=False, breakdown_factor=0.0)  # noqa: E731
    import paper_2011_05090_b200.gram_schmidt as gs
    orig = gs.RgsState.factorize_host_pipelined
    gs.RgsState.factorize_host_pipelined = lambda self, Wh, m, chunk=8, _o=orig, _e=early: _o(self, Wh, m, _e)
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        f()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    e = timeline(f)
    gs.RgsState.factorize_host_pipelined = orig
    print(f"ship={ship} late={late} early={early} ms={min(ts):.2f} lag=",
          [round(e[c] - res[c]) for c in cols], flush=True)
