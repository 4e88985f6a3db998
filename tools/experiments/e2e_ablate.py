"""Ablation of the c1 pinned-host pipelined factorisation: which of the H2D
stream of W, the D2H stream of Q, and the chunked sketch structure costs the
e2e path its ~10 ms over the resident step.  Variants are built by textual
edits of RgsState.factorize_host_pipelined (experiment only)."""
import inspect
import json
import sys
import textwrap
import time

import torch

sys.path.insert(0, ".")
import paper_2011_05090_b200 as sg  # noqa: E402
import paper_2011_05090_b200.gram_schmidt as gsm  # noqa: E402
from paper_2011_05090_b200.workloads import CONFIGS, make_w_device  # noqa: E402

cfg = CONFIGS["c1"]
n, m, k = cfg["n"], cfg["m"], cfg["k"]
pol = sg.policy_from_name(cfg["policy"])
th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
dev = torch.device("cuda", 0)
Wt = make_w_device(n, m, cfg["sigma_min"], 0, torch.float32, dev)
th.device_data(dev)
pin = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
pin.copy_(Wt[:, :n])
gsm._ABL_WD = Wt[:, :n].contiguous()
del Wt
Wh = pin.numpy().T
src = textwrap.dedent(inspect.getsource(gsm.RgsState.factorize_host_pipelined))
orig = gsm.RgsState.factorize_host_pipelined


def variant(no_h2d=False, no_d2h=False, late=None, ship=None):
    s = src
    if no_h2d:
        s = s.replace("Wd = torch.empty((m, n), dtype=dt, device=self.device)", "Wd = _ABL_WD")
        s = s.replace("Wd[c0:c1].copy_(Wt[c0:c1], non_blocking=True)", "pass")
    if no_d2h:
        s = s.replace("Qh[c0:c1].copy_(self._Q[c0:c1, :n], non_blocking=True)", "pass")
    ns = {}
    exec(compile(s, "<variant>", "exec"), gsm.__dict__, ns)
    return ns["factorize_host_pipelined"]


out = {}


def timed(tag, reps=4):
    ts, dig = [], None
    for rep in range(reps):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        f, _ = sg.rgs_factorize(Wh, th, pol, with_certificate=False, breakdown_factor=0.0)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        dig = (float(np.asarray(f.R, dtype=np.float64).sum()),
               float(np.asarray(f.Q[::4099, :], dtype=np.float64).sum()),
               float(np.asarray(f.P, dtype=np.float64).sum()))
        del f
    out[tag] = {"ms": [round(t, 2) for t in ts[1:]], "min_ms": round(min(ts[1:]), 2), "digest": dig}
    print(tag, out[tag], flush=True)


import numpy as np  # noqa: E402
R = gsm.RgsState
import os  # noqa: E402
if os.environ.get("ABL_QUICK"):
    for name, kw in [("full", {}), ("neither", {"no_h2d": True, "no_d2h": True})]:
        R.factorize_host_pipelined = variant(**kw)
        timed(name)
    R.factorize_host_pipelined = orig
    print(json.dumps(out))
    sys.exit(0)
for defer in (False, True):
    R._e2e_defer_d2h = defer
    timed(f"defer{int(defer)}")
R._e2e_defer_d2h = True
for late in [(192, 32), (160, 32), (128, 32), (192, 48)]:
    R._e2e_late = late
    timed(f"late{late}")
R._e2e_late = (192, 64)
for ch in (4, 16):
    o = R.factorize_host_pipelined
    R.factorize_host_pipelined = lambda self, Wh, m, chunk=8, _o=o, _c=ch: _o(self, Wh, m, chunk=_c)
    timed(f"chunk{ch}")
    R.factorize_host_pipelined = o
print(json.dumps(out))
