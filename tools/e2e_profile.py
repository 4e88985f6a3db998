"""Where the c1 end-to-end time goes: events on the compute stream around the
pinned-host pipelined rgs_factorize, against the resident eager and graph steps."""
import json
import sys
import time

import numpy as np
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
out = {}

# resident eager (no graph)
st = sg.RgsState(th, pol, capacity=m + 1, breakdown_factor=0.0)
for rep in range(3):
    st.m = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st.factorize_columns(Wt, Wt.shape[1], m)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out["eager_ms"] = 1e3 * (t2 - t0)
    out["eager_host_enqueue_ms"] = 1e3 * (t1 - t0)
del st
torch.cuda.empty_cache()

pin = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
pin.copy_(Wt[:, :n])
Wh = pin.numpy().T
del Wt
torch.cuda.empty_cache()
marks = {}
orig_col = gsm.RgsState._column


def col(self, i, *a, **kw):
    if i in (0, 25, 50, 100, 150, 200, 250, 300, 400, m - 1):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks[f"col{i}_enq"] = (e, time.perf_counter())
    return orig_col(self, i, *a, **kw)


gsm.RgsState._column = col
orig_norm, orig_sync = gsm.RgsState._normalize, gsm.RgsState._sync_status


def norm(self, *a, **kw):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    marks["normalize_enq"] = (e, time.perf_counter())
    return orig_norm(self, *a, **kw)


def sync(self, *a, **kw):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    marks["sync_enq"] = (e, time.perf_counter())
    r = orig_sync(self, *a, **kw)
    e2 = torch.cuda.Event(enable_timing=True)
    e2.record()
    marks["sync_done"] = (e2, time.perf_counter())
    return r


gsm.RgsState._normalize = norm
gsm.RgsState._sync_status = sync
for rep in range(4):
    marks.clear()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record()
    h0 = time.perf_counter()
    f, _ = sg.rgs_factorize(Wh, th, pol, with_certificate=False, breakdown_factor=0.0)
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record()
    torch.cuda.synchronize()
    h1 = time.perf_counter()
    res = {"total_host_ms": 1e3 * (h1 - h0), "total_dev_ms": e0.elapsed_time(e1)}
    for key, (e, h) in marks.items():
        res[key + "_dev_ms"] = e0.elapsed_time(e)
        res[key + "_host_ms"] = 1e3 * (h - h0)
    out[f"e2e_rep{rep}"] = res
gsm.RgsState._column = orig_col
print(json.dumps(out, indent=1))
