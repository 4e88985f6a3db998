"""c1 e2e time vs the pipelined path's chunk / ship granularity."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2011_05090_b200 as sg  # noqa: E402
from paper_2011_05090_b200.workloads import CONFIGS, make_w_device  # noqa: E402

cfg = CONFIGS["c1"]
n, m, k = cfg["n"], cfg["m"], cfg["k"]
pol = sg.policy_from_name(cfg["policy"])
th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
Wt = make_w_device(n, m, cfg["sigma_min"], 0, torch.float32, torch.device("cuda", 0))
th.device_data("cuda")
pin = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
pin.copy_(Wt[:, :n])
Wh = pin.numpy().T
del Wt
torch.cuda.empty_cache()
out = {}
for late, lc, ship in ((192, 64, 8), (10**9, 8, 8), (192, 64, 16), (192, 64, 32), (96, 64, 8),
                       (192, 128, 8), (0, 8, 10**9)):
    sg.RgsState._e2e_late = (late, lc)
    sg.RgsState._e2e_ship = ship
    ts = []
    for rep in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f, _ = sg.rgs_factorize(Wh, th, pol, with_certificate=False, breakdown_factor=0.0)
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
        del f
    out[f"late{late}_lc{lc}_ship{ship}"] = round(min(ts[2:]), 2)
print(json.dumps(out, indent=1))
