"""Per-solve times of c3 restarted RGMRES (fp64 and fp32 bases) with SM clocks."""
import json
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
import paper_2011_05090_b200 as sg  # noqa: E402
from paper_2011_05090_b200.workloads import CONFIGS, convdiff3d, rhs_gaussian  # noqa: E402

cfg = CONFIGS["c3"]
N = cfg["grid"]
rp, ci, va = convdiff3d(N)
A = sg.SparseMatrix(n=N ** 3, row_ptr=rp, col_idx=ci, values=va)
A.device_arrays()
b = torch.from_numpy(rhs_gaussian(A.n, 0)).cuda()
th = sg.make_sketch(sg.SketchKind.PSRHT, cfg["k"], A.n, 0)
th.device_data("cuda")
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        try:
            o = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks_throttle_reasons.active",
                                "--format=csv,noheader,nounits"], capture_output=True, text=True,
                               timeout=5).stdout.strip()
            samples.append((time.perf_counter(), o))
        except Exception:
            pass
        time.sleep(0.05)


th_s = threading.Thread(target=sampler, daemon=True)
th_s.start()
out = []
for pol_name, pol in (("f64", sg.UNIFIED64), ("mixed", sg.MIXED32_64)) * 3:
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = sg.gmres_restarted(A, b, th, pol, restart=300, max_iters=3000, tol=1e-8)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        clk = [s for (t, s) in samples if t0 <= t <= t1]
        out.append((pol_name, round(1e3 * (t1 - t0), 1), res.iterations, clk[:3]))
stop.set()
for o in out:
    print(o)
