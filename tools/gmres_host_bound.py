"""Is the RGMRES loop host-bound?  Host time spent enqueuing vs device time."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2011_05090_b200 as sg  # noqa: E402
import paper_2011_05090_b200.krylov as kr  # noqa: E402
from paper_2011_05090_b200.workloads import CONFIGS, convdiff3d, rhs_gaussian  # noqa: E402

cfg = CONFIGS["c3"]
N = cfg["grid"]
rp, ci, va = convdiff3d(N)
A = sg.SparseMatrix(n=N ** 3, row_ptr=rp, col_idx=ci, values=va)
b = torch.from_numpy(rhs_gaussian(A.n, 0)).cuda()
th = sg.make_sketch(sg.SketchKind.PSRHT, cfg["k"], A.n, 0)
out = {}
for pol_name, pol in (("f64", sg.UNIFIED64), ("mixed", sg.MIXED32_64)):
    eng = kr._ArnoldiEngine(A, th, pol, sg.HOUSEHOLDER_QR, 300)
    ws = eng.ws
    alpha = kr._operator_norm_estimate(A, ws)
    bn = torch.ones(1, dtype=torch.float64, device="cuda")
    for rep in range(2):
        eng = kr._ArnoldiEngine(A, th, pol, sg.HOUSEHOLDER_QR, 300)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        eng.start(b, None)
        for i in range(300):
            eng.step(i, alpha, None)
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        out[pol_name] = {"host_enqueue_us_per_step": 1e6 * (t1 - t0) / 300,
                         "device_us_per_step": 1e3 * e0.elapsed_time(e1) / 300,
                         "wall_us_per_step": 1e6 * (t2 - t0) / 300}
print(json.dumps(out, indent=1))
