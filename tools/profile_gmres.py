"""Kernel timeline of one RGMRES cycle on config 3 (CUPTI via torch.profiler)."""
import collections, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
import paper_2011_05090_b200 as sg
from paper_2011_05090_b200.workloads import convdiff3d, rhs_gaussian

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
pol = sg.policy_from_name(sys.argv[2] if len(sys.argv) > 2 else "f64")
m = int(sys.argv[3]) if len(sys.argv) > 3 else 300
rp, ci, va = convdiff3d(N)
A = sg.SparseMatrix(n=N ** 3, row_ptr=rp, col_idx=ci, values=va)
b = torch.from_numpy(rhs_gaussian(A.n, 0)).cuda()
th = sg.make_sketch(sg.SketchKind.PSRHT, 600, A.n, 0)
sg.gmres(A, b, m=20, theta=th, policy=pol)
torch.cuda.synchronize()
t0 = time.perf_counter()
res = sg.gmres(A, b, m=m, theta=th, policy=pol)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    res = sg.gmres(A, b, m=m, theta=th, policy=pol)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern = sorted([(e.time_range.start, e.time_range.end, e.name) for e in evs])
agg = collections.defaultdict(lambda: [0, 0.0])
for s, e, nm in kern:
    key = nm.split("<")[0].split("(")[0].replace("void ", "").replace("sgs::", "")[:60]
    agg[key][0] += 1
    agg[key][1] += e - s
span = kern[-1][1] - kern[0][0]
busy = sum(v[1] for v in agg.values())
print(json.dumps({"wall_s_unprofiled": wall, "iters": res.iterations, "span_us": span,
                  "busy_us": busy,
                  "kernels": {k: [v[0], round(v[1], 1), round(v[1] / v[0], 2)]
                              for k, v in sorted(agg.items(), key=lambda x: -x[1][1])}}, indent=1))
