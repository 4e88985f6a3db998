"""Time the device Rademacher sketch kernels at c0 shapes (argv: k n)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2011_05090_b200 as sg
from paper_2011_05090_b200 import _lib

k = int(sys.argv[1]) if len(sys.argv) > 1 else 600
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
th = sg.make_sketch(sg.SketchKind.RADEMACHER, k, n, 0)
t0 = time.perf_counter()
th.device_data()
torch.cuda.synchronize()
print("bits generation", round((time.perf_counter() - t0) * 1e3, 2), "ms (incl. first call)")
x = torch.randn(n, dtype=torch.float64, device="cuda")
X = torch.randn((300, n), dtype=torch.float64, device="cuda")
parts = torch.empty((300, th.nparts(), k), dtype=torch.float64, device="cuda")
for ncols, XX in ((1, x), (300, X)):
    for _ in range(3):
        th.partials_into(XX, _lib.SGS_F64, n, ncols, parts)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        th.partials_into(XX, _lib.SGS_F64, n, ncols, parts)
    e1.record()
    torch.cuda.synchronize()
    print(f"partials ncols={ncols}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
