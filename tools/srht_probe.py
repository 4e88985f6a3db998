"""Standalone P-SRHT of one fp64 vector at c3's shape (n = 2^21, k = 600)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2011_05090_b200 as sg  # noqa: E402
from paper_2011_05090_b200 import _lib  # noqa: E402

n, k = 2 ** 21, int(sys.argv[1]) if len(sys.argv) > 1 else 600
th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
th.device_data("cuda")
x = torch.randn(n, dtype=torch.float64, device="cuda")
parts = torch.empty((1, th.nparts(), k), dtype=torch.float64, device="cuda")
st = _lib.Status("cuda")
f = lambda: th.partials_into(x.data_ptr(), _lib.SGS_F64, n, 1, parts, status=st)  # noqa: E731
for _ in range(3):
    f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    f()
b.record()
b.synchronize()
print("srht_us", a.elapsed_time(b) / 50 * 1e3, "nparts", th.nparts())
