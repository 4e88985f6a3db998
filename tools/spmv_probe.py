"""Graph-replayed CSR SpMV on c3's 128^3 operator (fp64 and fp32 x)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2011_05090_b200 as sg  # noqa: E402
from paper_2011_05090_b200 import _lib  # noqa: E402
from paper_2011_05090_b200.workloads import convdiff3d  # noqa: E402

rp, ci, va = convdiff3d(128)
A = sg.SparseMatrix(n=128 ** 3, row_ptr=rp, col_idx=ci, values=va)
A.device_arrays()
n = A.n
alpha = torch.full((1,), 3.0, dtype=torch.float64, device="cuda")
for dt, code in ((torch.float64, 1), (torch.float32, 0)):
    x = torch.randn(n, dtype=dt, device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    f = lambda: A.spmv_into(x.data_ptr(), code, y, alpha=alpha)  # noqa: E731
    f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            for _ in range(20):
                f()
    torch.cuda.current_stream().wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    b.synchronize()
    us = a.elapsed_time(b) / 20 * 1e3
    nnz = len(ci)
    byts = nnz * 12 + (n + 1) * 4 + n * 8 + n * x.element_size()
    print(f"x={dt} us={us:.2f} GB/s={byts / us / 1e3:.0f}")
