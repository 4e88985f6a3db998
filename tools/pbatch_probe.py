"""Time the batched P = Theta W sketch of c1 (P-SRHT, 500 fp32 columns) with
CUDA events: the chunking of RgsState._enqueue_factorization."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2011_05090_b200 as sg
from paper_2011_05090_b200 import _lib
from paper_2011_05090_b200.workloads import make_w_device

n, m, k = 1_000_000, 500, 1500
th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
W = make_w_device(n, m, 1e-10, 0, torch.float32, "cuda")
ldw = W.shape[1]
npart = th.nparts(n)
chunk = max(1, min(m, (256 << 20) // (npart * k * 8)))
parts = torch.empty((chunk, npart, k), dtype=torch.float64, device="cuda")
for _ in range(2):
    for c0 in range(0, m, chunk):
        th.partials_into(W.data_ptr() + c0 * ldw * 4, _lib.SGS_F32, ldw, min(chunk, m - c0), parts)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for c0 in range(0, m, chunk):
    th.partials_into(W.data_ptr() + c0 * ldw * 4, _lib.SGS_F32, ldw, min(chunk, m - c0), parts)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"P batch: {ms:.3f} ms for {m} columns in chunks of {chunk} ({npart} parts); "
      f"{n * m * 4 / ms / 1e6:.0f} GB/s of W")
