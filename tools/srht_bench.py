"""Time the stand-alone SRHT partial sketches (srht_tile_kernel, or the
three-pass kernel with SGS_SRHT_LEGACY=1) at the BASELINE shapes with CUDA
events: c1's batched P = Theta W (500 fp32 columns of 1e6 rows), c3's sketch
of w (one fp64 column of 2^21), 50 fp64 columns of c2 (block-SRHT, 2^23) and
one fp32 column of c4 (2^25).  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_05090_b200 as sg  # noqa: E402
from paper_2011_05090_b200 import _lib  # noqa: E402


def timed(th, X, code, ld, m, chunk, reps=5):
    parts = torch.empty((chunk, th.nparts(th.n), th.k), dtype=torch.float64, device="cuda")

    def run():
        for c0 in range(0, m, chunk):
            th.partials_into(X.data_ptr() + c0 * ld * X.element_size(), code, ld,
                             min(chunk, m - c0), parts)
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {"legacy": os.environ.get("SGS_SRHT_LEGACY", "0")}
g = torch.Generator("cuda").manual_seed(0)
# c1 P batch
n, m, k = 1_000_000, 500, 1500
th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
W = torch.randn((m, n), dtype=torch.float32, device="cuda", generator=g)
chunk = max(1, min(m, (256 << 20) // (th.nparts(n) * k * 8)))
ms = timed(th, W, _lib.SGS_F32, n, m, chunk)
out["c1_pbatch_ms"] = round(ms, 4)
out["c1_pbatch_gbs"] = round(n * m * 4 / ms / 1e6, 1)
del W
# c3 sketch of w
n, k = 1 << 21, 600
th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
x = torch.randn((1, n), dtype=torch.float64, device="cuda", generator=g)
ms = timed(th, x, _lib.SGS_F64, n, 1, 1, reps=200)
out["c3_w_us"] = round(1e3 * ms, 2)
# c2: 50 fp64 columns of 2^23
n, m, k = 1 << 23, 50, 2000
th = sg.make_sketch(sg.SketchKind.BLOCK_SRHT, k, n, 0, block_log2=20)
W = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
ms = timed(th, W, _lib.SGS_F64, n, m, m)
out["c2_50cols_ms"] = round(ms, 4)
out["c2_gbs"] = round(n * m * 8 / ms / 1e6, 1)
del W
# c4: one fp32 column of 2^25
n, k = 1 << 25, 3000
th = sg.make_sketch(sg.SketchKind.BLOCK_SRHT, k, n, 0, block_log2=20)
x = torch.randn((1, n), dtype=torch.float32, device="cuda", generator=g)
ms = timed(th, x, _lib.SGS_F32, n, 1, 1, reps=50)
out["c4_col_us"] = round(1e3 * ms, 2)
out["c4_gbs"] = round(n * 4 / ms / 1e6, 1)
del x
# c0: Gaussian P = Theta W, 300 fp64 columns of 1e5 rows, k = 600 (DMMA, or
# the DFMA GEMM with SGS_DENSE_LEGACY=1)
n, m, k = 100_000, 300, 600
th = sg.make_sketch(sg.SketchKind.GAUSSIAN, k, n, 0)
W = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
ms = timed(th, W, _lib.SGS_F64, n, m, m)
out["c0_pbatch_ms"] = round(ms, 4)
out["c0_pbatch_tflops"] = round(2.0 * k * n * m / ms / 1e9, 2)
out["dense_legacy"] = os.environ.get("SGS_DENSE_LEGACY", "0")
print(json.dumps(out), flush=True)
