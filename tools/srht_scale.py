"""P-SRHT kernel time vs n (tiles of 4096, one tile per CTA up to 1024): latency vs throughput."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2011_05090_b200 as sg  # noqa: E402
from paper_2011_05090_b200 import _lib  # noqa: E402

k = 600
for n in (8 * 4096, 64 * 4096, 256 * 4096, 2 ** 21):
    th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
    th.device_data("cuda")
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    parts = torch.empty((1, th.nparts(), k), dtype=torch.float64, device="cuda")
    f = lambda: th.partials_into(x.data_ptr(), _lib.SGS_F64, n, 1, parts)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            for _ in range(50):
                f()
    torch.cuda.current_stream().wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    b.synchronize()
    print(f"n={n} tiles={n // 4096} us={a.elapsed_time(b) / 50 * 1e3:.2f} (graph)")
