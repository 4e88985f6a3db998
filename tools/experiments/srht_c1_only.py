"""One c1 P = Theta W batch launch chain (for ncu of srht_tile_kernel)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2011_05090_b200 as sg  # noqa: E402
from paper_2011_05090_b200 import _lib  # noqa: E402
n, m, k = 1_000_000, 500, 1500
th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
W = torch.randn((m, n), dtype=torch.float32, device="cuda")
chunk = max(1, min(m, (256 << 20) // (th.nparts(n) * k * 8)))
parts = torch.empty((chunk, th.nparts(n), k), dtype=torch.float64, device="cuda")
for rep in range(2):
    for c0 in range(0, m, chunk):
        th.partials_into(W.data_ptr() + c0 * n * 4, _lib.SGS_F32, n, min(chunk, m - c0), parts)
torch.cuda.synchronize()
print("ok", chunk)
