import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2011_05090_b200 as sg
from paper_2011_05090_b200 import _lib
def timed(th, X, code, ld, m, chunk, reps=10):
    parts = torch.empty((chunk, th.nparts(th.n), th.k), dtype=torch.float64, device="cuda")
    def run():
        for c0 in range(0, m, chunk):
            th.partials_into(X.data_ptr() + c0 * ld * X.element_size(), code, ld, min(chunk, m - c0), parts)
    run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): run()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
g = torch.Generator(device="cuda"); g.manual_seed(0)
n, m, k = 100_000, 300, 600
th = sg.make_sketch(sg.SketchKind.GAUSSIAN, k, n, 0)
W = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
ms = timed(th, W, _lib.SGS_F64, n, m, m)
x = W[:1].contiguous()
us1 = 1e3 * timed(th, x, _lib.SGS_F64, n, 1, 1, reps=50)
print(json.dumps({"maxsub": os.environ.get("SGS_MMA_MAXSUB"), "pbatch_ms": round(ms, 4), "tflops": round(2.0*k*n*m/ms/1e9, 2), "apply_us": round(us1, 1), "nparts": th.nparts(n)}))
