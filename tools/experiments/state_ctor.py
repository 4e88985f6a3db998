"""Device time of RgsState construction at c1 (buffer zeroing) - part of the
e2e call's critical path before column 0."""
import json, sys
import torch
sys.path.insert(0, ".")
import paper_2011_05090_b200 as sg  # noqa: E402
from paper_2011_05090_b200.workloads import CONFIGS  # noqa: E402
cfg = CONFIGS["c1"]
n, m, k = cfg["n"], cfg["m"], cfg["k"]
pol = sg.policy_from_name(cfg["policy"])
th = sg.as_device_sketch(sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)) if hasattr(sg, "as_device_sketch") else sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
out = {}
for rep in range(4):
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    z = torch.zeros((m + 1, n), dtype=torch.float32, device="cuda")
    e1.record()
    st = sg.RgsState(th, pol, capacity=m + 1, breakdown_factor=0.0)
    e2.record()
    torch.cuda.synchronize()
    out[f"rep{rep}"] = {"zeros_2GB_ms": e0.elapsed_time(e1), "state_ctor_ms": e1.elapsed_time(e2)}
    del z, st
print(json.dumps(out))
