"""Print the full-size parity numbers (GPU vs the oracle golden of
oracle/make_fullsize_golden.py) for DESIGN.md / profiles."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2011_05090_b200 as sg
from paper_2011_05090_b200.workloads import make_w
from test_gpu_full_size import _metrics_dev

g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "fullsize.npz"))
out = {}
for name, n, m, k, smin, kind, pol, bf, dt in (
        ("c0", 100_000, 300, 600, 1e-8, "gaussian", sg.UNIFIED64, 10.0, np.float64),
        ("c0twin", 100_000, 300, 600, 1e-2, "gaussian", sg.UNIFIED64, 10.0, np.float64),
        ("c1", 1_000_000, 500, 1500, 1e-10, "psrht", sg.MIXED32_64, 0.0, np.float32)):
    W = torch.from_numpy(make_w(n, m, smin, 0, dtype=dt)).cuda()
    th = sg.make_sketch(sg.SketchKind(kind), k, n, 0)
    f, _ = sg.rgs_factorize(W, th, pol, breakdown_factor=bf, device_factors=True)
    ours = _metrics_dev(W, f)
    out[name] = {key: {"gpu": v, "oracle": float(g[f"{name}_{key}"])} for key, v in ours.items()}
    if name == "c0twin":
        rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
        rows = torch.from_numpy(g["c0twin_rows"]).cuda()
        out[name]["rel_R"] = rel(f.R.cpu().numpy(), g["c0twin_R"])
        out[name]["rel_S"] = rel(f.S.cpu().numpy(), g["c0twin_S"])
        out[name]["rel_Qrows"] = rel(f.Q[rows].cpu().numpy(), g["c0twin_Qrows"])
gp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                  "c2m200.npz")
if os.path.exists(gp):  # c2's shape, 200 columns (oracle/make_c2_golden.py)
    g2 = np.load(gp)
    n, m, k = 1 << 23, 200, 2000
    W = torch.from_numpy(make_w(n, m, 1e-6, 0)).cuda()
    th = sg.make_sketch(sg.SketchKind.BLOCK_SRHT, k, n, 0, block_log2=20)
    f, _ = sg.rgs_factorize(W, th, sg.UNIFIED64, breakdown_factor=0.0, device_factors=True)
    ours = _metrics_dev(W, f)
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
    rows = torch.from_numpy(g2["c2_rows"]).cuda()
    out["c2m200"] = {key: {"gpu": v, "oracle": float(g2[f"c2_{key}"])} for key, v in ours.items()}
    out["c2m200"].update(rel_R=rel(f.R.cpu().numpy(), g2["c2_R"]),
                         rel_S=rel(f.S.cpu().numpy(), g2["c2_S"]),
                         rel_Qrows=rel(f.Q[rows].cpu().numpy(), g2["c2_Qrows"]))
g4p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "c4m64.npz")
if os.path.exists(g4p):  # c4's shape, 64 columns (oracle/make_c4_golden.py)
    g4 = np.load(g4p)
    n, m, k = 1 << 25, 64, 3000
    W = torch.from_numpy(make_w(n, m, 1e-10, 0, dtype=np.float32)).cuda()
    th = sg.make_sketch(sg.SketchKind.BLOCK_SRHT, k, n, 0, block_log2=20)
    f, _ = sg.rgs_factorize(W, th, sg.MIXED32_64, breakdown_factor=0.0, device_factors=True)
    ours = _metrics_dev(W, f)
    out["c4m64"] = {key: {"gpu": v, "oracle": float(g4[f"c4_{key}"])} for key, v in ours.items()}
    R = f.R.cpu().numpy()
    out["c4m64"]["rel_R"] = float(np.linalg.norm(R - g4["c4_R"]) / np.linalg.norm(g4["c4_R"]))
print(json.dumps(out, indent=1))
