"""LS kernel phase times with the k-dimensional state cold (L2 flushed) vs warm."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2011_05090_b200 as sg
from paper_2011_05090_b200.workloads import make_w_device

n, m, k = 1_000_000, 450, 1500
th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
W = make_w_device(n, m, 1e-10, 0, torch.float32, "cuda")
st = sg.RgsState(th, sg.MIXED32_64, capacity=m + 1, breakdown_factor=0.0)
st.factorize_columns(W, W.shape[1], m)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
tr = torch.zeros((m + 1, 16), dtype=torch.int64, device="cuda")
i = m - 1
# recompute finalize(i) (idempotent) with partials of the stored q'_i... use S col as s' proxy:
parts = torch.zeros((1, k), dtype=torch.float64, device="cuda")
parts[0] = st._S[i].to(torch.float64)
names = ["reduce", "exch1_local", "clsync1", "gather1", "s_matvec", "exch2", "reorth", "rinv_col"]
for label, do_flush in (("cold", True), ("warm", False), ("cold", True), ("warm", False)):
    if do_flush:
        flush.fill_(1)
    st._trace = tr
    st._ls(fin=i, s_parts=parts.data_ptr(), s_nparts=1, s_scale=1.0)
    torch.cuda.synchronize()
    st._trace = None
    t = tr[i].cpu().numpy().astype(float)
    d = {names[j - 1]: round((t[j] - t[j - 1]) / 1965.0, 2) for j in range(1, 9) if t[j] and t[j - 1]}
    print(label, "total", round((t[8] - t[0]) / 1965.0, 2), d)
