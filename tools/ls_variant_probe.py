"""Factor hashes for the LS kernel variant test (tests/test_gpu_ls_variants.py):
one batch factorisation and a streaming push sequence per sketch kind, SHA-256
of Q, R, S.  The LS kernel variant (SGS_LS_PLAIN) and the column kernels'
prefetch switches are read once per process, so the test runs this script in
fresh processes and compares the printed lines."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_05090_b200 as sg  # noqa: E402
from paper_2011_05090_b200.workloads import make_w  # noqa: E402

torch.cuda.set_device(0)


def h(*arrs):
    d = hashlib.sha256()
    for a in arrs:
        d.update(np.ascontiguousarray(a).tobytes())
    return d.hexdigest()[:32]


n, m = 5 * 4096 + 77, 40
for kind, k, pol in (("psrht", 200, sg.MIXED32_64), ("psrht", 130, sg.UNIFIED64),
                     ("gaussian", 96, sg.UNIFIED64), ("psrht", 160, sg.UNIFIED32)):
    th = sg.make_sketch(sg.SketchKind(kind), k, n, 3)
    W = make_w(n, m, 1e-6, 3, dtype=np.float64 if pol is sg.UNIFIED64 else np.float32)
    f, _ = sg.rgs_factorize(W, th, pol, breakdown_factor=0.0)
    print("batch", kind, k, pol.mode, h(f.Q, f.R, f.S), flush=True)
    st = sg.RgsState(th, pol, breakdown_factor=0.0)
    for j in range(12):
        st.push(W[:, j])
    g = st.factors()
    print("push", kind, k, pol.mode, h(g.Q, g.R, g.S), flush=True)
print("LS_VARIANT_PROBE_DONE")
