"""cond(Q) of the reference's acceptance problem (criterion 1: synthetic_matrix
n = 1e5, m = 300, P-SRHT k = 5000, seed 1, breakdown_factor 0) for the fp32
(UNIFIED32) and mixed policies: the numbers behind test_criterion_1 (reference:
cond rgs = 1.899, rgs-f32 = 53.7, pkg/test_output.txt).  Run with the A/B
switches (SGS_ACC_TWO, SGS_SRHT_LEGACY, SGS_LS_DEFER) to attribute a change."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2011_05090_b200 as sg  # noqa: E402
from oracle.ref_io import synthetic_matrix  # noqa: E402

W = synthetic_matrix(100_000, 300)
th = sg.make_sketch(sg.SketchKind.PSRHT, 5000, 100_000, 1)
out = {k: os.environ.get(k, "-") for k in ("SGS_ACC_TWO", "SGS_SRHT_LEGACY", "SGS_LS_DEFER")}
for name, pol in (("rgs", sg.MIXED32_64), ("rgs32", sg.UNIFIED32)):
    f, _ = sg.rgs_factorize(W, th, pol, with_certificate=False, breakdown_factor=0.0)
    Q = f.Q.astype(np.float64)
    S = f.S.astype(np.float64)
    out[name] = {"cond_Q": float(np.linalg.cond(Q)),
                 "orth_S_2": float(np.linalg.norm(np.eye(300) - S.T @ S, 2)),
                 "cond_S": float(np.linalg.cond(S))}
print(json.dumps(out), flush=True)
