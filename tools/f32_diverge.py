"""UNIFIED32 on the acceptance problem (synthetic_matrix 1e5 x 300, P-SRHT
k = 5000, seed 1, breakdown_factor 0), GPU against the oracle restatement of
the reference (fp32 Householder LS): per column, how far S drifts from
orthonormality (max |S[:, :j]^T S[:, j]|) on both sides, and |R_jj| / r
differences, to locate where the device's fp32 LS loses the sketched basis."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

import paper_2011_05090_b200 as sg  # noqa: E402
from oracle import OracleSketch, oracle_rgs_factorize  # noqa: E402
from oracle.ref_io import synthetic_matrix  # noqa: E402

N, M, K = 100_000, 300, 5000
W = synthetic_matrix(N, M)
th = sg.make_sketch(sg.SketchKind.PSRHT, K, N, 1)
pol = sg.policy_from_name(sys.argv[1] if len(sys.argv) > 1 else "f32")
f, _ = sg.rgs_factorize(W, th, pol, with_certificate=False, breakdown_factor=0.0)
with threadpool_limits(limits=os.cpu_count()):
    ref = oracle_rgs_factorize(W, OracleSketch("psrht", K, N, 1),
                               "f32" if pol is sg.UNIFIED32 else "mixed", 0.0, capacity=M)


def drift(S):
    S = S.astype(np.float64)
    G = S.T @ S
    return [float(np.max(np.abs(G[:j, j]))) if j else 0.0 for j in range(S.shape[1])]


dg, dr = drift(f.S), drift(ref["S"])
Rg, Rr = f.R.astype(np.float64), ref["R"].astype(np.float64)
out = {"policy": pol.name if hasattr(pol, "name") else str(pol),
       "cond_Q_gpu": float(np.linalg.cond(f.Q.astype(np.float64))),
       "cond_Q_ref": float(np.linalg.cond(ref["Q"].astype(np.float64))),
       "cols": []}
for j in list(range(0, 40, 2)) + list(range(40, M, 10)):
    out["cols"].append({"j": j, "drift_gpu": dg[j], "drift_ref": dr[j],
                        "rjj_gpu": float(Rg[j, j]), "rjj_ref": float(Rr[j, j]),
                        "rcol_rel": float(np.linalg.norm(Rg[:j, j] - Rr[:j, j])
                                          / max(np.linalg.norm(Rr[:j, j]), 1e-300)) if j else 0.0})
print(json.dumps(out), flush=True)
