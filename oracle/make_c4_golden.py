"""Oracle results at BASELINE c4's shape with 64 of its 1500 columns - TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).

n = 2^25, block-SRHT k = 3000 over 32 seeded 2^20-row blocks (scale 1/sqrt 32),
W fp32 (sigma_min = 1e-10), MIXED32_64, breakdown_factor 0.  c4 itself needs 4
GPUs (W and Q are 201 GB each); 64 columns keep its sketch, row count and
block structure on one GPU.  Keeps the metrics, R and S (tests/golden/c4m64.npz).
Usage: python oracle/make_c4_golden.py
"""

import os
import sys
import time

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

from oracle import OracleSketch, oracle_rgs_factorize  # noqa: E402
from paper_2011_05090_b200.workloads import make_w  # noqa: E402


def metrics_chunked(W, Q, R, S, rows=1 << 20):
    """oracle.factor_metrics in fp64 over row blocks (the fp64 copies of W and
    Q at n = 2^25 would not fit this host)."""
    m = Q.shape[1]
    G = np.zeros((m, m))
    num = den = 0.0
    for r0 in range(0, W.shape[0], rows):
        Qb = np.asarray(Q[r0:r0 + rows], dtype=np.float64)
        Wb = np.asarray(W[r0:r0 + rows], dtype=np.float64)
        G += Qb.T @ Qb
        num += float(np.sum((Wb - Qb @ R) ** 2))
        den += float(np.sum(Wb ** 2))
    S = np.asarray(S, dtype=np.float64)
    eye = np.eye(m)
    return {"orth_S_2": float(np.linalg.norm(eye - S.T @ S, 2)),
            "orth_Q_2": float(np.linalg.norm(eye - G, 2)),
            "relres_F": float(np.sqrt(num) / np.sqrt(den))}


def main():
    t0 = time.time()
    n, m, k = 1 << 25, 64, 3000
    W = make_w(n, m, 1e-10, 0, dtype=np.float32)
    print("W", round(time.time() - t0, 1), "s", flush=True)
    ref = oracle_rgs_factorize(W, OracleSketch("block_srht", k, n, 0), "mixed",
                               breakdown_factor=0.0)
    met = metrics_chunked(W, ref["Q"], ref["R"], ref["S"])
    print("c4m64", met, round(time.time() - t0, 1), "s", flush=True)
    d = {f"c4_{key}": v for key, v in met.items()}
    d["c4_R"], d["c4_S"] = ref["R"], ref["S"]
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "c4m64.npz"), **d)


if __name__ == "__main__":
    main()
