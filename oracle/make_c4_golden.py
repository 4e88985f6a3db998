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

from oracle import OracleSketch, factor_metrics, oracle_rgs_factorize  # noqa: E402
from paper_2011_05090_b200.workloads import make_w  # noqa: E402


def main():
    t0 = time.time()
    n, m, k = 1 << 25, 64, 3000
    W = make_w(n, m, 1e-10, 0, dtype=np.float32)
    print("W", round(time.time() - t0, 1), "s", flush=True)
    ref = oracle_rgs_factorize(W, OracleSketch("block_srht", k, n, 0), "mixed",
                               breakdown_factor=0.0)
    met = factor_metrics(W, ref["Q"], ref["R"], ref["S"])
    print("c4m64", met, round(time.time() - t0, 1), "s", flush=True)
    d = {f"c4_{key}": v for key, v in met.items()}
    d["c4_R"], d["c4_S"] = ref["R"], ref["S"]
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "c4m64.npz"), **d)


if __name__ == "__main__":
    main()
