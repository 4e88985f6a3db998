"""Oracle results at BASELINE c2's shape with 200 of its 1000 columns -
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

n = 2^23, block-SRHT k = 2000 over 8 seeded 2^20-row blocks (scale 1/sqrt 8),
fp64, breakdown_factor 0, W = make_w(n, 200, 1e-6, 0).  The full m = 1000
does not fit this host (W alone is 67 GB); 200 columns keep the sketch, the
row count and the block structure of c2.  Keeps the metrics, R and S
(tests/golden/c2m200.npz).  Usage: python oracle/make_c2_golden.py
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
    n, m, k = 1 << 23, 200, 2000
    W = make_w(n, m, 1e-6, 0)
    print("W", round(time.time() - t0, 1), "s", flush=True)
    ref = oracle_rgs_factorize(W, OracleSketch("block_srht", k, n, 0), "f64",
                               breakdown_factor=0.0)
    met = factor_metrics(W, ref["Q"], ref["R"], ref["S"])
    print("c2m200", met, round(time.time() - t0, 1), "s", flush=True)
    d = {f"c2_{key}": v for key, v in met.items()}
    d["c2_R"], d["c2_S"] = ref["R"], ref["S"]
    rows = np.arange(0, n, 83_887)
    d["c2_rows"], d["c2_Qrows"] = rows, ref["Q"][rows]
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "c2m200.npz"), **d)


if __name__ == "__main__":
    main()
