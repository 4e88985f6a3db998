"""Full-size (BASELINE configs 0 and 1) oracle results for the GPU parity
tests - TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Runs the oracle restatement (pinned bit for bit to the reference by
tests/test_oracle_golden.py) at the BASELINE sizes on the host and keeps what
the north_star gates need, small enough to commit (tests/golden/fullsize.npz):
  * c0 (n=1e5, m=300, k=600 Gaussian, fp64, sigma_min=1e-8): the three 2-norm
    metrics (the 10x gates: c0 is beyond the 1e-10 Q/R noise floor);
  * its well-conditioned twin (sigma_min=1e-2): R, S and 101 sampled rows of Q
    for the 1e-10 gates;
  * c1 (n=1e6, m=500, k=1500 P-SRHT, MIXED32_64, breakdown_factor=0): the
    metrics and diag(R).
W comes from paper_2011_05090_b200.workloads.make_w (numpy Philox, the same
generator the GPU tests call; bit-identical for any thread count).  The
metrics come from oracle.factor_metrics_blocked, the function the GPU tests
apply to their own factors.  Usage: python oracle/make_fullsize_golden.py
"""

import os
import sys
import time

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

from oracle import OracleSketch, factor_metrics_blocked, oracle_rgs_factorize  # noqa: E402
from paper_2011_05090_b200.workloads import make_w  # noqa: E402

QROWS = np.arange(0, 100_000, 997)


def main():
    d = {}
    t0 = time.time()
    n, m, k = 100_000, 300, 600
    W = make_w(n, m, 1e-8, 0)
    ref = oracle_rgs_factorize(W, OracleSketch("gaussian", k, n, 0), "f64")
    met = factor_metrics_blocked(W, ref["Q"], ref["R"], ref["S"])
    for key, v in met.items():
        d[f"c0_{key}"] = v
    print("c0", met, round(time.time() - t0, 1), "s", flush=True)
    t0 = time.time()
    W = make_w(n, m, 1e-2, 0)
    ref = oracle_rgs_factorize(W, OracleSketch("gaussian", k, n, 0), "f64")
    d["c0twin_R"], d["c0twin_S"] = ref["R"], ref["S"]
    d["c0twin_Qrows"], d["c0twin_rows"] = ref["Q"][QROWS], QROWS
    met = factor_metrics_blocked(W, ref["Q"], ref["R"], ref["S"])
    for key, v in met.items():
        d[f"c0twin_{key}"] = v
    print("c0 twin", met, round(time.time() - t0, 1), "s", flush=True)
    del W, ref
    t0 = time.time()
    n, m, k = 1_000_000, 500, 1500
    W = make_w(n, m, 1e-10, 0, dtype=np.float32)
    ref = oracle_rgs_factorize(W, OracleSketch("psrht", k, n, 0), "mixed", breakdown_factor=0.0)
    met = factor_metrics_blocked(W, ref["Q"], ref["R"], ref["S"])
    for key, v in met.items():
        d[f"c1_{key}"] = v
    d["c1_Rdiag"] = np.diag(ref["R"]).copy()
    print("c1", met, round(time.time() - t0, 1), "s", flush=True)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "fullsize.npz"), **d)


if __name__ == "__main__":
    main()
