"""Pin the RGMRES(300) iteration counts of BASELINE config 3 with the oracle
(bit-identical to the reference; restart wrapper of SURVEY.md 8(d)):
128^3 convection-diffusion, b = default_rng(0), Theta = P-SRHT(600, 2^21, 0).
Writes tests/golden/c3_oracle.json.  ~8-10 min per basis single-threaded."""
import json, os, sys, time
for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
    os.environ[v] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from oracle import OracleSketch, csr_matvec, oracle_gmres_restarted
from paper_2011_05090_b200.workloads import convdiff3d, rhs_gaussian

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
rp, ci, va = convdiff3d(N)
n = N ** 3
b = rhs_gaussian(n, 0)
op = OracleSketch("psrht", 600, n, 0)
mv = lambda x: csr_matvec(rp, ci, va, n, x)
out = {"grid": N, "k": 600, "restart": 300, "tol": 1e-8}
for pol in ("f64", "mixed"):
    t0 = time.time()
    r = oracle_gmres_restarted(mv, n, b, op, pol, restart=300, max_iters=3000, tol=1e-8)
    out[pol] = {"iterations": r["iterations"], "cycles": r["cycles"],
                "final_residual": r["final_residual"], "seconds": time.time() - t0}
    print(pol, out[pol], flush=True)
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden",
                    f"c3_oracle_{N}.json")
json.dump(out, open(path, "w"), indent=1)
