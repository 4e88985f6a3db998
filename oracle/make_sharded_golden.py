"""Oracle results at the row-sharded BASELINE configs - TEST INFRASTRUCTURE
ONLY (see oracle/__init__.py).

* c2 at full size: n = 2^23, m = 1000, block-SRHT k = 2000 over 8 seeded
  2^20-row blocks (scale 1/sqrt 8), fp64, sigma_min = 1e-6, breakdown_factor 0
  -> tests/golden/c2full.npz.
* c4's shape with m columns (default 400; the full m = 1500 needs 4 GPUs):
  n = 2^25, block-SRHT k = 3000 over 32 blocks (scale 1/sqrt 32), W fp32,
  MIXED32_64, sigma_min = 1e-10, W = make_w(n, m, ...) -> tests/golden/c4m<m>.npz.

Both need more host RAM than the build container has (c2's W and Q are 67 GB
each), so this runs on the GPU box's host (`gpurun`), with every host thread:
W blocks on parallel threads (make_w is bit-identical for any thread count),
the 8 / 32 block transforms of each sketch apply on parallel threads (summed
in block order, bit-identical to one thread), multi-threaded BLAS for the
reference's step-3 GEMV.  The oracle restatement itself is unchanged and is
pinned bit for bit to the reference by tests/test_oracle_golden.py.

Kept: R, S, P, sampled rows of Q, and the three 2-norm metrics computed by
oracle.factor_metrics_blocked - the same function the GPU test applies to its
own factors.

Usage: python oracle/make_sharded_golden.py c2|c4 [--m M] [--out FILE] [--n N]
(--n shrinks the row count for a functional dry run only.)
"""

import argparse
import os
import platform
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

from oracle import OracleSketch, factor_metrics_blocked, oracle_rgs_factorize  # noqa: E402
from paper_2011_05090_b200.workloads import CONFIGS, make_w  # noqa: E402


def host_info() -> dict:
    cpu = platform.processor()
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if line.startswith("Model name:"):
                cpu = line.split(":", 1)[1].strip()
    except Exception:
        pass
    mem = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    return {"cpu": cpu, "threads": os.cpu_count(), "mem_gb": round(mem / 2**30, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=("c2", "c4"))
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    from threadpoolctl import threadpool_limits
    cfg = CONFIGS[args.config]
    n = args.n or cfg["n"]
    m = args.m or (cfg["m"] if args.config == "c2" else 400)
    k = cfg["k"]
    tag = "c2full" if (args.config == "c2" and m == cfg["m"]) else f"{args.config}m{m}"
    out = args.out or os.path.join(ROOT, "tests", "golden", f"{tag}.npz")
    info = host_info()
    print(tag, "n", n, "m", m, "k", k, info, flush=True)
    threads = os.cpu_count() or 1
    import psutil
    need = 2 * n * m * (4 if cfg["policy"] == "mixed" else 8) + 8 * 2**30
    avail = psutil.virtual_memory().available
    if avail < 1.1 * need:  # W + Q + working set; never drive the host out of memory
        print(f"SKIP {tag}: needs {need / 2**30:.0f} GiB, {avail / 2**30:.0f} GiB available",
              flush=True)
        sys.exit(3)
    dt = np.float32 if cfg["policy"] == "mixed" else np.float64
    t0 = time.time()
    W = make_w(n, m, cfg["sigma_min"], 0, dtype=dt, threads=threads)
    t_w = time.time() - t0
    print(f"W {W.shape} {W.dtype} in {t_w:.1f} s", flush=True)
    th = OracleSketch("block_srht", k, n, 0, block_log2=cfg["block_log2"], threads=threads)
    t1 = time.time()

    def progress(j):
        if (j + 1) % 50 == 0 or j + 1 == m:
            print(f"  column {j + 1}/{m}  {time.time() - t1:.1f} s", flush=True)

    with threadpool_limits(limits=threads, user_api="blas"):
        ref = oracle_rgs_factorize(W, th, cfg["policy"], breakdown_factor=cfg["breakdown_factor"],
                                   capacity=m, progress=progress)
    t_f = time.time() - t1
    met = factor_metrics_blocked(W, ref["Q"], ref["R"], ref["S"])
    print(tag, met, f"factorize {t_f:.1f} s", flush=True)
    rows = np.unique(np.linspace(0, n - 1, 101).astype(np.int64))
    d = {f"{key}": v for key, v in met.items()}
    d.update(R=ref["R"], S=ref["S"], rows=rows, Qrows=ref["Q"][rows],
             meta=np.array([n, m, k]), seconds=np.array([t_w, t_f]),
             host=np.array(f"{info['cpu']} / {info['threads']} threads / {info['mem_gb']} GB"))
    if args.config == "c2":  # (c4's P is left out to keep the fixture small)
        d["P"] = ref["P"]
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    np.savez_compressed(out, **d)
    print("wrote", out, flush=True)


if __name__ == "__main__":
    main()
