"""Small-shape workload touching every kernel family once, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

  fused SRHT column kernel (TMA bulk-copy ring, mbarriers, 8-CTA DSMEM sum),
  LS cluster kernel (16-CTA DSMEM exchanges, PDL), stand-alone SRHT tile
  kernel, dense ring kernel + split-K GEMM/GEMV (Gaussian), device Rademacher
  generator + partials, generic update kernel, CSR SpMV (staged bulk copies),
  Givens / Arnoldi engine (standard and one-synchronisation), ILU(0) analysis,
  factorisation and the sync-free sweeps, sketched_lsq, FWHT.

Usage: compute-sanitizer --tool <tool> python tools/sanitize_small.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_05090_b200 as sg  # noqa: E402
from paper_2011_05090_b200.workloads import convdiff3d, make_w, rhs_gaussian  # noqa: E402

torch.cuda.set_device(0)
rng = np.random.default_rng(0)
n, m = 3 * 4096 + 515, 12
for kind, k, pol in (("psrht", 96, sg.MIXED32_64), ("psrht", 64, sg.UNIFIED64),
                     ("gaussian", 48, sg.UNIFIED64), ("rademacher", 40, sg.UNIFIED64)):
    th = sg.make_sketch(sg.SketchKind(kind), k, n, 1)
    W = make_w(n, m, 1e-3, 1, dtype=np.float32 if pol is sg.MIXED32_64 else np.float64)
    f, cert = sg.rgs_factorize(W, th, pol, breakdown_factor=0.0)      # batch path
    st = sg.RgsState(th, pol, breakdown_factor=0.0)                   # streaming path
    for j in range(4):
        st.push(W[:, j])
    th.apply(W[:, 0])
    th.apply_block(W[:, :3])
    print(kind, "ok", float(cert.delta_m), flush=True)
# block-SRHT with 4096-row blocks, fp64
th = sg.make_sketch(sg.SketchKind.BLOCK_SRHT, 64, 4 * 4096, 2, block_log2=12)
sg.rgs_factorize(make_w(4 * 4096, 8, 1e-2, 2), th, sg.UNIFIED64)
sg.fwht(rng.standard_normal(8192))
S = np.linalg.qr(rng.standard_normal((60, 8)))[0]
sg.sketched_lsq(S, rng.standard_normal(60))
# Krylov: SpMV, Givens, standard + lagged Arnoldi, ILU(0)
N = 10
rp, ci, va = convdiff3d(N)
A = sg.SparseMatrix(n=N ** 3, row_ptr=rp, col_idx=ci, values=va)
b = rhs_gaussian(A.n, 0)
th = sg.make_sketch(sg.SketchKind.PSRHT, 80, A.n, 0)
for lag in (False, True):
    for pol in (sg.UNIFIED64, sg.MIXED32_64):
        r = sg.gmres(A, b, m=30, theta=th, policy=pol, tol=1e-8, lagged=lag)
        print("gmres", lag, r.iterations, flush=True)
M = sg.ilu0(A)
r = sg.gmres(A, b, m=30, theta=th, policy=sg.UNIFIED64, tol=1e-8, preconditioner=M)
print("ilu gmres", r.iterations, flush=True)
torch.cuda.synchronize()
from paper_2011_05090_b200 import _lib  # noqa: E402
print("LIBRARY", _lib.LIB_PATH, flush=True)
print("SANITIZE_WORKLOAD_DONE", flush=True)
