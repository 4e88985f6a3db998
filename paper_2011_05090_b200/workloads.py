"""Seeded synthetic inputs of the BASELINE.json configurations.

The reference has no generator for these: W =
G diag(sigma) V^T, the 3D convection-diffusion operator and the Gaussian
right-hand side are defined here once and fed to both the GPU path and the
CPU oracle, so parity compares identical inputs.

* ``make_w(n, m, sigma_min, seed, dtype)``: G ~ N(0, 1/n) drawn in 2^20-row
  blocks, block b from ``Philox((seed << 64) | (0x10000 + b))`` (so a shard can
  generate its rows independently); V Haar-orthogonal = Q of the QR of an
  m x m N(0,1) matrix from ``Philox((seed << 64) | 0x7A11)`` with sign(diag R)
  folded into Q; sigma = logspace(0, log10 sigma_min, m); W = (G diag sigma) V^T
  in binary64 per block, then stored as ``dtype``.
* ``make_w_device``: the same distribution generated on the GPU with torch's
  Philox (a different stream than numpy's) for the full-size benchmark, where
  no CPU oracle runs on the same matrix.
* ``convdiff3d(N, beta)``: -Lap u + beta . grad u, 7-point centred differences
  on the N^3 interior grid of the unit cube, h = 1/(N+1), Dirichlet zero, row
  index p = i + N j + N^2 l (x fastest), columns sorted within a row.  All
  coefficients are integers for integer beta, so the CSR is exact.
* ``rhs_gaussian(n, seed)``: b = default_rng(seed).standard_normal(n).
"""

from __future__ import annotations

import math
import os

import numpy as np

ROW_BLOCK = 1 << 20

CONFIGS = {
    # BASELINE.json configs[0..4]
    "c0": dict(kind="gaussian", n=100_000, m=300, k=600, sigma_min=1e-8, policy="f64",
               breakdown_factor=10.0),
    # c0 shapes with the reference's own Rademacher sketch, generated on the
    # device from its Philox streams (not a BASELINE config)
    "c0r": dict(kind="rademacher", n=100_000, m=300, k=600, sigma_min=1e-8, policy="f64",
                breakdown_factor=10.0),
    "c1": dict(kind="psrht", n=1_000_000, m=500, k=1500, sigma_min=1e-10, policy="mixed",
               breakdown_factor=0.0),
    "c2": dict(kind="block_srht", n=1 << 23, m=1000, k=2000, sigma_min=1e-6, policy="f64",
               breakdown_factor=0.0, block_log2=20),
    "c3": dict(kind="psrht", grid=128, beta=20.0, k=600, restart=300, max_iters=3000,
               tol=1e-8),
    "c4": dict(kind="block_srht", n=1 << 25, m=1500, k=3000, sigma_min=1e-10, policy="mixed",
               breakdown_factor=0.0, block_log2=20),
}


def _philox(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=(int(seed) << 64) | int(stream)))


def haar_and_sigma(m: int, sigma_min: float, seed: int):
    A = _philox(seed, 0x7A11).standard_normal((m, m))
    V, Rv = np.linalg.qr(A)
    d = np.sign(np.diag(Rv))
    d[d == 0] = 1.0
    V = V * d
    sigma = np.logspace(0.0, math.log10(sigma_min), m)
    return V, sigma


def make_w_rows(n: int, m: int, sigma_min: float, seed: int, r0: int, r1: int,
                dtype=np.float64, threads: int | None = None) -> np.ndarray:
    """Rows [r0, r1) of W (row-major), generated blockwise.

    The product (G diag sigma) V^T is formed in fixed 2^22-element row chunks
    (boundaries relative to the 2^20-row block) with single-threaded BLAS, so
    the bits of W depend neither on the BLAS thread count nor on [r0, r1):
    OpenBLAS dgemm results change with both.  Blocks are independent, so
    `threads` Python threads generate them in parallel (numpy's generator and
    BLAS release the GIL)."""
    from threadpoolctl import threadpool_limits
    out = np.empty((r1 - r0, m), dtype=dtype)
    b0, b1 = r0 // ROW_BLOCK, (r1 - 1) // ROW_BLOCK
    step = max(1, (1 << 22) // m)
    scale = math.sqrt(n)

    with threadpool_limits(limits=1, user_api="blas"):
        V, sigma = haar_and_sigma(m, sigma_min, seed)
        M = sigma[:, None] * V.T  # diag(sigma) V^T

        def one(b):
            lo, hi = b * ROW_BLOCK, min((b + 1) * ROW_BLOCK, n)
            a, c = max(lo, r0), min(hi, r1)
            gen = _philox(seed, 0x10000 + b)
            for c0 in range(lo, c, step):
                c1 = min(c0 + step, hi)
                G = gen.standard_normal((c1 - c0, m))  # the block's stream, in order
                if c1 <= a:
                    continue
                G /= scale
                blk = G @ M
                x0, x1 = max(c0, a), min(c1, c)
                out[x0 - r0:x1 - r0] = blk[x0 - c0:x1 - c0]

        blocks = range(b0, b1 + 1) if r1 > r0 else range(0)
        nt = min(len(blocks), threads if threads is not None else (os.cpu_count() or 1))
        if nt > 1:
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor(nt) as ex:
                list(ex.map(one, blocks))
        else:
            for b in blocks:
                one(b)
    return out


def make_w(n: int, m: int, sigma_min: float, seed: int, dtype=np.float64,
           threads: int | None = None) -> np.ndarray:
    return make_w_rows(n, m, sigma_min, seed, 0, n, dtype, threads)


def make_w_device(n: int, m: int, sigma_min: float, seed: int, dtype, device,
                  row0: int = 0, n_local: int | None = None, ld: int | None = None):
    """Column-major W rows [row0, row0+n_local) on the GPU: returns a tensor of
    shape (m, ld) whose row j is column j.  Same distribution as make_w."""
    import torch
    n_local = n - row0 if n_local is None else n_local
    ld = ld or ((n_local + 31) // 32 * 32)
    V, sigma = haar_and_sigma(m, sigma_min, seed)
    Mt = torch.from_numpy((sigma[:, None] * V.T).T.copy()).to(device)  # (m, m) = V diag(sigma)
    out = torch.zeros((m, ld), dtype=dtype, device=device)
    gen = torch.Generator(device=device)
    step = 1 << 18
    for r in range(0, n_local, step):
        rr = min(step, n_local - r)
        gen.manual_seed((seed << 20) ^ (row0 + r))
        G = torch.randn((m, rr), dtype=torch.float64, device=device, generator=gen)
        G /= math.sqrt(n)
        # column-major block: W_blk^T = (V diag sigma) G^T  (m x rr)
        out[:, r:r + rr] = (Mt @ G).to(dtype)
    return out


def convdiff3d(N: int, beta=(20.0, 20.0, 20.0)):
    """CSR arrays (row_ptr, col_idx, values) of the 7-point conv-diff operator."""
    n = N * N * N
    inv_h2 = float((N + 1) ** 2)
    half_inv_h = 0.5 * (N + 1)
    idx = np.arange(n, dtype=np.int64)
    i = idx % N
    j = (idx // N) % N
    l = idx // (N * N)
    # neighbour offsets in sorted column order: -N^2, -N, -1, 0, +1, +N, +N^2
    offs = [-(N * N), -N, -1, 0, 1, N, N * N]
    bx, by, bz = beta
    coef = [-inv_h2 - bz * half_inv_h, -inv_h2 - by * half_inv_h, -inv_h2 - bx * half_inv_h,
            6.0 * inv_h2,
            -inv_h2 + bx * half_inv_h, -inv_h2 + by * half_inv_h, -inv_h2 + bz * half_inv_h]
    valid = [l > 0, j > 0, i > 0, np.ones(n, bool), i < N - 1, j < N - 1, l < N - 1]
    mask = np.stack(valid, axis=1)                    # (n, 7)
    cols = idx[:, None] + np.asarray(offs)[None, :]
    vals = np.broadcast_to(np.asarray(coef), (n, 7))
    counts = mask.sum(axis=1)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    col_idx = cols[mask].astype(np.int32)
    values = np.ascontiguousarray(vals[mask], dtype=np.float64)
    return row_ptr.astype(np.int32), col_idx, values


def rhs_gaussian(n: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal(n)


def shard_rows(n: int, world: int, rank: int, align: int = 4096) -> tuple[int, int]:
    """Contiguous, `align`-aligned row range of this rank: (row0, n_local)."""
    units = (n + align - 1) // align
    u0 = (units * rank) // world
    u1 = (units * (rank + 1)) // world
    r0 = min(n, u0 * align)
    r1 = min(n, u1 * align)
    return r0, r1 - r0
