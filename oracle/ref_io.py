"""Problem generators of the reference (TEST INFRASTRUCTURE ONLY, see
oracle/__init__.py): io.synthetic_matrix (io.py:84-100), generate_laplacian_2d
(io.py:103-117) and generate_random_sparse (io.py:120-141), restated for the
acceptance-criteria ports (tests/test_gpu_acceptance.py).  Pinned against the
reference's own outputs by tests/test_oracle_golden.py (tests/golden/io_gen.npz,
oracle/make_golden.py io)."""

from __future__ import annotations

import numpy as np
import scipy.sparse


def synthetic_matrix(n: int, m: int) -> np.ndarray:
    """W[i, j] = sin(10 (mu_j + x_i)) / (cos(100 (mu_j - x_i)) + 1.1) on the
    inclusive grids x_i = i/(n-1), mu_j = j/(m-1), binary64 (io.py:84-100)."""
    if n < 2 or m < 2:
        raise ValueError("need n >= 2 and m >= 2")
    x = np.arange(n, dtype=np.float64) / (n - 1)
    W = np.empty((n, m))
    for j in range(m):
        mu = j / (m - 1)
        W[:, j] = np.sin(10.0 * (mu + x)) / (np.cos(100.0 * (mu - x)) + 1.1)
    return W


def _csr(n, rows, cols, vals):
    # SparseMatrix.from_coo (krylov.py:42-69): duplicates summed, CSR order
    m = scipy.sparse.coo_matrix((np.asarray(vals, dtype=np.float64),
                                 (np.asarray(rows), np.asarray(cols))), shape=(n, n)).tocsr()
    m.sum_duplicates()
    return m.indptr.copy(), m.indices.copy(), m.data.astype(np.float64)


def laplacian_2d(grid: int):
    """5-point Laplacian on a grid x grid mesh (io.py:103-117) as CSR arrays."""
    if grid < 2:
        raise ValueError("grid must be at least 2")
    n = grid * grid
    rows, cols, vals = [], [], []
    for iy in range(grid):
        for ix in range(grid):
            p = iy * grid + ix
            rows.append(p); cols.append(p); vals.append(4.0)
            for qx, qy in ((ix - 1, iy), (ix + 1, iy), (ix, iy - 1), (ix, iy + 1)):
                if 0 <= qx < grid and 0 <= qy < grid:
                    rows.append(p); cols.append(qy * grid + qx); vals.append(-1.0)
    return (n,) + _csr(n, rows, cols, vals)


def random_sparse(n: int, nnz_per_row: int, seed: int, diag_shift: float = 1.0):
    """Seeded diagonally dominant random sparse matrix (io.py:120-141) as CSR."""
    if n < 1 or nnz_per_row < 0 or nnz_per_row > n - 1:
        raise ValueError("invalid size or fill")
    rng = np.random.Generator(np.random.Philox(key=(int(seed) << 64) | 0x5BA5))
    rows, cols, vals = [], [], []
    offdiag_abs = np.zeros(n)
    for i in range(n):
        choices = rng.choice(n - 1, size=nnz_per_row, replace=False)
        choices = np.where(choices >= i, choices + 1, choices)
        v = rng.uniform(-1.0, 1.0, size=nnz_per_row)
        rows.extend([i] * nnz_per_row)
        cols.extend(choices.tolist())
        vals.extend(v.tolist())
        offdiag_abs[i] = np.abs(v).sum()
    for i in range(n):
        rows.append(i); cols.append(i); vals.append(offdiag_abs[i] + diag_shift)
    return (n,) + _csr(n, rows, cols, vals)
