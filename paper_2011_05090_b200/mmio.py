"""Matrix Market ingest for the RGMRES operators (reference io.py:24-81).

``read_matrix_market(path) -> SparseMatrix`` and ``write_matrix_market(A,
path)`` keep the reference's names, accepted formats and
``MatrixMarketError`` (a ``ValueError``).  Parsing is native
(``sgs_mm_read_header`` / ``sgs_mm_read_entries`` in the C-ABI library, host
code: no GPU needed); CSR assembly is ``SparseMatrix.from_coo`` (duplicates
summed, symmetric storage mirrored), as in the reference.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from .krylov import SparseMatrix

__all__ = ["MatrixMarketError", "read_matrix_market", "write_matrix_market"]


class MatrixMarketError(ValueError):
    pass


def _raise_from_lib(rc: int) -> None:
    if rc != 0:
        raise MatrixMarketError(_lib.load().sgs_last_error().decode(errors="replace"))


def read_matrix_market(path) -> SparseMatrix:
    """Real/integer coordinate Matrix Market file -> square CSR SparseMatrix
    (io.py:24-70): general or symmetric storage, 1-based indices converted,
    duplicates summed; pattern, complex, array, skew-symmetric and hermitian
    files, non-square sizes and out-of-bounds entries raise MatrixMarketError."""
    lib = _lib.load()
    p = os.fsencode(os.fspath(path))
    if not os.path.exists(p):
        raise FileNotFoundError(path)
    nr, nc, nnz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    sym = ctypes.c_int()
    _raise_from_lib(lib.sgs_mm_read_header(p, ctypes.byref(nr), ctypes.byref(nc),
                                           ctypes.byref(nnz), ctypes.byref(sym)))
    z = int(nnz.value)
    rows = np.empty(z, dtype=np.int64)
    cols = np.empty(z, dtype=np.int64)
    vals = np.empty(z, dtype=np.float64)
    _raise_from_lib(lib.sgs_mm_read_entries(p, z, rows.ctypes.data, cols.ctypes.data,
                                            vals.ctypes.data))
    return SparseMatrix.from_coo(int(nr.value), rows, cols, vals, symmetric=bool(sym.value))


def write_matrix_market(A: SparseMatrix, path) -> None:
    """Coordinate real general, 17 significant digits (io.py:73-81)."""
    coo = A.to_scipy().tocoo()
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{A.n} {A.n} {coo.nnz}\n")
        for i, j, v in zip(coo.row, coo.col, coo.data):
            fh.write(f"{i + 1} {j + 1} {v:.17g}\n")
