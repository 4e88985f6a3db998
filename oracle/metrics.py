"""Parity metrics (TEST INFRASTRUCTURE ONLY): the 2-norm gates BASELINE.json
names, which the reference lacks (it reports Frobenius norms,
gram_schmidt.py:482, :490-494)."""

from __future__ import annotations

import numpy as np


def rel_diff(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def factor_metrics(W, Q, R, S) -> dict:
    """||I - S^T S||_2, ||I - Q^T Q||_2, ||W - QR||_F / ||W||_F."""
    Q = np.asarray(Q, dtype=np.float64)
    S = np.asarray(S, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    m = Q.shape[1]
    I = np.eye(m)
    return {
        "orth_S_2": float(np.linalg.norm(I - S.T @ S, 2)),
        "orth_Q_2": float(np.linalg.norm(I - Q.T @ Q, 2)),
        "relres_F": float(np.linalg.norm(W - Q @ np.asarray(R)) / np.linalg.norm(W)),
    }
