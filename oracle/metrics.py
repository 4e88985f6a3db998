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


def factor_metrics_blocked(W, Q, R, S, device=None, rows: int = 1 << 18) -> dict:
    """factor_metrics in fp64 over row blocks - ONE function for both sides of
    a parity check, so the GPU factors and the oracle's are measured by the
    same arithmetic (fp64 torch on `device`: the GPU when there is one).

    W, Q: (n, m) numpy arrays or torch tensors (any dtype, any device/layout);
    R: (m, m); S: (k, m).  Returns the three 2-norm gates of BASELINE.json:
    ||I - S^T S||_2, ||I - Q^T Q||_2 and ||W - QR||_F / ||W||_F.  Row blocks
    keep the fp64 copies small (c2: W and Q are 67 GB each); the Gram matrix
    and the residual sums accumulate in block order."""
    import torch
    if device is None:
        device = "cuda" if torch.cuda.is_available() else "cpu"

    def t(x):
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(np.ascontiguousarray(x))
        return x.to(device=device, dtype=torch.float64).contiguous()

    n, m = Q.shape
    Rt = t(R)
    G = torch.zeros((m, m), dtype=torch.float64, device=device)
    num = torch.zeros((), dtype=torch.float64, device=device)
    den = torch.zeros((), dtype=torch.float64, device=device)
    for r0 in range(0, n, rows):
        Qb, Wb = t(Q[r0:r0 + rows]), t(W[r0:r0 + rows])
        G += Qb.t() @ Qb
        num += torch.sum((Wb - Qb @ Rt) ** 2)
        den += torch.sum(Wb ** 2)
    St = t(S)
    eye = torch.eye(m, dtype=torch.float64, device=device)
    return {"orth_S_2": float(torch.linalg.matrix_norm(eye - St.t() @ St, ord=2)),
            "orth_Q_2": float(torch.linalg.matrix_norm(eye - G, ord=2)),
            "relres_F": float(torch.sqrt(num) / torch.sqrt(den))}
