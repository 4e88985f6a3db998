"""Randomized GMRES on the B200 (reference ``krylov.py``: SparseMatrix
``:28-83``, arnoldi ``:176-199``, gmres ``:229-319``).

The Arnoldi step is the device RGS column step fed by a CSR SpMV kernel.
The whole step - SpMV (with the 1/alpha scaling), sketch of w, sketched
least-squares solve, projection update, sketch of q', finalize/append,
normalisation and the progressive Givens rotation - is enqueued on one
stream without host synchronisation; the host polls the device status block
(convergence / lucky breakdown) every few steps and the kernels enqueued
past a stop return immediately.  The final (k x k) triangular solve for y
runs on the host, x = (||b|| / alpha) Q y on the device.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse
import torch

from . import _lib
from ._lib import call, stream_ptr
from .gram_schmidt import (BREAKDOWN_FACTOR, HOUSEHOLDER_QR, GsVariant, LazyFactors, LsqSolver,
                           QrFactors, RgsState)
from .precision import MIXED32_64, PrecisionPolicy
from .sketch import SketchKind

# SGS_W_SMALL_GRID=1: sketch w = A q with one CTA per 4 tiles (128 CTAs at c3)
# instead of one tile per CTA (same partials): the LS cluster that follows
# then launches beside it and overlaps its pre-wait part (srht -> LS gap
# 8.6 -> 0.8 us), but one fp64 column on 64 CTAs takes 46 us instead of 9
# (c3 fp32 basis, one-sync: 3686 -> 3310 steps/s).  Off by default.
_W_SMALL_GRID = os.environ.get("SGS_W_SMALL_GRID", "0") == "1"

# SGS_SPMV_SRHT=1: the SRHT of w fused into the SpMV (sgs_csr_spmv_srht: the
# CTA completing a 4096-row tile transforms it from L2, bit-identical
# partials).  Off by default: measured slower at c3 - the per-CTA publication
# (fence + tile counter) and the tile transforms inside the SpMV grid cost
# 46.7 - 35.0 us of SpMV time against the 9.6 us launch they replace (one-sync
# fp32 basis 3763 -> 3628 Arnoldi steps/s, profiles/r02g_spmv_srht_ab.json).
_SPMV_SRHT = os.environ.get("SGS_SPMV_SRHT", "0") == "1"

__all__ = ["SparseMatrix", "Ilu0Preconditioner", "ilu0", "arnoldi", "gmres", "gmres_restarted",
           "ArnoldiDecomposition", "GmresResult", "RestartedResult"]

_POLL = 8  # Arnoldi steps between status polls
_HALO = os.environ.get("SGS_HALO", "1") != "0"  # row-sharded SpMV: halo window (else all-gather)


@dataclass
class SparseMatrix:
    """Square CSR matrix with explicit index arrays (krylov.py:28-83)."""

    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    symmetric_expansion_applied: bool = False

    @classmethod
    def from_coo(cls, n: int, rows, cols, vals, symmetric: bool = False) -> "SparseMatrix":
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.float64)
        if not (rows.shape == cols.shape == vals.shape):
            raise ValueError("coordinate arrays have mismatched lengths")
        if rows.size and (rows.min() < 0 or rows.max() >= n or cols.min() < 0 or cols.max() >= n):
            raise ValueError("coordinate index out of range")
        if symmetric:
            off = rows != cols
            rows, cols, vals = (np.concatenate([rows, cols[off]]),
                                np.concatenate([cols, rows[off]]),
                                np.concatenate([vals, vals[off]]))
        m = scipy.sparse.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr()
        m.sum_duplicates()
        return cls(n=n, row_ptr=m.indptr.copy(), col_idx=m.indices.copy(),
                   values=m.data.astype(np.float64), symmetric_expansion_applied=symmetric)

    @classmethod
    def from_scipy(cls, m) -> "SparseMatrix":
        m = scipy.sparse.csr_matrix(m)
        if m.shape[0] != m.shape[1]:
            raise ValueError("matrix must be square")
        m.sum_duplicates()
        return cls(n=m.shape[0], row_ptr=m.indptr.copy(), col_idx=m.indices.copy(),
                   values=m.data.astype(np.float64))

    def to_scipy(self) -> scipy.sparse.csr_matrix:
        return scipy.sparse.csr_matrix((self.values, self.col_idx, self.row_ptr),
                                       shape=(self.n, self.n))

    # ---- device ------------------------------------------------------------------
    def device_arrays(self, device=None) -> tuple:
        _lib.require_cuda()
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        cache = self.__dict__.setdefault("_dev_cache", {})
        d = cache.get(str(dev))
        if d is None:
            if int(self.row_ptr[-1]) >= 2**31:
                raise ValueError("nnz exceeds int32 CSR indexing")
            d = (torch.from_numpy(np.asarray(self.row_ptr, dtype=np.int32)).to(dev),
                 torch.from_numpy(np.asarray(self.col_idx, dtype=np.int32)).to(dev),
                 torch.from_numpy(np.asarray(self.values, dtype=np.float64)).to(dev))
            cache[str(dev)] = d
        return d

    def spmv_into(self, x_ptr: int, x_code: int, y: torch.Tensor, alpha=None, status=None,
                  xdiv_ptr=None):
        rp, ci, va = self.device_arrays(y.device)
        call("sgs_csr_spmv", self.n, rp.data_ptr(), ci.data_ptr(), va.data_ptr(), x_ptr, x_code,
             xdiv_ptr, alpha.data_ptr() if alpha is not None else None, y.data_ptr(),
             status.ptr if status is not None else None, stream_ptr())

    def matvec(self, x):
        """A @ x in binary64 (numpy in -> numpy out; CUDA tensor in -> CUDA out)."""
        if isinstance(x, torch.Tensor) and x.is_cuda:
            xd = x if x.dtype in (torch.float32, torch.float64) else x.to(torch.float64)
            xd = xd.contiguous()
            y = torch.empty(self.n, dtype=torch.float64, device=x.device)
            self.spmv_into(xd.data_ptr(), _lib.dtype_code(xd.dtype), y)
            return y
        xn = np.asarray(x, dtype=np.float64)
        _lib.require_cuda()
        xd = torch.from_numpy(np.ascontiguousarray(xn)).cuda()
        y = torch.empty(self.n, dtype=torch.float64, device=xd.device)
        self.spmv_into(xd.data_ptr(), _lib.SGS_F64, y)
        return y.cpu().numpy()

    def __post_init__(self):
        self.__dict__.setdefault("_dev_cache", {})

    def row_block(self, row0: int, n_rows: int, device=None) -> "_RowBlock":
        """Rows [row0, row0 + n_rows) of the operator (global column indices),
        for a row-sharded solve."""
        return _RowBlock(self, row0, n_rows, device)


class _RowBlock:
    """A contiguous row block of a SparseMatrix on the device; its SpMV takes
    the full input vector and writes the block's rows."""

    def __init__(self, A: SparseMatrix, row0: int, n_rows: int, device=None, col0: int = 0):
        """``col0``: the input vector starts at global column col0 (a halo
        window); column indices are stored relative to it."""
        _lib.require_cuda()
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        lo, hi = int(A.row_ptr[row0]), int(A.row_ptr[row0 + n_rows])
        rp = np.asarray(A.row_ptr[row0:row0 + n_rows + 1], dtype=np.int64) - lo
        self.n, self.n_rows, self.row0 = A.n, n_rows, row0
        self.rp = torch.from_numpy(rp.astype(np.int32)).to(dev)
        ci = np.asarray(A.col_idx[lo:hi], dtype=np.int64) - int(col0)
        self.ci = torch.from_numpy(ci.astype(np.int32)).to(dev)
        self.va = torch.from_numpy(np.asarray(A.values[lo:hi], dtype=np.float64)).to(dev)

    def spmv_into(self, x_ptr: int, x_code: int, y: torch.Tensor, alpha=None, status=None):
        call("sgs_csr_spmv", self.n_rows, self.rp.data_ptr(), self.ci.data_ptr(),
             self.va.data_ptr(), x_ptr, x_code, None,
             alpha.data_ptr() if alpha is not None else None, y.data_ptr(),
             status.ptr if status is not None else None, stream_ptr())


class Ilu0Preconditioner:
    """Zero-fill incomplete LU factors on A's pattern (krylov.py:86-100).

    The factors live on the device as one CSR array F (strict lower part = L
    with an implied unit diagonal, the rest = U), with the two level orders of
    ``sgs_ilu0_analyse``; ``solve(v)`` applies M^{-1} v = U^{-1} (L^{-1} v)
    with the two sync-free sweep kernels of ``sgs_ilu0_solve``.  ``L`` and
    ``U`` are the reference's scipy CSR matrices, copied from the device on
    first use.  Built by ``ilu0(A)``, or from host factors
    ``Ilu0Preconditioner(L, U)`` as the reference's dataclass is.  One
    preconditioner runs one solve at a time (its control block and sweep
    buffer are shared by its launches)."""

    def __init__(self, L=None, U=None, *, _device=None):
        if _device is not None:
            (self.n, self._rp, self._ci, self._F, self._perm_l, self._perm_u, self._ctl) = _device
            self._L = self._U = None
        else:
            if L is None or U is None:
                raise TypeError("Ilu0Preconditioner needs L and U")
            _lib.require_cuda()
            L = scipy.sparse.csr_matrix(L)
            U = scipy.sparse.csr_matrix(U)
            n = L.shape[0]
            full = (scipy.sparse.tril(L, k=-1, format="csr") + U).tocsr()
            full.sum_duplicates()
            full.sort_indices()
            if np.any(full.diagonal() == 0.0):
                raise np.linalg.LinAlgError("A is singular: zero entry on diagonal.")
            dev = torch.device("cuda", torch.cuda.current_device())
            self.n = n
            self._rp = torch.from_numpy(full.indptr.astype(np.int32)).to(dev)
            self._ci = torch.from_numpy(full.indices.astype(np.int32)).to(dev)
            self._F = torch.from_numpy(full.data.astype(np.float64)).to(dev)
            self._ctl = torch.zeros(2, dtype=torch.int64, device=dev)
            self._perm_l, self._perm_u = _ilu_analyse(n, self._rp, self._ci, self._ctl)
            self._L, self._U = L, U
        self._tmp = torch.empty(max(self.n, 1), dtype=torch.float64, device=self._F.device)
        call("sgs_ilu0_pending_fill", self._tmp.data_ptr(), self.n, stream_ptr())

    # ---- host views (reference dataclass fields) ----------------------------------
    def _host_full(self):
        return scipy.sparse.csr_matrix((self._F.cpu().numpy(), self._ci.cpu().numpy(),
                                        self._rp.cpu().numpy()), shape=(self.n, self.n))

    @property
    def L(self) -> scipy.sparse.csr_matrix:
        if self._L is None:
            full = self._host_full()
            self._L = (scipy.sparse.tril(full, k=-1, format="csr")
                       + scipy.sparse.eye(self.n, format="csr")).tocsr()
        return self._L

    @property
    def U(self) -> scipy.sparse.csr_matrix:
        if self._U is None:
            self._U = scipy.sparse.triu(self._host_full(), k=0, format="csr")
        return self._U

    # ---- device solve ---------------------------------------------------------
    def solve_into(self, x_ptr: int, x_code: int, out: torch.Tensor, xdiv_ptr=None,
                   status=None) -> None:
        """out = M^{-1} x on the current stream (x binary32/64 at x_ptr, distinct
        from out; with xdiv_ptr the input is cast(x / *xdiv) first, as
        SparseMatrix.spmv_into)."""
        call("sgs_ilu0_solve", self.n, self._rp.data_ptr(), self._ci.data_ptr(),
             self._F.data_ptr(), self._perm_l.data_ptr(), self._perm_u.data_ptr(), x_ptr, x_code,
             xdiv_ptr, self._tmp.data_ptr(), out.data_ptr(), self._ctl.data_ptr(),
             status.ptr if status is not None else None, stream_ptr())

    def solve(self, v):
        """M^{-1} v in binary64 (numpy in -> numpy out; CUDA tensor in -> CUDA out)."""
        on_dev = isinstance(v, torch.Tensor) and v.is_cuda
        if on_dev:
            vd = v if v.dtype in (torch.float32, torch.float64) else v.to(torch.float64)
            vd = vd.contiguous()
        else:
            vd = torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=np.float64))).to(
                self._F.device)
        if tuple(vd.shape) != (self.n,):
            raise ValueError("vector length mismatch")
        out = torch.empty(self.n, dtype=torch.float64, device=self._F.device)
        self.solve_into(vd.data_ptr(), _lib.dtype_code(vd.dtype), out)
        return out if on_dev else out.cpu().numpy()


def _ilu_analyse(n, rp, ci, ctl):
    dev = rp.device
    perm_l = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    perm_u = torch.empty_like(perm_l)
    work = torch.empty(int(_lib.load().sgs_ilu0_analysis_work_elems(n)), dtype=torch.int32,
                       device=dev)
    call("sgs_ilu0_analyse", n, rp.data_ptr(), ci.data_ptr(), perm_l.data_ptr(),
         perm_u.data_ptr(), work.data_ptr(), ctl.data_ptr(), stream_ptr())
    return perm_l, perm_u


def ilu0(A: SparseMatrix, pivot_tol: float = 1e-30) -> Ilu0Preconditioner:
    """ILU(0) on the device (krylov.py:103-151): the reference's row-oriented
    IKJ elimination, bit-identical (one thread per row, rows released in
    level order).  Raises ValueError on a structural zero diagonal and
    ZeroDivisionError on a pivot below pivot_tol, naming the same row."""
    rp, ci, va = A.device_arrays()
    n = A.n
    dev = va.device
    ctl = torch.zeros(2, dtype=torch.int64, device=dev)
    perm_l, perm_u = _ilu_analyse(n, rp, ci, ctl)
    F = torch.empty_like(va)
    diag = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    flags = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
    aux = torch.empty(2, dtype=torch.int64, device=dev)
    call("sgs_ilu0_factor", n, rp.data_ptr(), ci.data_ptr(), va.data_ptr(), F.data_ptr(),
         diag.data_ptr(), perm_l.data_ptr(), flags.data_ptr(), ctl.data_ptr(), aux.data_ptr(),
         float(pivot_tol), stream_ptr())
    if n:
        a = aux.cpu().numpy().view(np.uint64)
        if int(a[0]) != n:
            raise ValueError(f"structural zero diagonal at row {int(a[0])}")
        if int(a[1]) != 2**64 - 1:
            key = int(a[1])
            raise ZeroDivisionError(f"ILU(0) pivot too small at row {key >> 1 if key & 1 else 0}")
    return Ilu0Preconditioner(_device=(n, rp, ci, F, perm_l, perm_u, ctl))


def _as_preconditioner(pre):
    if pre is None or isinstance(pre, Ilu0Preconditioner):
        return pre
    if hasattr(pre, "L") and hasattr(pre, "U"):  # the reference's Ilu0Preconditioner
        return Ilu0Preconditioner(pre.L, pre.U)
    raise TypeError("preconditioner must be an Ilu0Preconditioner (or carry L and U factors)")


@dataclass
class ArnoldiDecomposition:
    Q: np.ndarray
    H: np.ndarray
    R: np.ndarray
    beta: float
    breakdown: bool = False


@dataclass
class GmresResult:
    x: object
    residual_history: np.ndarray
    final_residual: float
    iterations: int
    converged: bool
    breakdown: bool
    factors: QrFactors | None = None


def _check_variant(variant):
    if variant is not GsVariant.RGS and getattr(variant, "value", None) != "rgs":
        raise NotImplementedError("the device Krylov path implements the randomized "
                                  "Gram-Schmidt variant (GsVariant.RGS)")


def _to_device_f64(b, n: int, device) -> torch.Tensor:
    if isinstance(b, torch.Tensor) and b.is_cuda:
        t = b.to(torch.float64).contiguous()
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(b, dtype=np.float64))).to(device)
    if tuple(t.shape) != (n,):
        raise ValueError("right-hand side length mismatch")
    return t


class _Workspace:
    def __init__(self, n: int, device):
        self.w = torch.empty(n, dtype=torch.float64, device=device)
        self.v = torch.empty(n, dtype=torch.float64, device=device)
        self.z = None  # M^{-1} x when preconditioned
        self.nrm = torch.zeros(4, dtype=torch.float64, device=device)
        self.work = torch.empty(int(_lib.load().sgs_norm2_work_elems(n)), dtype=torch.float64,
                                device=device)

    def norm(self, x: torch.Tensor, out_slot: int = 0) -> None:
        call("sgs_norm2", x.data_ptr(), _lib.dtype_code(x.dtype), x.numel(),
             self.nrm[out_slot:].data_ptr(), self.work.data_ptr(), stream_ptr())


class _Dist:
    """Row sharding of an RGMRES solve: this rank owns
    operator rows [row0, row0 + n_loc) and the same rows of every n-vector
    (shard_rows, aligned to the sketch's tiles).  The RGS state is sharded as
    in RgsState(comm=...): one k-vector all-reduce per sketch, replicated LS
    and Givens.  Norms all-reduce their squares.  The SpMV input is a halo
    window: the columns this rank's rows touch form [wlo, whi), and each
    step receives only the other ranks' rows inside it by point-to-point
    messages (for c3's stencil one 128 x 128 plane per neighbour instead of
    the whole vector); a window wider than half the vector falls back to the
    all-gather."""

    def __init__(self, comm, A: SparseMatrix, align: int, device):
        from .workloads import shard_rows
        self.comm = comm
        self.n = A.n
        self.counts = [shard_rows(A.n, comm.world, r, align)[1] for r in range(comm.world)]
        self.row0, self.n_loc = shard_rows(A.n, comm.world, comm.rank, align)
        if self.n_loc < 1:
            raise ValueError("more ranks than row blocks")
        self.block = A.row_block(self.row0, self.n_loc, device)
        self.device = device
        self._full = {}
        self._win = {}
        self._plan_halo(A)

    def _plan_halo(self, A: SparseMatrix) -> None:
        import torch.distributed as tdist
        lo, hi = int(A.row_ptr[self.row0]), int(A.row_ptr[self.row0 + self.n_loc])
        cols = np.asarray(A.col_idx[lo:hi])
        wlo = min(int(cols.min()) if cols.size else self.row0, self.row0)
        whi = max(int(cols.max()) + 1 if cols.size else 0, self.row0 + self.n_loc)
        world, me = self.comm.world, self.comm.rank
        win = torch.tensor([wlo, whi], dtype=torch.int64, device=self.device)
        allw = [torch.empty_like(win) for _ in range(world)]
        tdist.all_gather(allw, win, group=self.comm.group)
        allw = [tuple(int(v) for v in t.cpu()) for t in allw]
        rows = [sum(self.counts[:r]) for r in range(world)]  # first row of each rank
        self.recvs, self.sends = [], []
        for q in range(world):
            if q == me:
                continue
            q0, q1 = rows[q], rows[q] + self.counts[q]
            a, b = max(wlo, q0), min(whi, q1)
            if a < b:
                self.recvs.append((q, a, b))       # rows [a, b) of rank q into the window
            r0_, r1_ = allw[q]
            a, b = max(r0_, self.row0), min(r1_, self.row0 + self.n_loc)
            if a < b:
                self.sends.append((q, a, b))       # my rows [a, b) to rank q
        # the halo path when the window is small; every rank decides identically
        # (each rank's choice only affects its own receives and the matching sends)
        widths = [w[1] - w[0] for w in allw]
        self.halo = _HALO and max(widths) <= self.n // 2
        self.wlo, self.whi = wlo, whi
        if self.halo:
            self.wblock = _RowBlock(A, self.row0, self.n_loc, self.device, col0=wlo)

    def window(self, x_local: torch.Tensor):
        """(input vector, row block) for this rank's SpMV: the halo window of
        x (or the all-gathered x when the window is wide)."""
        if not self.halo:
            return self.full(x_local), self.block
        import torch.distributed as tdist
        buf = self._win.get(x_local.dtype)
        if buf is None:
            buf = self._win[x_local.dtype] = torch.empty(self.whi - self.wlo,
                                                          dtype=x_local.dtype,
                                                          device=self.device)
        o = self.row0 - self.wlo
        buf[o:o + self.n_loc].copy_(x_local)
        ops = []
        # q is a rank WITHIN comm.group (TorchComm.rank is dist.get_rank(group)):
        # pass it as group_peer (P2POp's positional peer is a global rank)
        for q, a, b in self.recvs:
            ops.append(tdist.P2POp(tdist.irecv, buf[a - self.wlo:b - self.wlo],
                                   group=self.comm.group, group_peer=q))
        for q, a, b in self.sends:
            ops.append(tdist.P2POp(tdist.isend, x_local[a - self.row0:b - self.row0],
                                   group=self.comm.group, group_peer=q))
        if ops:
            for req in tdist.batch_isend_irecv(ops):
                req.wait()
        return buf, self.wblock

    def full(self, x_local: torch.Tensor) -> torch.Tensor:
        buf = self._full.get(x_local.dtype)
        if buf is None:
            buf = self._full[x_local.dtype] = torch.empty(self.n, dtype=x_local.dtype,
                                                          device=self.device)
        self.comm.allgather_rows(x_local, self.counts, buf)
        return buf

    def norm_(self, nrm: torch.Tensor, slot: int) -> None:
        """nrm[slot] holds this rank's norm; make it the global one."""
        t = nrm[slot:slot + 1]
        sq = t * t
        self.comm.allreduce_(sq)
        torch.sqrt(sq, out=t)

    def local(self, v_full: torch.Tensor) -> torch.Tensor:
        return v_full[self.row0:self.row0 + self.n_loc]


def _eff_matvec_into(A: SparseMatrix, M, ws: _Workspace, x_ptr: int, x_code: int,
                     out: torch.Tensor, alpha=None, status=None, xdiv_ptr=None) -> None:
    """out = A M^{-1} x (/ alpha): the right-preconditioned operator of
    krylov.py:251-255 (M = None: plain A)."""
    if M is None:
        A.spmv_into(x_ptr, x_code, out, alpha=alpha, status=status, xdiv_ptr=xdiv_ptr)
        return
    if ws.z is None:
        ws.z = torch.empty(A.n, dtype=torch.float64, device=out.device)
    M.solve_into(x_ptr, x_code, ws.z, xdiv_ptr=xdiv_ptr, status=status)
    A.spmv_into(ws.z.data_ptr(), _lib.SGS_F64, out, alpha=alpha, status=status)


def _operator_norm_estimate(A: SparseMatrix, ws: _Workspace, iters: int = 20,
                            M=None, dist: _Dist | None = None) -> torch.Tensor:
    """Device power iteration (krylov.py:213-226) on A M^{-1}; returns a
    1-element device tensor (-1 when the reference would return 0.0)."""
    n = A.n if dist is None else dist.n_loc
    sigma = torch.ones(1, dtype=torch.float64, device=ws.v.device)
    call("sgs_cos_init_at", ws.v.data_ptr(), n, 0 if dist is None else dist.row0, stream_ptr())
    ws.norm(ws.v, 0)
    if dist is not None:
        dist.norm_(ws.nrm, 0)
    call("sgs_scale", ws.v.data_ptr(), 1.0, ws.nrm.data_ptr(), 1, ws.v.data_ptr(), n, stream_ptr())
    for _ in range(iters):
        if dist is None:
            _eff_matvec_into(A, M, ws, ws.v.data_ptr(), _lib.SGS_F64, ws.w)
        else:
            xw, blk = dist.window(ws.v)
            blk.spmv_into(xw.data_ptr(), _lib.SGS_F64, ws.w)
        ws.norm(ws.w, 1)
        if dist is not None:
            dist.norm_(ws.nrm, 1)
        call("sgs_power_step", ws.w.data_ptr(), ws.nrm[1:].data_ptr(), ws.v.data_ptr(),
             sigma.data_ptr(), n, stream_ptr())
    return sigma


class _ArnoldiEngine:
    """Device Arnoldi driver over an RgsState (one stream, no per-step sync).

    With an SRHT sketch on 4096-row tiles a step is: the head (in-place
    normalisation q_i = q'_i / r_ii together with the previous step's Givens
    update), the SpMV (1/alpha folded in), the SRHT of w, the LS solve, the
    fused column kernel (update + sketch of q'_{i+1}) and the LS finalize.
    Otherwise the generic path (separate SpMV, sketch and normalisation).

    ``lagged``: the one-synchronisation RGS-Arnoldi of PAPER.md:260-261.  The
    matvec runs on the unnormalised q'_c right after its column kernel, and
    one LS launch finalizes column c (r_cc = ||s'_c||) and solves column c+1
    from p_{c+1} = (Theta A q'_c) / r_cc.  A step is then the column kernel
    (w = A q'_c / r_cc formed on the fly, q_c normalised in its stream), the
    SpMV, the SRHT of w and that LS launch, which also applies the Givens
    update of step c - 1; sharded, the two k-vectors share one all-reduce."""

    def __init__(self, A: SparseMatrix, theta, policy, solver, m: int,
                 breakdown_factor: float = BREAKDOWN_FACTOR, phi=None, M=None,
                 dist: _Dist | None = None, lagged: bool = False):
        self.A = A
        self.M = M
        self.m = m
        self.dist = dist
        self.lagged = bool(lagged)
        if self.lagged and phi is not None:
            raise NotImplementedError("certification sketches (phi) are not formed by the "
                                      "one-synchronisation Arnoldi")
        shard = {} if dist is None else {"comm": dist.comm, "row0": dist.row0,
                                         "n_local": dist.n_loc}
        self.state = RgsState(theta, policy, solver, phi=phi, capacity=m + 2,
                              breakdown_factor=breakdown_factor, **shard)
        st = self.state
        if st.n != A.n:
            raise ValueError("sketch ambient dimension does not match the operator")
        self.fused = st.fused
        self.n_loc = st.n_local
        dev = st.device
        self.ws = _Workspace(self.n_loc, dev)
        self.cs = torch.zeros(m + 1, dtype=torch.float64, device=dev)
        self.sn = torch.zeros_like(self.cs)
        self.g = torch.zeros(m + 2, dtype=torch.float64, device=dev)
        self.T = torch.zeros((m + 1, m + 2), dtype=torch.float64, device=dev)  # T[i] = column i
        self.hist = torch.zeros(m + 1, dtype=torch.float64, device=dev)
        self.norm_flag = torch.full((1,), -1, dtype=torch.int32, device=dev)
        self._owed = None  # step whose Givens update rides on the next step's head
        self._spsr = self._spmv_srht_scratch()
        if self.lagged:
            self._kv2 = (torch.empty(2 * st.k, dtype=torch.float64, device=dev)
                         if dist is not None else None)
            if not self.fused:
                self._wdiv = torch.empty(self.n_loc, dtype=torch.float64, device=dev)

    def _spmv_srht_scratch(self):
        """Scratch of the fused SpMV + SRHT launch (tile vectors, monotonic
        counters), or None when the step takes two launches: a preconditioner
        (w = A M^-1 q), a sketch other than 4096-row-tile SRHT, k > 2048, or
        the generic (unfused) engine."""
        st = self.state
        th = st.theta
        if not (_SPMV_SRHT and not _W_SMALL_GRID and self.fused and self.M is None
                and th.kind in (SketchKind.PSRHT, SketchKind.BLOCK_SRHT)
                and th.log2_block >= 12 and st.k <= 2048 and st.row0 % 4096 == 0):
            return None
        lib = _lib.load()
        ntv = int(lib.sgs_spmv_srht_tilevec_elems(self.n_loc, st.k))
        nct = int(lib.sgs_spmv_srht_counter_elems(self.n_loc))
        if ntv <= 0 or nct <= 0:
            return None
        dev = st.device
        return (torch.empty(ntv, dtype=torch.float64, device=dev),
                torch.zeros(nct, dtype=torch.int64, device=dev))

    def _matvec_sketch(self, i: int, alpha) -> None:
        """w = (A q_i) / alpha into ws.w (q_i as stored, this rank's rows) and
        the SRHT partials of w into the state's p partials (st.nparts of
        them): one fused launch when possible, else the SpMV and the
        stand-alone sketch."""
        st, ws = self.state, self.ws
        if self._spsr is None:
            self._matvec(i, ws.w, alpha, st.status)
            st.theta.partials_into(ws.w.data_ptr(), _lib.SGS_F64, self.n_loc, 1, st._parts_p,
                                   n_local=self.n_loc, row0=st.row0, status=st.status,
                                   small_grid=_W_SMALL_GRID)
            return
        tv, cnt = self._spsr
        th = st.theta
        d = th.device_data(ws.w.device)
        if self.dist is None:
            rp, ci, va = self.A.device_arrays(ws.w.device)
            nrows, xp = self.A.n, st._qcol_ptr(i)
        else:
            xw, blk = self.dist.window(st._Q[i, :self.n_loc])
            rp, ci, va, nrows, xp = blk.rp, blk.ci, blk.va, blk.n_rows, xw.data_ptr()
        call("sgs_csr_spmv_srht", nrows, rp.data_ptr(), ci.data_ptr(), va.data_ptr(), xp,
             st.ccode, None, alpha.data_ptr() if alpha is not None else None, ws.w.data_ptr(),
             st.row0, th.log2_block, d["bits"].data_ptr() + (st.row0 // 32) * 4,
             d["samples"].data_ptr(), st.k, tv.data_ptr(), cnt.data_ptr(),
             st._parts_p.data_ptr(), st.status.ptr, stream_ptr())

    def _matvec(self, i: int, out: torch.Tensor, alpha, status) -> None:
        """out = (A M^{-1} q_i) / alpha over this rank's rows."""
        st = self.state
        if self.dist is None:
            _eff_matvec_into(self.A, self.M, self.ws, st._qcol_ptr(i), st.ccode, out,
                             alpha=alpha, status=status)
        else:
            xw, blk = self.dist.window(st._Q[i, :self.n_loc])
            blk.spmv_into(xw.data_ptr(), st.ccode, out, alpha=alpha, status=status)

    # ---- one-synchronisation (lagged) steps -----------------------------------------
    def _giv(self, c: int, alpha, tol):
        """Givens arrays for the LS launch finalizing column c (step c - 1)."""
        if c < 1 or (tol is None and alpha is None):
            return None
        return (self.cs, self.sn, self.g, self.T, self.hist, tol)

    def _lag_tail(self, c: int, s_raw, alpha, tol=None) -> None:
        """w = A M^{-1} q'_c (/ alpha) from the unnormalised column c, its sketch
        p', and the LS launch finalizing c and solving c + 1 (p = p' / r_cc).
        ``s_raw``: raw partials of s'_c (None for c = 0: s'_0 = p_0)."""
        st = self.state
        self._matvec_sketch(c, alpha)
        p_raw = (st._parts_p.data_ptr(), st.nparts, st.theta.scale)
        if self.dist is not None:  # one all-reduce of [s'; p'] (2k)
            k, kv = st.k, self._kv2
            srcs = [(p_raw, kv[k:])] if s_raw is None else [(s_raw, kv[:k]), (p_raw, kv[k:])]
            for (ptr, npart, _), dst in srcs:
                call("sgs_partials_reduce", ptr, npart, k, 1, 1.0, dst.data_ptr(), _lib.SGS_F64,
                     k, st.status.ptr, stream_ptr())
            self.dist.comm.allreduce_(kv if s_raw is not None else kv[k:])
            if s_raw is not None:
                s_raw = (kv.data_ptr(), 1, st.theta.scale)
            p_raw = (kv[k:].data_ptr(), 1, st.theta.scale)
        s_ptr, s_np, s_sc = s_raw if s_raw is not None else (None, 0, 1.0)
        st._ls(fin=c, s_parts=s_ptr, s_nparts=s_np, s_scale=s_sc, sol=c + 1, p_parts=p_raw[0],
               p_nparts=p_raw[1], p_scale=p_raw[2], lag=True, giv=self._giv(c, alpha, tol))

    def _start_lagged(self, bn: torch.Tensor, alpha) -> None:
        st, n = self.state, self.n_loc
        pp, pn, ps = st._sketch_parts(bn.data_ptr(), _lib.SGS_F64, n, st._parts_p,
                                      getattr(st, "_kvec_p", None))
        call("sgs_partials_reduce", pp, pn, st.k, 1, ps, st._P.data_ptr(), st.fcode, st.k,
             st.status.ptr, stream_ptr())
        st._column(0, bn.data_ptr(), _lib.SGS_F64, False, False)
        if self.m >= 1:
            self._lag_tail(0, None, alpha)
        else:
            st._ls(fin=0)
        st.m = 1

    def _step_lagged(self, i: int, alpha, tol) -> None:
        """Column i + 1 (its predecessor launch finalized column i and solved i + 1)."""
        st, ws = self.state, self.ws
        c = i + 1
        rii = st._R.data_ptr() + (i * st._cap + i) * 8
        if self.fused:
            s_raw = st._column(c, ws.w.data_ptr(), _lib.SGS_F64, True, True, w_div=rii,
                               combine=False)
        else:
            call("sgs_cast_div", ws.w.data_ptr(), _lib.SGS_F64, self._wdiv.data_ptr(),
                 _lib.SGS_F64, rii, self.n_loc, stream_ptr())
            s_raw = st._column(c, self._wdiv.data_ptr(), _lib.SGS_F64, True, True, combine=False)
        if c < self.m:
            self._lag_tail(c, s_raw, alpha, tol)
        else:  # last column: finalize only
            if self.dist is not None:
                k, kv = st.k, self._kv2
                call("sgs_partials_reduce", s_raw[0], s_raw[1], k, 1, 1.0, kv.data_ptr(),
                     _lib.SGS_F64, k, st.status.ptr, stream_ptr())
                self.dist.comm.allreduce_(kv[:k])
                s_raw = (kv.data_ptr(), 1, st.theta.scale)
            st._ls(fin=c, s_parts=s_raw[0], s_nparts=s_raw[1], s_scale=s_raw[2],
                   giv=self._giv(c, alpha, tol))
        st.m = c + 1  # the Givens update of step i ran in that LS launch

    def start(self, b_dev: torch.Tensor, b_norm_ptr, alpha=None) -> None:
        """Push b (this rank's rows; divided by ||b|| when b_norm_ptr is given)
        as column 0 (lagged: and run the first matvec, with ``alpha``)."""
        st, n = self.state, self.n_loc
        bn = self.ws.v
        call("sgs_cast_div", b_dev.data_ptr(), _lib.SGS_F64, bn.data_ptr(), _lib.SGS_F64,
             b_norm_ptr, n, stream_ptr())
        if self.lagged:
            self._start_lagged(bn, alpha)
            return
        if not self.fused:
            st._push_async(bn)
            return
        pp, pn, ps = st._sketch_parts(bn.data_ptr(), _lib.SGS_F64, n, st._parts_p,
                                      getattr(st, "_kvec_p", None))
        call("sgs_partials_reduce", pp, pn, st.k, 1, ps, st._P.data_ptr(), st.fcode, st.k,
             st.status.ptr, stream_ptr())
        st._phi_w(0, bn.data_ptr(), _lib.SGS_F64, n)
        st._column(0, bn.data_ptr(), _lib.SGS_F64, False, False)
        phq = st._phi_q_parts(0)
        st._ls(fin=0)
        st._phi_q_finish(0, phq)
        st.m = 1

    def step(self, i: int, alpha: torch.Tensor | None, tol: float | None) -> None:
        if self.lagged:
            self._step_lagged(i, alpha, tol)
            return
        st = self.state
        A, ws = self.A, self.ws
        if self.fused:
            # step head: q_i = cast(q'_i / r_ii) once, in place (one division per
            # entry instead of one per stored nonzero in the SpMV; the column
            # kernel then has no previous column left to normalise), and the
            # Givens update of step i-1 in the same launch (sgs_arnoldi_head)
            gi = -1 if self._owed is None else self._owed
            self._owed = None
            call("sgs_arnoldi_head", st._Q.data_ptr(), st.ccode, st.ldq, self.n_loc, i,
                 st._R.data_ptr(), st._cap, self.norm_flag.data_ptr(), gi, self.cs.data_ptr(),
                 self.sn.data_ptr(), self.g.data_ptr(), self.T.data_ptr(), self.T.shape[1],
                 self.hist.data_ptr(), -1.0 if tol is None else float(tol), st.status.ptr,
                 stream_ptr())
            self._matvec_sketch(i, alpha)
            pp, pn, ps = st._combine(st._parts_p, st.nparts, getattr(st, "_kvec_p", None))
            st._phi_w(i + 1, ws.w.data_ptr(), _lib.SGS_F64, self.n_loc)
            st._ls(sol=i + 1, p_parts=pp, p_nparts=pn, p_scale=ps)
            sp, sn, ss = st._column(i + 1, ws.w.data_ptr(), _lib.SGS_F64, False, True)
            phq = st._phi_q_parts(i + 1)
            st._ls(fin=i + 1, s_parts=sp, s_nparts=sn, s_scale=ss)
            st._phi_q_finish(i + 1, phq)
            st.m = i + 2
        else:
            self._matvec(i, ws.w, alpha, st.status)
            st._push_async(ws.w)
        if tol is not None or alpha is not None:
            if self.fused:
                self._owed = i
            else:
                self._givens(i, tol)

    def _givens(self, i: int, tol: float | None) -> None:
        st = self.state
        call("sgs_givens_step", st._R.data_ptr(), st._cap, i, self.cs.data_ptr(),
             self.sn.data_ptr(), self.g.data_ptr(), self.T.data_ptr(), self.T.shape[1],
             self.hist.data_ptr(), -1.0 if tol is None else float(tol), st.status.ptr,
             stream_ptr())

    def run(self, alpha, tol) -> dict:
        """Steps 0..m-1 with periodic status polls; returns the final status."""
        st = self.state
        pending = []
        for i in range(self.m):
            self.step(i, alpha, tol)
            if (i + 1) % _POLL == 0 and i + 1 < self.m:
                hb = torch.empty(8, dtype=torch.int64, pin_memory=True)
                hb.copy_(st.status.buf, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record()
                pending.append((ev, hb))
                if len(pending) >= 2:
                    ev0, hb0 = pending.pop(0)
                    ev0.synchronize()
                    if int(hb0[0]) != 0:
                        break
        if self._owed is not None:  # the last step's Givens update (no head follows)
            self._givens(self._owed, tol)
            self._owed = None
        out = st._sync_status()
        if self.lagged:
            # every committed column but the newest was normalised by its
            # successor's column kernel; a breakdown in the finalize of column
            # ncols means that kernel ran for the newest committed one too
            nc = out["ncols"]
            covered = (out["code"] == _lib.ST_BREAKDOWN
                       and out["column"] == nc + 1)
            if nc > 0 and not covered:
                st._normalize(nc - 1, guarded=False)
            return out
        # fused path: columns are normalised by the step heads; the newest
        # committed one is still q'/r_ii unless a head (run after a stop, or a
        # breakdown that left the previous column newest) already covered it
        if self.fused and out["ncols"] > 0 and int(self.norm_flag) < out["ncols"] - 1:
            st._normalize(out["ncols"] - 1, guarded=False)
        return out


def _make_dist(comm, A: SparseMatrix, theta, M) -> _Dist | None:
    if comm is None:
        return None
    if M is not None:
        raise NotImplementedError("ILU(0) preconditioning is single-GPU (its sweeps run in "
                                  "global dependency order)")
    from .sketch import as_device_sketch
    device = torch.device("cuda", torch.cuda.current_device())
    return _Dist(comm, A, as_device_sketch(theta).row_align(), device)


def arnoldi(A: SparseMatrix, b, m: int, variant: GsVariant = GsVariant.RGS, theta=None,
            policy: PrecisionPolicy = MIXED32_64, solver: LsqSolver = HOUSEHOLDER_QR,
            phi=None, *, comm=None, lagged: bool = False) -> ArnoldiDecomposition:
    """m-step RGS-Arnoldi (krylov.py:176-199); fewer columns on a lucky
    breakdown.  With ``comm`` the rows are sharded across the ranks (b is the
    full vector on every rank; Q holds this rank's rows, H and R are
    replicated).  ``lagged``: the one-synchronisation variant of
    PAPER.md:260-261 (see _ArnoldiEngine)."""
    _check_variant(variant)
    if theta is None:
        raise ValueError("the randomized variant needs a sketch operator")
    _lib.require_cuda()
    dist = _make_dist(comm, A, theta, None)
    eng = _ArnoldiEngine(A, theta, policy, solver, m, phi=phi, dist=dist, lagged=lagged)
    st = eng.state
    b_dev = _to_device_f64(b, A.n, st.device)
    eng.start(b_dev if dist is None else dist.local(b_dev).contiguous(), None)
    s0 = eng.run(alpha=None, tol=None)
    breakdown = s0["code"] == _lib.ST_BREAKDOWN
    if s0["code"] == _lib.ST_RANK:
        raise np.linalg.LinAlgError("sketched basis numerically rank deficient")
    if s0["code"] and s0["ncols"] == 0:
        st._raise_status(s0)
    R = st.R
    return ArnoldiDecomposition(Q=st.Q, H=R[:, 1:].copy(), R=R, beta=float(R[0, 0]),
                                breakdown=breakdown)


def gmres(A: SparseMatrix, b, m: int, variant: GsVariant = GsVariant.RGS, theta=None,
          policy: PrecisionPolicy = MIXED32_64, solver: LsqSolver = HOUSEHOLDER_QR,
          preconditioner=None, tol: float | None = None, phi=None, *,
          comm=None, lagged: bool = False) -> GmresResult:
    """Single-cycle RGS-GMRES(m) with progressive Givens rotations (krylov.py:229-319),
    right-preconditioned by an ILU(0) ``preconditioner`` when given.  With
    ``comm`` (distributed.TorchComm) the operator rows and every n-vector are
    sharded across the ranks (one tile-aligned row block each); b is the full
    vector on every rank and so is the returned x.  ``lagged``: Arnoldi by the
    one-synchronisation RGS of PAPER.md:260-261 (see _ArnoldiEngine)."""
    _check_variant(variant)
    M = _as_preconditioner(preconditioner)
    if theta is None:
        raise ValueError("the randomized variant needs a sketch operator")
    _lib.require_cuda()
    device = torch.device("cuda", torch.cuda.current_device())
    return_numpy = not (isinstance(b, torch.Tensor) and b.is_cuda)
    dist = _make_dist(comm, A, theta, M)
    b_dev = _to_device_f64(b, A.n, device)
    b_loc = b_dev if dist is None else dist.local(b_dev).contiguous()
    n_loc = A.n if dist is None else dist.n_loc
    ws0 = _Workspace(n_loc, device)
    ws0.norm(b_loc, 0)
    if dist is not None:
        dist.norm_(ws0.nrm, 0)
    b_norm = float(ws0.nrm[0])  # host sync: the zero-rhs branch needs it
    if b_norm == 0.0:
        x0 = np.zeros(A.n) if return_numpy else torch.zeros(A.n, dtype=torch.float64,
                                                             device=device)
        return GmresResult(x=x0, residual_history=np.zeros(0), final_residual=0.0,
                           iterations=0, converged=True, breakdown=False)
    eng = _ArnoldiEngine(A, theta, policy, solver, m, phi=phi, M=M, dist=dist, lagged=lagged)
    st = eng.state
    alpha = _operator_norm_estimate(A, eng.ws, M=M, dist=dist)
    if float(alpha) <= 0.0:
        raise np.linalg.LinAlgError("operator norm estimate is zero")
    eng.start(b_loc, ws0.nrm.data_ptr(), alpha)
    s1 = eng.run(alpha=alpha, tol=tol)
    code = s1["code"]
    if code == _lib.ST_RANK:
        raise np.linalg.LinAlgError("sketched basis numerically rank deficient")
    if code and s1["ncols"] == 0:
        st._raise_status(s1)
    breakdown = code == _lib.ST_BREAKDOWN
    k = s1["iters"]
    hist = eng.hist[:k].cpu().numpy()
    x = torch.zeros(n_loc, dtype=torch.float64, device=device)
    if k > 0:
        T = eng.T[:k, :k].t().cpu().numpy()
        g = eng.g[:k].cpu().numpy()
        y = scipy.linalg.solve_triangular(T, g, lower=False)
        yd = torch.from_numpy(y).to(device)
        z = torch.empty(n_loc, dtype=torch.float64, device=device)
        call("sgs_gemv_f64", st._Q.data_ptr(), st.ccode, st.ldq, n_loc, k, yd.data_ptr(),
             z.data_ptr(), stream_ptr())
        call("sgs_scale", z.data_ptr(), b_norm, alpha.data_ptr(), 0, x.data_ptr(), n_loc,
             stream_ptr())
        if M is not None:  # x = M^{-1} x_tilde (krylov.py:309-310)
            M.solve_into(x.data_ptr(), _lib.SGS_F64, z)
            x = z
    # true residual ||b - A x|| / ||b|| in binary64
    ax = eng.ws.w
    if dist is None:
        A.spmv_into(x.data_ptr(), _lib.SGS_F64, ax)
    else:
        x = dist.full(x).clone()
        dist.block.spmv_into(x.data_ptr(), _lib.SGS_F64, ax)
    call("sgs_rsub", b_loc.data_ptr(), ax.data_ptr(), n_loc, stream_ptr())
    eng.ws.norm(ax, 2)
    if dist is not None:
        dist.norm_(eng.ws.nrm, 2)
    true_res = float(eng.ws.nrm[2]) / b_norm
    converged = (true_res <= max(tol, 0.0)) if tol is not None else False
    return GmresResult(x=x.cpu().numpy() if return_numpy else x,
                       residual_history=np.asarray(hist), final_residual=true_res,
                       iterations=k, converged=converged or breakdown, breakdown=breakdown,
                       factors=LazyFactors(st, st.m, device=not return_numpy))


@dataclass
class RestartedResult:
    x: object
    iterations: int
    cycles: list
    final_residual: float
    converged: bool


def gmres_restarted(A: SparseMatrix, b, theta, policy: PrecisionPolicy = MIXED32_64,
                    restart: int = 300, max_iters: int = 3000, tol: float = 1e-8,
                    solver: LsqSolver = HOUSEHOLDER_QR, preconditioner=None, *,
                    comm=None, lagged: bool = False) -> RestartedResult:
    """Restarted RGMRES(restart) for BASELINE config 3 (the reference is
    single-cycle, krylov.py:236-241; the wrapper is shared verbatim with the
    oracle): each cycle runs gmres(A, r, min(restart, max_iters - its), tol =
    tol * ||b|| / ||r||), then x += dx and r = b - A x in binary64; stop at
    ||r|| / ||b|| <= tol or its >= max_iters.  ``comm``: row-sharded, as gmres;
    ``lagged``: one-synchronisation Arnoldi, as gmres."""
    _lib.require_cuda()
    device = torch.device("cuda", torch.cuda.current_device())
    return_numpy = not (isinstance(b, torch.Tensor) and b.is_cuda)
    M = _as_preconditioner(preconditioner)
    dist = _make_dist(comm, A, theta, M)
    n_loc = A.n if dist is None else dist.n_loc
    b_dev = _to_device_f64(b, A.n, device)
    b_loc = b_dev if dist is None else dist.local(b_dev).contiguous()
    ws = _Workspace(n_loc, device)

    def rnorm(v, slot):
        ws.norm(v, slot)
        if dist is not None:
            dist.norm_(ws.nrm, slot)
        return float(ws.nrm[slot])

    b_norm = rnorm(b_loc, 0)
    x = torch.zeros(A.n, dtype=torch.float64, device=device)
    r = b_dev.clone()
    r_loc = torch.empty(n_loc, dtype=torch.float64, device=device)
    its, cycles = 0, []
    r_norm = b_norm
    while True:
        if b_norm == 0.0 or r_norm / b_norm <= tol or its >= max_iters:
            break
        res = gmres(A, r, m=min(restart, max_iters - its), theta=theta, policy=policy,
                    solver=solver, tol=tol * b_norm / r_norm, preconditioner=M, comm=comm,
                    lagged=lagged)
        cycles.append(res.iterations)
        its += res.iterations
        x += res.x
        if dist is None:
            A.spmv_into(x.data_ptr(), _lib.SGS_F64, r)
            call("sgs_rsub", b_dev.data_ptr(), r.data_ptr(), A.n, stream_ptr())
            r_norm = rnorm(r, 1)
        else:
            dist.block.spmv_into(x.data_ptr(), _lib.SGS_F64, r_loc)
            call("sgs_rsub", b_loc.data_ptr(), r_loc.data_ptr(), n_loc, stream_ptr())
            r_norm = rnorm(r_loc, 1)
            r.copy_(dist.full(r_loc))
        if res.iterations == 0:
            break
    rel = r_norm / b_norm if b_norm else 0.0
    return RestartedResult(x=x.cpu().numpy() if return_numpy else x, iterations=its,
                           cycles=cycles, final_residual=rel, converged=rel <= tol)
