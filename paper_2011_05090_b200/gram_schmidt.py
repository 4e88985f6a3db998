"""Randomized Gram-Schmidt on the B200: ``RgsState`` / ``rgs_factorize``.

Interface mirror of the reference's ``gram_schmidt.py`` (RgsState
``:228-347``, rgs_factorize ``:350-375``, certificates ``:474-487``,
BreakdownError ``:35-43``).  Per column the device runs, on torch's current
stream and without host synchronisation (SRHT sketches on 4096-row tiles):

1. ``sgs_rgs_update_srht``: q'_i = w_i - Q_{i-1} r in the coarse format
   (step 3), normalising q'_{i-1} in the same pass, with the sketch partials
   of q'_i in the epilogue (step 4);
2. ``sgs_ls_step``: finalize column i - r_ii, breakdown guard, S, R and the
   LS append (steps 5-7) - fused with the solve for column i+1 (step 2),
   whose work on the existing columns runs before the dependency wait.

In ``rgs_factorize`` the sketches P = Theta W of all columns are computed up
front in batched launches (bit-identical to per-column sketches), so a column
costs two launches; ``push`` (streaming) issues the solve and the finalize
as separate launches with the same arithmetic, so both paths agree bit for
bit.  Other sketch kinds take the generic path (separate update, sketch and
normalisation kernels).  Breakdown and rank deficiency are recorded on the
device and raised at the next synchronisation with the reference's exception
types and column numbers.
"""

from __future__ import annotations

import os

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _lib
from ._lib import call, stream_ptr
from .precision import MIXED32_64, UNIFIED64, PrecisionPolicy
from .sketch import SketchKind, SketchOperator, as_device_sketch

__all__ = [
    "GsVariant", "LsqSolver", "HOUSEHOLDER_QR", "QrFactors", "StabilityCertificate",
    "BreakdownError", "RgsState", "rgs_factorize", "certificates", "loss_of_orthogonality",
    "BREAKDOWN_FACTOR", "sketched_lsq",
]

BREAKDOWN_FACTOR = 10.0


class BreakdownError(RuntimeError):
    """Vanishing projection residual at a given (1-based) column index."""

    def __init__(self, column: int, r_ii: float, tol: float):
        super().__init__(f"breakdown at column {column}: r_ii={r_ii:.3e} <= tol={tol:.3e}")
        self.column = column
        self.r_ii = r_ii
        self.tol = tol


class GsVariant(Enum):
    CGS = "cgs"
    MGS = "mgs"
    CGS2 = "cgs2"
    RGS = "rgs"


@dataclass(frozen=True)
class LsqSolver:
    """Sketched least-squares solver selection (reference gram_schmidt.py:53-77).

    The device implements the direct QR-based solver, selected by the
    reference's name "householder" (``HOUSEHOLDER_QR``) so callers keep their
    arguments.  It is NOT a Householder chain: the reference appends
    reflectors one column at a time (``_IncrementalHouseholderQR``,
    gram_schmidt.py:122-190), a serial chain of i dependent reflections per
    solve.  The device factors the sketched basis S = T diag(alpha)^-1 R_S by
    classical Gram-Schmidt with selective reorthogonalisation (a second pass
    only when ||t||^2 < ||s||^2 / 2), keeps R_S^-1 explicitly and solves
    r = R_S^-1 Q_s^T p, split over a thread-block cluster (sgs_ls_step,
    DESIGN.md section 3).  Any backward-stable solver meets the RGS analysis
    (PAPER.md:455-459), and this one is for the well-conditioned S that RGS
    maintains; the rank test (gram_schmidt.py:186-189) runs on alpha and
    raises ``np.linalg.LinAlgError`` as the reference does.  ``sketched_lsq``
    exposes it on an arbitrary S.  The iterative alternatives ("richardson",
    "smgs") are outside the B200 hot path."""

    method: str = "householder"
    iterations: int = 4

    def __post_init__(self):
        if self.method not in ("householder", "richardson", "smgs"):
            raise ValueError(f"unknown least-squares method {self.method!r}")
        if self.method == "richardson" and self.iterations < 1:
            raise ValueError("richardson needs at least one iteration")


HOUSEHOLDER_QR = LsqSolver("householder")  # the device QR solver (see LsqSolver)


@dataclass
class QrFactors:
    """Q (n x m), upper-triangular R (m x m), sketches S = Theta Q, P = Theta W.

    numpy arrays by default; CUDA tensors when requested with ``device=True``."""

    Q: object
    R: object
    S: object = None
    P: object = None
    S_phi: object = None
    P_phi: object = None


class LazyFactors:
    """QrFactors view of a device state whose host copies are made on first
    access (the Krylov drivers return factors like the reference, but most
    callers never read them; copying an n x m basis back per cycle would
    dominate the solve)."""

    def __init__(self, state: "RgsState", m: int, device: bool = False):
        self._state, self._m, self._device = state, m, device
        self._cache = {}

    def _get(self, name):
        if name not in self._cache:
            st, m = self._state, self._m
            t = {"Q": lambda: st._Q[:m, :st.n_local].t(), "R": lambda: st._R[:m, :m].t(),
                 "S": lambda: st._S[:m].t(), "P": lambda: st._P[:m].t(),
                 "S_phi": lambda: st._S_phi[:m].t(), "P_phi": lambda: st._P_phi[:m].t()}[name]()
            self._cache[name] = t.clone() if self._device else t.cpu().numpy()
        return self._cache[name]

    Q = property(lambda self: self._get("Q"))
    R = property(lambda self: self._get("R"))
    S = property(lambda self: self._get("S"))
    P = property(lambda self: self._get("P"))
    S_phi = property(lambda self: self._get("S_phi") if self._state.phi is not None else None)
    P_phi = property(lambda self: self._get("P_phi") if self._state.phi is not None else None)


@dataclass
class StabilityCertificate:
    delta_m: float
    delta_tilde_m: float
    cond_S: float
    omega: float | None = None
    omega_bar: float | None = None
    omega_bar_w: float | None = None
    omega_bar_margin: float | None = None
    omega_bar_w_margin: float | None = None
    margin_precondition_ok: bool | None = None
    omega_bar_halved: float | None = None

    def passes_gate(self) -> bool:
        return self.delta_m <= 0.1 and self.delta_tilde_m <= 0.1

    def sigma_enclosure(self, eps: float, u_crs: float) -> tuple[float, float]:
        lo = (1.0 + eps) ** -0.5 * (1.0 - self.delta_m - 0.1 * u_crs)
        hi = (1.0 - eps) ** -0.5 * (1.0 + self.delta_m + 0.1 * u_crs)
        return lo, hi


def _round_up(x: int, a: int) -> int:
    return (x + a - 1) // a * a


class RgsState:
    """Device-resident streaming state of the randomized factorizer.

    ``push(w)`` runs one column and returns r_ii (it synchronises to do so, as
    the reference returns a float).  ``Q``, ``R``, ``S``, ``P`` return host
    copies trimmed to the committed columns; ``device_factors()`` returns the
    CUDA tensors.  Device layout: Q is column-major (column j contiguous,
    leading dimension a multiple of 32 rows), R column-major cap x cap fp64,
    S/P column-major k x cap in the fine dtype.

    ``comm`` (optional) row-shards the state: this rank holds rows
    [row0, row0 + n_local) of W and Q, the sketch partials of the shard are
    summed locally and combined with one all-reduce of the k-vector per
    sketch; the k-dimensional work is then replicated bit-identically on all
    ranks (no broadcast).
    """

    def __init__(self, theta, policy: PrecisionPolicy = MIXED32_64,
                 solver: LsqSolver = HOUSEHOLDER_QR, phi=None, capacity: int = 16,
                 breakdown_factor: float = BREAKDOWN_FACTOR, *, comm=None,
                 row0: int = 0, n_local: int | None = None):
        _lib.require_cuda()
        if solver.method != "householder":
            raise NotImplementedError("the device factorizer implements the direct "
                                      "QR least-squares solver only (HOUSEHOLDER_QR)")
        self.theta = as_device_sketch(theta)
        self.phi = as_device_sketch(phi) if phi is not None else None
        if self.phi is not None and self.phi.n != self.theta.n:
            raise ValueError("certification sketch has mismatched ambient dimension")
        self.policy = policy
        self.solver = solver
        self.breakdown_factor = float(breakdown_factor)
        self.comm = comm
        self.n = self.theta.n
        self.k = self.theta.k
        self.row0 = int(row0)
        self.n_local = self.n if n_local is None else int(n_local)
        if comm is None and (self.row0 != 0 or self.n_local != self.n):
            raise ValueError("row sharding needs a communicator")
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.cdt = _lib.torch_dtype(policy.coarse_dtype)
        self.fdt = _lib.torch_dtype(policy.fine_dtype)
        self.ccode = _lib.dtype_code(self.cdt)
        self.fcode = _lib.dtype_code(self.fdt)
        self.ldq = _round_up(self.n_local, 32)
        self.m = 0
        self.status = _lib.Status(self.device)
        self.nparts = self.theta.nparts(self.n_local)
        # fused update + sketch column kernel for SRHT kinds with 4096-row tiles
        self.fused = (not self.theta.is_dense and self.theta.log2_block >= 12
                      and self.row0 % 4096 == 0)
        if self.fused:
            self.nparts_q = int(_lib.load().sgs_column_nparts(self.n_local))
        elif self.theta.is_gaussian or (self.theta.is_dense and _RAD_FUSED):
            # the dense column kernel's own row chunks (Gaussian, fused Rademacher)
            self.nparts_q = int(_lib.load().sgs_dense_column_nparts(self.n_local, self.k))
        else:
            self.nparts_q = self.nparts
        self._cap = 0
        self._alloc(max(int(capacity), 2))
        self._parts_s = torch.empty((self.nparts_q, self.k), dtype=torch.float64,
                                    device=self.device)
        self._parts_p = torch.empty((self.nparts, self.k), dtype=torch.float64,
                                    device=self.device)
        if comm is not None:
            self._kvec_s = torch.empty(self.k, dtype=torch.float64, device=self.device)
            self._kvec_p = torch.empty_like(self._kvec_s)
        self._theta_dev = self.theta.device_data(self.device)
        if self.phi is not None:  # certification sketches (gram_schmidt.py:304-305, 333-335)
            self.phi.device_data(self.device)
            self.nparts_phi = self.phi.nparts(self.n_local)
            self._parts_phi = torch.empty((self.nparts_phi, self.phi.k), dtype=torch.float64,
                                          device=self.device)
            if comm is not None:
                self._kvec_phi = torch.empty(self.phi.k, dtype=torch.float64, device=self.device)
        # Phi q' in the fused column kernel's epilogue (same tile, no re-read of
        # q') when Phi is an SRHT kind with the column kernel's tile structure
        self.phi_fused = (self.phi is not None and self.fused and not self.phi.is_dense
                          and self.phi.log2_block >= 12 and _PHI_FUSED
                          and self.phi.nparts(self.n_local) == self.nparts_q)
        self._phi_col = None

    # ---- storage ----------------------------------------------------------------
    def _alloc(self, cap: int) -> None:
        dev, k = self.device, self.k
        old = None
        if self._cap:
            old = (self._Q, self._R, self._S, self._P, self._Qs, self._Rinv, self._alpha,
                   self._cap)
        # Q columns are written before they are read (q'_i by the column
        # kernel i, in place): only the pad rows past n_local need zeros, and
        # zeroing 2 GB at c1 cost 0.3 ms of every end-to-end call.
        # SGS_DEBUG_POISON=1 fills Q with NaN instead (tests prove the claim).
        if _POISON:
            self._Q = torch.full((cap, self.ldq), float("nan"), dtype=self.cdt, device=dev)
        else:
            self._Q = torch.empty((cap, self.ldq), dtype=self.cdt, device=dev)
        if self.ldq > self.n_local:
            self._Q[:, self.n_local:].zero_()
        self._R = torch.zeros((cap, cap), dtype=torch.float64, device=dev)
        self._S = torch.zeros((cap, k), dtype=self.fdt, device=dev)
        self._P = torch.zeros((cap, k), dtype=self.fdt, device=dev)
        self._Qs = torch.zeros((cap, k), dtype=self.fdt, device=dev)
        self._Rinv = torch.zeros((cap, cap), dtype=self.fdt, device=dev)
        self._alpha = torch.zeros(cap, dtype=self.fdt, device=dev)
        if self.phi is not None:
            kp = self.phi.k
            old_phi = (self._S_phi, self._P_phi) if self._cap else None
            self._S_phi = torch.zeros((cap, kp), dtype=self.fdt, device=dev)
            self._P_phi = torch.zeros((cap, kp), dtype=self.fdt, device=dev)
            if old_phi is not None:
                self._S_phi[:self._cap] = old_phi[0]
                self._P_phi[:self._cap] = old_phi[1]
        self._scratch = torch.zeros(int(_lib.load().sgs_ls_scratch_elems(k, cap)),
                                    dtype=torch.float64, device=dev)
        # deferred formation of the newest T column (sgs_ls_args.t_pend / t_coef)
        old_coef = self.__dict__.get("_tcoef")
        self._tcoef = torch.zeros(cap + k, dtype=self.fdt, device=dev)  # [c1 (cap) | s' (k)]
        if old_coef is not None:
            oc_ = old_coef.shape[0] - k
            self._tcoef[:oc_] = old_coef[:oc_]
            self._tcoef[cap:] = old_coef[oc_:]
        if "_tpend" not in self.__dict__:
            self._tpend = torch.full((2,), -1, dtype=torch.int32, device=dev)
        self._rc = torch.zeros(cap, dtype=self.cdt, device=dev)
        if old is not None:
            Q, R, S, P, Qs, Rinv, alpha, oc = old
            self._Q[:oc] = Q
            self._R[:oc, :oc] = R
            self._S[:oc] = S
            self._P[:oc] = P
            self._Qs[:oc] = Qs
            self._Rinv[:oc, :oc] = Rinv
            self._alpha[:oc] = alpha
        self._cap = cap

    def _grow(self) -> None:
        if self.m + 1 >= self._cap:
            self._alloc(2 * self._cap)

    # ---- kernels ---------------------------------------------------------------
    def _ls(self, *, fin: int | None = None, s_parts=None, s_nparts=0, s_scale=1.0,
            sol: int | None = None, p_parts=None, p_nparts=0, p_scale=1.0,
            lag: bool = False, giv=None, peer: bool = False) -> None:
        a = self.__dict__.get("_ls_args")
        if a is None:
            a = self._ls_args = _lib.LsArgs()  # reused: the library copies it at launch
        a.k, a.cap, a.fine_dtype, a.coarse_dtype = self.k, self._cap, self.fcode, self.ccode
        a.do_finalize = 1 if fin is not None else 0
        a.col_fin = fin if fin is not None else 0
        a.s_partials = s_parts
        a.s_nparts = s_nparts
        a.s_scale = s_scale
        a.do_solve = 1 if sol is not None else 0
        a.col_sol = sol if sol is not None else 0
        a.p_partials = p_parts
        a.p_nparts = p_nparts
        a.p_scale = p_scale
        a.p_lag = 1 if lag else 0
        if giv is None:
            a.giv_on = 0
        else:  # (cs, sn, g, T, hist, tol) device tensors of the GMRES driver
            cs, sn, g, T, hist, tol = giv
            a.giv_on = 1
            a.giv_cs, a.giv_sn, a.giv_g = cs.data_ptr(), sn.data_ptr(), g.data_ptr()
            a.giv_T, a.giv_ldt, a.giv_hist = T.data_ptr(), T.shape[1], hist.data_ptr()
            a.giv_tol = -1.0 if tol is None else float(tol)
        a.peer = self._peer.desc if peer else None  # s' summed across ranks in the LS launch
        a.bf_ucrs = self.breakdown_factor * self.policy.u_crs
        a.S, a.P, a.R = self._S.data_ptr(), self._P.data_ptr(), self._R.data_ptr()
        a.Qs, a.Rinv, a.alpha = self._Qs.data_ptr(), self._Rinv.data_ptr(), self._alpha.data_ptr()
        a.scratch, a.r_crs, a.st = self._scratch.data_ptr(), self._rc.data_ptr(), self.status.ptr
        a.trace = self._trace_ptr(fin if fin is not None else sol)
        # The fast path publishes r from Pythagorean identities (||t||^2 =
        # ||s||^2 - sum c1^2, t^T p = s^T p - sum c1_j z_j).  In fp64 they are
        # as accurate as the explicit dots (c1-shaped mixed emulation: the
        # same metrics to 1e-16), but with an fp32 LS (UNIFIED32) the t^T p
        # identity cancels catastrophically once W is numerically rank
        # deficient (numpy emulation of the acceptance problem: cond(Q) 2.5e7
        # against 47 with explicit dots and 23 for the reference's Householder).
        if _LS_DEFER and self.fdt != torch.float32:
            a.t_pend, a.t_coef = self._tpend.data_ptr(), self._tcoef.data_ptr()
        else:
            a.t_pend = a.t_coef = None
        _lib.check(_lib.load().sgs_ls_step(ctypes_byref(a), stream_ptr()), "sgs_ls_step")

    _trace = None  # optional (cap, 16) int64 device tensor: per-column LS phase clocks
    _e2e_late = (192, 64)  # pipelined path: (column from which chunks grow, late chunk cap)
    _e2e_ship = 8          # pipelined path: Q columns per D2H copy
    _e2e_tail = 32         # pipelined path: last columns shipped two at a time
    _e2e_side = os.environ.get("SGS_E2E_SIDE", "1") != "0"  # pipelined path: side-stream sketches
    _e2e_ship_far = 32     # side-stream path: Q columns per copy between chunk boundaries
    _e2e_ahead = 4         # pipelined path: W chunks enqueued ahead of the column loop
    # side-stream path: no Q copies before this column - both directions at
    # once run at ~48 GB/s each against ~55 GB/s for H2D alone, and the early
    # columns are bound by W's arrival
    _e2e_ship_from = 192

    def _trace_ptr(self, col):
        t = self._trace
        if t is None or col is None or col >= t.shape[0]:
            return None
        return t.data_ptr() + col * t.shape[1] * 8

    def _combine(self, out: torch.Tensor, nparts: int, kvec: torch.Tensor | None):
        """(pointer, nparts, scale) of a sketch for sgs_ls_step; sharded states
        first sum the local partials and all-reduce the k-vector."""
        if self.comm is None:
            return out.data_ptr(), nparts, self.theta.scale
        call("sgs_partials_reduce", out.data_ptr(), nparts, self.k, 1, 1.0,
             kvec.data_ptr(), _lib.SGS_F64, self.k, self.status.ptr, stream_ptr())
        self.comm.allreduce_(kvec)
        return kvec.data_ptr(), 1, self.theta.scale

    def _sketch_parts(self, x_ptr: int, x_code: int, ldx: int, out: torch.Tensor,
                      kvec: torch.Tensor | None, small_grid: bool = False):
        """Partials of one local column via the stand-alone sketch kernel."""
        kw = {"small_grid": True} if small_grid and not self.theta.is_dense else {}
        self.theta.partials_into(x_ptr, x_code, ldx, 1, out, n_local=self.n_local,
                                 row0=self.row0, status=self.status, **kw)
        return self._combine(out, self.nparts, kvec)

    def _peer_ok(self) -> bool:
        """The in-LS peer exchange of s' serves row-sharded fused SRHT states on
        an NCCL group (one node) with an fp64 LS (SGS_PEER=0 keeps the
        per-column NCCL all-reduce)."""
        c = self.comm
        return (_PEER and c is not None and getattr(c, "backend", None) == "nccl"
                and getattr(c, "world", 1) <= 8 and self.fused and not self.phi_fused
                and self.fdt == torch.float64)

    def _peer_begin(self) -> bool:
        """Set up (first call, collective) and open the peer exchange for one
        factorisation; False when it does not apply or is unavailable on some
        rank (then every rank uses the NCCL all-reduce)."""
        if not self._peer_ok():
            return False
        if "_peer" not in self.__dict__:
            from .distributed import PeerExchange
            self._peer = PeerExchange.get(self.comm, self.k,
                                          int(_lib.load().sgs_ls_cluster_size(self.k)))
        if self._peer is None:
            return False
        self._peer.begin(stream_ptr())
        return True

    def _update(self, i: int, w_ptr: int, w_code: int, normalize_prev: bool) -> None:
        call("sgs_rgs_update", self._Q.data_ptr(), self.ccode, self.ldq, self.n_local, i,
             w_ptr, w_code, self._rc.data_ptr(), 1 if normalize_prev else 0,
             self._R.data_ptr(), self._cap, self.status.ptr, stream_ptr())

    def _column(self, i: int, w_ptr: int, w_code: int, normalize_prev: bool, sketch: bool,
                w_div: int | None = None, combine: bool = True):
        """Step 3 (and step 4 when ``sketch``): q'_i = w - Q r into Q[:, i] and the
        partial sketches of q'_i.  Returns (pointer, nparts, scale) or None.
        ``w_div`` (device fp64 scalar, fused SRHT path only): the column is
        cast(w / w_div).  ``combine=False`` leaves the partials unsummed (the
        caller combines them, e.g. with another sketch in one all-reduce)."""
        kvec = getattr(self, "_kvec_s", None)
        if w_div is not None and not self.fused:
            raise ValueError("w_div needs the fused SRHT column kernel")
        if self.fused:
            d = self._theta_dev
            if sketch and self.phi_fused:  # Phi q'_i from the same epilogue
                pd = self.phi.device_data(self.device)
                call("sgs_rgs_update_srht_phi", self._Q.data_ptr(), self.ccode, self.ldq,
                     self.n_local, i, w_ptr, w_code, w_div, self._rc.data_ptr(),
                     1 if normalize_prev else 0, self._R.data_ptr(), self._cap, 1, self.row0,
                     self.theta.log2_block, d["bits"].data_ptr() + (self.row0 // 32) * 4,
                     d["samples"].data_ptr(), self.k, self._parts_s.data_ptr(),
                     pd["bits"].data_ptr() + (self.row0 // 32) * 4, pd["samples"].data_ptr(),
                     self.phi.k, self.phi.log2_block, self._parts_phi.data_ptr(),
                     self.status.ptr, stream_ptr())
                self._phi_col = i
            else:
                call("sgs_rgs_update_srht", self._Q.data_ptr(), self.ccode, self.ldq,
                     self.n_local, i, w_ptr, w_code, w_div, self._rc.data_ptr(),
                     1 if normalize_prev else 0, self._R.data_ptr(), self._cap,
                     1 if sketch else 0, self.row0, self.theta.log2_block,
                     d["bits"].data_ptr() + (self.row0 // 32) * 4, d["samples"].data_ptr(),
                     self.k, self._parts_s.data_ptr(), self.status.ptr, stream_ptr())
            if not sketch:
                return None
            if not combine:
                return self._parts_s.data_ptr(), self.nparts_q, self.theta.scale
            return self._combine(self._parts_s, self.nparts_q, kvec)
        if self.theta.is_gaussian:
            d = self._theta_dev
            call("sgs_rgs_update_dense", self._Q.data_ptr(), self.ccode, self.ldq, self.n_local,
                 i, w_ptr, w_code, self._rc.data_ptr(), 1 if normalize_prev else 0,
                 self._R.data_ptr(), self._cap, 1 if sketch else 0,
                 d["thetaT"].data_ptr() + self.row0 * d["ldt"] * 8, d["ldt"], self.k,
                 self._parts_s.data_ptr(), self.status.ptr, stream_ptr())
            if not sketch:
                return None
            if not combine:
                return self._parts_s.data_ptr(), self.nparts_q, self.theta.scale
            return self._combine(self._parts_s, self.nparts_q, kvec)
        if self.theta.kind is SketchKind.RADEMACHER and _RAD_FUSED:
            # fused: q' streamed once, Theta q' from the packed device signs
            d = self._theta_dev
            call("sgs_rgs_update_rademacher", self._Q.data_ptr(), self.ccode, self.ldq,
                 self.n_local, i, w_ptr, w_code, self._rc.data_ptr(), 1 if normalize_prev else 0,
                 self._R.data_ptr(), self._cap, 1 if sketch else 0,
                 d["rbits"].data_ptr() + self.row0 * d["kw"] * 4, self.k,
                 self._parts_s.data_ptr(), self.status.ptr, stream_ptr())
            if not sketch:
                return None
            if not combine:
                return self._parts_s.data_ptr(), self.nparts_q, self.theta.scale
            return self._combine(self._parts_s, self.nparts_q, kvec)
        self._update(i, w_ptr, w_code, normalize_prev)
        if not sketch:
            return None
        if not combine:
            self.theta.partials_into(self._qcol_ptr(i), self.ccode, self.ldq, 1, self._parts_s,
                                     n_local=self.n_local, row0=self.row0, status=self.status)
            return self._parts_s.data_ptr(), self.nparts, self.theta.scale
        return self._sketch_parts(self._qcol_ptr(i), self.ccode, self.ldq, self._parts_s, kvec)

    # ---- certification sketches ------------------------------------------------------
    def _phi_parts(self, x_ptr: int, x_code: int, ldx: int, ncols: int = 1,
                   launched: bool = False):
        """Partials of Phi x over the local rows (summed across ranks when
        sharded).  ``launched``: the column kernel already wrote them."""
        ph = self.phi
        if not launched:
            self.phi.partials_into(x_ptr, x_code, ldx, ncols, self._parts_phi,
                                   n_local=self.n_local, row0=self.row0, status=self.status)
        if self.comm is None:
            return self._parts_phi.data_ptr(), self.nparts_phi
        call("sgs_partials_reduce", self._parts_phi.data_ptr(), self.nparts_phi, ph.k, 1, 1.0,
             self._kvec_phi.data_ptr(), _lib.SGS_F64, ph.k, self.status.ptr, stream_ptr())
        self.comm.allreduce_(self._kvec_phi)
        return self._kvec_phi.data_ptr(), 1

    def _phi_w(self, i: int, w_ptr: int, w_code: int, ldw: int) -> None:
        """P_phi[:, i] = Phi w_i (gram_schmidt.py:304-305)."""
        if self.phi is None:
            return
        pp, pn = self._phi_parts(w_ptr, w_code, ldw)
        call("sgs_partials_reduce", pp, pn, self.phi.k, 1, self.phi.scale,
             self._P_phi.data_ptr() + i * self.phi.k * self._P_phi.element_size(), self.fcode,
             self.phi.k, self.status.ptr, stream_ptr())

    def _phi_q_parts(self, i: int):
        """Partials of Phi q'_i while Q[:, i] still holds the unnormalised q'."""
        if self.phi is None:
            return None
        fused_here, self._phi_col = self._phi_col == i, None
        return self._phi_parts(self._qcol_ptr(i), self.ccode, self.ldq, launched=fused_here)

    def _phi_q_finish(self, i: int, parts) -> None:
        """S_phi[:, i] = (Phi q'_i) / r_ii (gram_schmidt.py:333-335)."""
        if self.phi is None:
            return
        pp, pn = parts
        call("sgs_partials_reduce_div", pp, pn, self.phi.k, 1, self.phi.scale,
             self._R.data_ptr() + (i * self._cap + i) * 8,
             self._S_phi.data_ptr() + i * self.phi.k * self._S_phi.element_size(), self.fcode,
             self.phi.k, self.status.ptr, stream_ptr())

    def _normalize(self, col: int, guarded: bool = True) -> None:
        call("sgs_normalize_column", self._Q.data_ptr(), self.ccode, self.ldq, self.n_local,
             col, self._R.data_ptr(), self._cap, self.status.ptr if guarded else None,
             stream_ptr())

    def _qcol_ptr(self, j: int) -> int:
        return self._Q.data_ptr() + j * self.ldq * self._Q.element_size()

    def _raise_status(self, st: dict) -> None:
        code = st["code"]
        if code == _lib.ST_BREAKDOWN:
            raise BreakdownError(st["column"], st["r_ii"], st["tol"])
        if code == _lib.ST_RANK:
            raise np.linalg.LinAlgError("sketched basis numerically rank deficient")
        if code == _lib.ST_TIMEOUT:
            raise RuntimeError("the LS step timed out waiting for another rank's sketch "
                               "(peer exchange; SGS_PEER=0 uses NCCL all-reduces)")

    # ---- streaming API -----------------------------------------------------------
    def _as_device_column(self, w) -> torch.Tensor:
        if isinstance(w, torch.Tensor) and w.is_cuda:
            t = w
            if t.dtype not in (torch.float32, torch.float64):
                t = t.to(torch.float64)
        else:
            t = torch.from_numpy(np.ascontiguousarray(np.asarray(w, dtype=np.float64)))
            t = t.to(self.device)
        if tuple(t.shape) != (self.n_local,):
            raise ValueError("column length mismatch")
        return t.contiguous()

    def _push_async(self, w: torch.Tensor) -> None:
        """Enqueue one column (column-at-a-time path, no host sync)."""
        self._grow()
        i = self.m
        wc = _lib.dtype_code(w.dtype)
        pp, pn, ps = self._sketch_parts(w.data_ptr(), wc, self.n_local, self._parts_p,
                                        getattr(self, "_kvec_p", None))
        self._phi_w(i, w.data_ptr(), wc, self.n_local)
        if i == 0:
            call("sgs_partials_reduce", pp, pn, self.k, 1, ps, self._P.data_ptr(), self.fcode,
                 self.k, self.status.ptr, stream_ptr())
            self._column(0, w.data_ptr(), wc, False, False)
            phq = self._phi_q_parts(0)
            self._ls(fin=0)
        else:
            self._ls(sol=i, p_parts=pp, p_nparts=pn, p_scale=ps)
            sp, sn, ss = self._column(i, w.data_ptr(), wc, False, True)
            phq = self._phi_q_parts(i)
            self._ls(fin=i, s_parts=sp, s_nparts=sn, s_scale=ss)
        self._phi_q_finish(i, phq)
        self._normalize(i)
        self.m += 1  # provisional; reconciled with the device count at sync

    def _sync_status(self) -> dict:
        st = self.status.read()
        self.m = st["ncols"]
        return st

    def push(self, w) -> float:
        """Run one iteration on the next column; returns the diagonal r_ii."""
        st = self.status.read()
        if st["code"]:
            self.status.clear_code()
        t = self._as_device_column(w)
        self._push_async(t)
        st = self._sync_status()
        if st["code"]:
            self.status.clear_code()
            self._raise_status(st)
        return st["r_ii"]

    # ---- views -------------------------------------------------------------------
    def device_factors(self) -> QrFactors:
        m = self.m
        f = QrFactors(Q=self._Q[:m, :self.n_local].t(), R=self._R[:m, :m].t(),
                      S=self._S[:m].t(), P=self._P[:m].t())
        if self.phi is not None:
            f.S_phi, f.P_phi = self._S_phi[:m].t(), self._P_phi[:m].t()
        return f

    @property
    def Q(self):
        return self._Q[:self.m, :self.n_local].t().cpu().numpy()

    @property
    def R(self):
        return self._R[:self.m, :self.m].t().cpu().numpy()

    @property
    def S(self):
        return self._S[:self.m].t().cpu().numpy()

    @property
    def P(self):
        return self._P[:self.m].t().cpu().numpy()

    def factors(self, device: bool = False) -> QrFactors:
        if device:
            f = self.device_factors()
            out = QrFactors(Q=f.Q.clone(), R=f.R.clone(), S=f.S.clone(), P=f.P.clone())
            if self.phi is not None:
                out.S_phi, out.P_phi = f.S_phi.clone(), f.P_phi.clone()
            return out
        out = QrFactors(Q=self.Q, R=self.R, S=self.S, P=self.P)
        if self.phi is not None:
            out.S_phi = self._S_phi[:self.m].t().cpu().numpy()
            out.P_phi = self._P_phi[:self.m].t().cpu().numpy()
        return out

    # ---- batch path ----------------------------------------------------------------
    def _reserve(self, ncols: int) -> None:
        while self._cap < ncols:
            self._alloc(2 * self._cap)

    def _enqueue_factorization(self, Wcm: torch.Tensor, ldw: int, m: int) -> None:
        """Enqueue a complete factorisation of m columns of a device
        column-major W (column j at offset j*ldw) on the current stream: status
        reset, batched P = Theta W, then per column the fused column kernel and
        one LS launch (finalize i + solve i+1).  No host synchronisation, so the
        sequence can be captured in a CUDA graph."""
        self.status.reset()
        wc = _lib.dtype_code(Wcm.dtype)
        esz = Wcm.element_size()
        base = Wcm.data_ptr()
        k, sp = self.k, stream_ptr()
        # P = Theta W, batched in column chunks (same kernel and parts as per column)
        # the chunk size sets the all-reduce message size, so a sharded state
        # sizes it from the global row count (identical on every rank)
        np_size = self.nparts if self.comm is None else max(self.nparts, self.theta.nparts(self.n))
        # P_phi = Phi W in the same pass when Phi has Theta's tile structure
        pair = self.phi_fused and not _lib.srht_legacy()
        kk = k + (self.phi.k if pair else 0)
        chunk = max(1, min(m, (256 << 20) // max(1, np_size * kk * 8)))
        parts = torch.empty((chunk, self.nparts, k), dtype=torch.float64, device=self.device)
        if pair:
            ph, kp_ = self.phi, self.phi.k
            pparts = torch.empty((chunk, self.nparts_phi, kp_), dtype=torch.float64,
                                 device=self.device)
            d, pd = self._theta_dev, ph.device_data(self.device)
            if self.comm is not None:
                kbp = torch.empty((chunk, kp_), dtype=torch.float64, device=self.device)
            self._keep_phi = pparts
        if self.comm is not None:
            kbuf = torch.empty((chunk, k), dtype=torch.float64, device=self.device)
        for c0 in range(0, m, chunk):
            nc = min(chunk, m - c0)
            if pair:
                call("sgs_srht_partials_pair", base + c0 * ldw * esz, wc, ldw, nc, self.n_local,
                     self.row0, self.theta.log2_block, d["bits"].data_ptr() + (self.row0 // 32) * 4,
                     d["samples"].data_ptr(), k, parts.data_ptr(), ph.log2_block,
                     pd["bits"].data_ptr() + (self.row0 // 32) * 4, pd["samples"].data_ptr(), kp_,
                     pparts.data_ptr(), self.status.ptr, sp)
                pdst = self._P_phi.data_ptr() + c0 * kp_ * self._P_phi.element_size()
                if self.comm is None:
                    call("sgs_partials_reduce", pparts.data_ptr(), self.nparts_phi, kp_, nc,
                         ph.scale, pdst, self.fcode, kp_, self.status.ptr, sp)
                else:
                    call("sgs_partials_reduce", pparts.data_ptr(), self.nparts_phi, kp_, nc, 1.0,
                         kbp.data_ptr(), _lib.SGS_F64, kp_, self.status.ptr, sp)
                    self.comm.allreduce_(kbp[:nc])
                    call("sgs_partials_reduce", kbp.data_ptr(), 1, kp_, nc, ph.scale, pdst,
                         self.fcode, kp_, self.status.ptr, sp)
            else:
                self.theta.partials_into(base + c0 * ldw * esz, wc, ldw, nc, parts,
                                         n_local=self.n_local, row0=self.row0,
                                         status=self.status)
            pdst = self._P.data_ptr() + c0 * k * self._P.element_size()
            if self.comm is None:
                call("sgs_partials_reduce", parts.data_ptr(), self.nparts, k, nc,
                     self.theta.scale, pdst, self.fcode, k, self.status.ptr, sp)
            else:
                call("sgs_partials_reduce", parts.data_ptr(), self.nparts, k, nc, 1.0,
                     kbuf.data_ptr(), _lib.SGS_F64, k, self.status.ptr, sp)
                self.comm.allreduce_(kbuf[:nc])
                call("sgs_partials_reduce", kbuf.data_ptr(), 1, k, nc, self.theta.scale,
                     pdst, self.fcode, k, self.status.ptr, sp)
        if self.phi is not None and not pair:  # P_phi = Phi W, batched (same bits as per column)
            ph, kp_ = self.phi, self.phi.k
            np_phi = (self.nparts_phi if self.comm is None
                      else max(self.nparts_phi, ph.nparts(self.n)))
            chp = max(1, min(m, (128 << 20) // max(1, np_phi * kp_ * 8)))
            pparts = torch.empty((chp, self.nparts_phi, kp_), dtype=torch.float64,
                                 device=self.device)
            if self.comm is not None:
                kbp = torch.empty((chp, kp_), dtype=torch.float64, device=self.device)
            for c0 in range(0, m, chp):
                nc = min(chp, m - c0)
                ph.partials_into(base + c0 * ldw * esz, wc, ldw, nc, pparts,
                                 n_local=self.n_local, row0=self.row0, status=self.status)
                pdst = self._P_phi.data_ptr() + c0 * kp_ * self._P_phi.element_size()
                if self.comm is None:
                    call("sgs_partials_reduce", pparts.data_ptr(), self.nparts_phi, kp_, nc,
                         ph.scale, pdst, self.fcode, kp_, self.status.ptr, sp)
                else:
                    call("sgs_partials_reduce", pparts.data_ptr(), self.nparts_phi, kp_, nc, 1.0,
                         kbp.data_ptr(), _lib.SGS_F64, kp_, self.status.ptr, sp)
                    self.comm.allreduce_(kbp[:nc])
                    call("sgs_partials_reduce", kbp.data_ptr(), 1, kp_, nc, ph.scale, pdst,
                         self.fcode, kp_, self.status.ptr, sp)
            self._keep_phi = pparts
        # row-sharded over NCCL: the LS launch sums s' across the ranks by
        # NVLink stores into the peers' exchange areas (no all-reduce per column)
        peer = self._peer_begin()
        for i in range(m):
            sol = i + 1 if i + 1 < m else None
            if i == 0:
                self._column(0, base, wc, False, False)
                phq = self._phi_q_parts(0)
                self._ls(fin=0, sol=sol)
            else:
                spp, snp, ssc = self._column(i, base + i * ldw * esz, wc, True, True,
                                             combine=not peer)
                phq = self._phi_q_parts(i)
                self._ls(fin=i, s_parts=spp, s_nparts=snp, s_scale=ssc, sol=sol, peer=peer)
            self._phi_q_finish(i, phq)
        self._normalize(m - 1)
        self._keep = parts  # keep the chunk buffer alive for graph replays

    def factorize_columns(self, Wcm: torch.Tensor, ldw: int, m: int) -> None:
        """Factorise m columns of a device column-major W with two launches per
        column; raises at the end on a device-recorded breakdown / rank
        deficiency (reference exception types and column numbers)."""
        if self.m != 0:
            raise RuntimeError("factorize_columns needs a fresh state")
        self._reserve(m + 1)
        self._enqueue_factorization(Wcm, ldw, m)
        self.finish()

    def finish(self) -> None:
        """Synchronise with the device status and raise what it recorded."""
        st = self._sync_status()
        if st["code"]:
            self._raise_status(st)

    def factorize_host_pipelined(self, Wh: np.ndarray, m: int, chunk: int = 8) -> QrFactors:
        """End-to-end factorisation of a pinned, column-major host W (n x m,
        Fortran order): W streams to the GPU in column chunks on one copy
        stream, a side stream sketches each chunk as it lands (P = Theta W),
        and the compute stream runs the column loop, waiting on a chunk's
        sketch only before the LS launch that first reads it; finished Q
        columns stream back to a pinned host buffer on a second copy stream.
        Returns host factors (Q is a view of pinned memory).  Schedule knobs:
        the ``_e2e_*`` class attributes."""
        if self.m != 0:
            raise RuntimeError("factorize_host_pipelined needs a fresh state")
        n, k = self.n_local, self.k
        self._reserve(m + 1)
        dt = _lib.torch_dtype(Wh.dtype)
        Wt = torch.from_numpy(Wh.T)  # (m, n) view of the pinned buffer
        Wd = torch.empty((m, n), dtype=dt, device=self.device)
        comp = torch.cuda.current_stream()
        h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
        h2d.wait_stream(comp)
        # graduated chunks (2, 4, 8, ... up to `chunk` columns) so the column
        # loop starts after a few MB have landed instead of a full chunk
        # Early columns outrun PCIe (~50 GB/s) and need fine arrival steps; past
        # `late` the GPU is the bottleneck and larger chunks mean fewer
        # cross-stream waits in the kernel chain.
        late, late_chunk = self._e2e_late
        bounds, c0, sz = [0], 0, 2
        if self.theta.is_gaussian:
            # the dense P = Theta W GEMM reads all of Theta and fills 64-column
            # tiles per launch: sketch whole tiles (a chunk of 8 columns would
            # cost as much as 64)
            bounds = list(range(0, m, 64)) + [m]
            c0 = m
        while c0 < m:  # 2, 4, ..., chunk; past `late` doubling again up to late_chunk
            step = min(sz, chunk if c0 < late else late_chunk)
            c0 = min(m, c0 + step)
            bounds.append(c0)
            sz = 2 * step
        nchunks = len(bounds) - 1
        chunk_of = np.zeros(m + 1, dtype=np.int64)
        for c in range(nchunks):
            chunk_of[bounds[c]:bounds[c + 1]] = c
        # Copies and side-stream sketches are enqueued a few chunks ahead of
        # the column loop rather than all up front: ~40 host calls each would
        # hold back column 0 by ~1.3 ms of host time, while the host stays well
        # ahead of the device once the loop runs.
        landed = []

        def copy_until(c_end):
            with torch.cuda.stream(h2d):
                while len(landed) < min(nchunks, c_end):
                    c0, c1 = bounds[len(landed)], bounds[len(landed) + 1]
                    Wd[c0:c1].copy_(Wt[c0:c1], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(h2d)
                    landed.append(ev)

        copy_until(self._e2e_ahead)
        Qh, Qarr = _pinned_buffer((m, n), self.cdt)
        wc, esz, base = _lib.dtype_code(dt), Wd.element_size(), Wd.data_ptr()
        pmax = max(chunk, self._e2e_late[1])
        parts = torch.empty((pmax, self.nparts, k), dtype=torch.float64, device=self.device)
        self.status.reset()

        kbuf = (torch.empty((pmax, k), dtype=torch.float64, device=self.device)
                if self.comm is not None else None)

        # Unsharded states sketch each chunk on a side stream as soon as it
        # lands, so the compute stream only waits on an event (one broken PDL
        # edge, before the LS that first reads the chunk's P columns) instead
        # of running the sketch between an LS and the next column kernel.
        side = self.comm is None and self._e2e_side
        sk = torch.cuda.Stream() if side else None
        sketched = []

        def sketch_chunk(c):
            copy_until(c + self._e2e_ahead)
            torch.cuda.current_stream().wait_event(landed[c])
            c0, c1 = bounds[c], bounds[c + 1]
            self.theta.partials_into(base + c0 * n * esz, wc, n, c1 - c0, parts,
                                     n_local=n, row0=self.row0, status=self.status)
            pdst = self._P.data_ptr() + c0 * k * self._P.element_size()
            if self.comm is None:
                call("sgs_partials_reduce", parts.data_ptr(), self.nparts, k, c1 - c0,
                     self.theta.scale, pdst, self.fcode, k, self.status.ptr, stream_ptr())
            else:  # same order as _enqueue_factorization: local sum, all-reduce, scale
                call("sgs_partials_reduce", parts.data_ptr(), self.nparts, k, c1 - c0, 1.0,
                     kbuf.data_ptr(), _lib.SGS_F64, k, self.status.ptr, stream_ptr())
                self.comm.allreduce_(kbuf[:c1 - c0])
                call("sgs_partials_reduce", kbuf.data_ptr(), 1, k, c1 - c0, self.theta.scale,
                     pdst, self.fcode, k, self.status.ptr, stream_ptr())

        def ship(c0, c1):
            ev = torch.cuda.Event()
            ev.record(comp)
            d2h.wait_event(ev)
            with torch.cuda.stream(d2h):
                Qh[c0:c1].copy_(self._Q[c0:c1, :n], non_blocking=True)

        Ph, Parr = _pinned_buffer((m, k), self.fdt)

        def ship_p():  # P is final once the last chunk is sketched
            ev = torch.cuda.Event()
            ev.record(sk if side else comp)
            d2h.wait_event(ev)
            with torch.cuda.stream(d2h):
                Ph.copy_(self._P[:m], non_blocking=True)

        peer = self._peer_begin()  # s' summed across ranks in the LS launch (as the device path)
        def sketch_until(c_end):
            with torch.cuda.stream(sk):
                while len(sketched) < min(nchunks, c_end):
                    sketch_chunk(len(sketched))
                    ev = torch.cuda.Event()
                    ev.record(sk)
                    sketched.append(ev)
                    if len(sketched) == nchunks:
                        ship_p()

        if side:
            sk.wait_stream(comp)  # status reset and state set-up
            sketch_until(2)
        else:
            sketch_chunk(0)
            if nchunks == 1:
                ship_p()
        shipped, ship_chunk = 0, self._e2e_ship
        for i in range(m):
            nxt = i + 1
            new_chunk = nxt < m and bounds[chunk_of[nxt]] == nxt
            if i == 0 and side:
                comp.wait_event(sketched[0])
            if new_chunk and not side:
                sketch_chunk(int(chunk_of[nxt]))
                if int(chunk_of[nxt]) == nchunks - 1:
                    ship_p()
            sol = nxt if nxt < m else None
            if i == 0:
                self._column(0, base, wc, False, False)
                if new_chunk and side:
                    sketch_until(int(chunk_of[nxt]) + 2)
                    comp.wait_event(sketched[int(chunk_of[nxt])])
                self._ls(fin=0, sol=sol)
            else:
                spp, snp, ssc = self._column(i, base + i * n * esz, wc, True, True,
                                             combine=not peer)
                # columns < i are final once the column kernel i has normalised
                # i-1; finer copies over the last columns keep the tail short.
                # On the side-stream path the copies start where the chunk wait
                # already breaks the PDL chain (an event record breaks it too).
                step = ship_chunk if i < m - self._e2e_tail else min(ship_chunk, 2)
                if side:
                    if new_chunk:
                        sketch_until(int(chunk_of[nxt]) + 2)
                        comp.wait_event(sketched[int(chunk_of[nxt])])
                    if i >= self._e2e_ship_from and i - shipped >= (
                            step if new_chunk or i >= m - self._e2e_tail else self._e2e_ship_far):
                        ship(shipped, i)
                        shipped = i
                self._ls(fin=i, s_parts=spp, s_nparts=snp, s_scale=ssc, sol=sol, peer=peer)
                if not side and i - shipped >= step:
                    ship(shipped, shipped + step)
                    shipped += step
        self._normalize(m - 1)
        # the tail: last Q columns and R, S into pinned buffers on the copy
        # stream (pageable .cpu() copies of R/S/P cost ~3.5 ms at c1)
        Rh, Rarr = _pinned_buffer((m, m), torch.float64)
        Sh, Sarr = _pinned_buffer((m, k), self.fdt)
        ev = torch.cuda.Event()
        ev.record(comp)
        d2h.wait_event(ev)
        with torch.cuda.stream(d2h):
            if shipped < m:
                Qh[shipped:m].copy_(self._Q[shipped:m, :n], non_blocking=True)
            Rh.copy_(self._R[:m, :m], non_blocking=True)
            Sh.copy_(self._S[:m], non_blocking=True)
        comp.wait_stream(d2h)
        if side:
            comp.wait_stream(sk)
        st = self._sync_status()
        if st["code"]:
            self._raise_status(st)
        return QrFactors(Q=Qarr.T, R=Rarr.T, S=Sarr.T, P=Parr.T)

    def capture_factorization(self, Wcm: torch.Tensor, ldw: int, m: int):
        """Capture the whole factorisation in a CUDA graph; ``graph.replay()``
        re-runs every kernel (status reset included) and ``finish()`` reads the
        outcome.  Used for repeated factorisations of same-shaped inputs."""
        self._reserve(m + 1)
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        # a sharded state captures its collectives too (NCCL all-reduces are
        # stream-ordered and capturable once the communicator is up; the
        # process group's watchdog thread keeps querying its events, hence a
        # thread-local capture mode)
        mode = "global" if self.comm is None else "thread_local"
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side, capture_error_mode=mode):
                self._enqueue_factorization(Wcm, ldw, m)
        torch.cuda.current_stream().wait_stream(side)
        return g


_PINNED_POOL: list = []


# SGS_RAD_FUSED=1: Rademacher states use the fused column kernel
# (sgs_rgs_update_rademacher: one pass, q' never re-read).  Off by default: at
# c0r's shapes it measured 9957 columns/s against 12047 for the generic update
# + packed-sign sketch pair - the +-1 GEMV is compute-bound (k n signed adds
# per column) and runs after the Q stream inside each of the fused kernel's
# CTAs, while the separate sketch kernel runs it at full occupancy; the q'
# re-read it saves is an L2 hit.
_RAD_FUSED = os.environ.get("SGS_RAD_FUSED", "0") == "1"

# SGS_DEBUG_POISON=1: fill new Q storage with NaN (uninitialised-read check)
_POISON = os.environ.get("SGS_DEBUG_POISON", "0") == "1"

# SGS_PEER=0: row-sharded states all-reduce s' with NCCL per column instead of
# the peer-memory exchange inside the LS launch (A/B switch)
_PEER = os.environ.get("SGS_PEER", "1") != "0"

# SGS_PHI_FUSED=0 sketches Phi q' with its own launch (A/B and parity switch)
_PHI_FUSED = os.environ.get("SGS_PHI_FUSED", "1") != "0"

# SGS_LS_DEFER=0 forms every T column inside its own finalize (A/B switch)
_LS_DEFER = os.environ.get("SGS_LS_DEFER", "1") != "0"


def _pinned_buffer(shape, dtype):
    """Pinned host buffer (tensor, numpy view) for returned factors.

    Page-locking gigabytes on every call would dominate the end-to-end time, so
    buffers are pooled.  Ownership is explicit: each hand-out creates a fresh
    numpy array over the buffer and the pool keeps only a weak reference to
    it.  The buffer is reused once that array - and every view of it (views
    hold their base) - has been garbage collected; while a caller holds any of
    them, a new buffer is allocated.  (A raw data pointer is not ownership:
    copy the array to keep data past the result's lifetime.)"""
    import weakref
    for ent in _PINNED_POOL:
        t, ref = ent
        if tuple(t.shape) == tuple(shape) and t.dtype == dtype and ref() is None:
            arr = t.numpy()
            ent[1] = weakref.ref(arr)
            return t, arr
    t = torch.empty(shape, dtype=dtype, pin_memory=True)
    arr = t.numpy()  # arr.base is t: the array keeps the pinned storage alive
    _PINNED_POOL.append([t, weakref.ref(arr)])
    if len(_PINNED_POOL) > 12:  # Q, R, S, P of three live results
        _PINNED_POOL.pop(0)
    return t, arr


def _is_pinned(a: np.ndarray) -> bool:
    try:
        return torch.from_numpy(a.T if a.flags.f_contiguous else a).is_pinned()
    except Exception:
        return False


def ctypes_byref(a):
    import ctypes
    return ctypes.byref(a)


def _device_columns(W, device) -> tuple[torch.Tensor, int]:
    """Column-major device copy (or view) of an n x m W: returns (tensor whose
    column j starts at j*ld, ld)."""
    if isinstance(W, torch.Tensor) and W.is_cuda:
        n, m = W.shape
        if W.dtype not in (torch.float32, torch.float64):
            W = W.to(torch.float64)
        if W.stride(0) == 1 and W.stride(1) >= n and W.stride(1) % 4 == 0:
            return W, W.stride(1)
        Wt = torch.empty((m, _round_up(n, 4)), dtype=W.dtype, device=W.device)
        Wt[:, :n] = W.t()
        return Wt.t()[:n], Wt.stride(0)
    Wn = np.asarray(W)
    if Wn.dtype not in (np.float32, np.float64):
        Wn = Wn.astype(np.float64)
    n, m = Wn.shape
    ld = _round_up(n, 4)
    dt = _lib.torch_dtype(Wn.dtype)
    Wt = torch.empty((m, ld), dtype=dt, device=device)
    if Wn.flags.f_contiguous:
        Wt[:, :n].copy_(torch.from_numpy(Wn.T))
    else:
        tmp = torch.from_numpy(np.ascontiguousarray(Wn)).to(device)
        call("sgs_transpose", tmp.data_ptr(), m, Wt.data_ptr(), ld, n, m,
             _lib.dtype_code(dt), stream_ptr())
        del tmp
    return Wt, ld


def rgs_factorize(W, theta, policy: PrecisionPolicy = MIXED32_64,
                  solver: LsqSolver = HOUSEHOLDER_QR, with_certificate: bool = True,
                  phi=None, breakdown_factor: float = BREAKDOWN_FACTOR, *,
                  device_factors: bool = False, comm=None, row0: int = 0):
    """Randomized Gram-Schmidt QR of the columns of W on the GPU.

    Returns (QrFactors, StabilityCertificate or None) like the reference
    (gram_schmidt.py:350-375).  W may be an n x m numpy array, a CUDA tensor
    (column-major views are used in place), or an iterable of columns
    (streamed through ``RgsState.push``).  ``device_factors=True`` keeps the
    factors on the GPU as CUDA tensors.  With ``comm`` W holds this rank's
    rows [row0, row0 + n_local) of a row-sharded matrix.
    """
    theta = as_device_sketch(theta)
    if isinstance(W, (np.ndarray, torch.Tensor)):
        if W.ndim != 2:
            raise ValueError("W must be a matrix")
        n_loc, m = W.shape
        n = theta.n if comm is not None else n_loc
        if not (theta.k >= m and n >= m >= 1):
            raise ValueError(f"need k >= m and n >= m >= 1, got "
                             f"k={theta.k}, n={n}, m={m}")
        if comm is None and n_loc != theta.n:
            raise ValueError("column length mismatch")
        state = RgsState(theta, policy, solver, phi=phi, capacity=m + 1,
                         breakdown_factor=breakdown_factor, comm=comm, row0=row0,
                         n_local=n_loc)
        if (isinstance(W, np.ndarray) and not device_factors and phi is None
                and W.dtype in (np.float32, np.float64) and W.flags.f_contiguous
                and _is_pinned(W)):
            factors = state.factorize_host_pipelined(W, m)
            cert = certificates(factors) if with_certificate else None
            return factors, cert
        Wd, ld = _device_columns(W, state.device)
        state.factorize_columns(Wd, ld, m)
    else:
        state = RgsState(theta, policy, solver, phi=phi, breakdown_factor=breakdown_factor)
        for w in W:
            state.push(w)
    factors = state.factors(device=device_factors)
    cert = certificates(factors) if with_certificate else None
    return factors, cert


def sketched_lsq(S_prev, p, solver: LsqSolver = HOUSEHOLDER_QR):
    """min_y ||S_prev y - p||_2 on the device (reference gram_schmidt.py:193-205,
    the "householder" branch; tests/test_gram_schmidt.py:96-114).

    Runs the least-squares kernel of the factorizer (``sgs_ls_step``): each
    column s_j is appended as RGS appends s'_j - normalised by r_jj = ||s_j||
    into the QR of the sketched basis - and p is solved against it, so
    y_j = r_j / r_jj.  That QR is NOT a Householder chain: it is the parallel
    selective-reorthogonalisation Gram-Schmidt QR documented in DESIGN.md
    section 3 (an orthogonal factor T, column norms alpha, explicit R_S^-1),
    backward stable for the well-conditioned bases RGS keeps.
    The reference's rank test (min|diag R| < 1e-8 max(max|diag R|, 1),
    gram_schmidt.py:186-189) runs on the column-normalised basis and raises
    ``np.linalg.LinAlgError``; a zero column (r_jj = 0) raises it too (the
    reference's Householder step gives it a zero diagonal).  numpy in -> numpy
    out, CUDA tensor in -> CUDA tensor out."""
    if solver.method != "householder":
        raise NotImplementedError("the device least-squares kernel is the QR solver "
                                  "(HOUSEHOLDER_QR)")
    _lib.require_cuda()
    on_dev = isinstance(S_prev, torch.Tensor) and S_prev.is_cuda
    S = S_prev if isinstance(S_prev, torch.Tensor) else torch.from_numpy(np.asarray(S_prev))
    if S.ndim == 1:
        S = S.reshape(-1, 1)
    if S.ndim != 2:
        raise ValueError("S_prev must be a k x i matrix")
    k, i = S.shape
    fdt = torch.float32 if S.dtype == torch.float32 else torch.float64
    dev = S.device if on_dev else torch.device("cuda", torch.cuda.current_device())
    pv = p if isinstance(p, torch.Tensor) else torch.from_numpy(np.asarray(p, dtype=np.float64))
    if tuple(pv.shape) != (k,):
        raise ValueError("right-hand side length mismatch")
    if i == 0:
        out = torch.zeros(0, dtype=fdt, device=dev)
        return out if on_dev else out.cpu().numpy()
    if i >= k:
        raise ValueError("cannot append more columns than rows")
    cols = S.to(device=dev, dtype=torch.float64).t().contiguous()  # (i, k): row j = s_j
    pd = pv.to(device=dev, dtype=torch.float64).contiguous()
    st = RgsState.__new__(RgsState)  # the LS half of a state: no basis Q
    st.device, st.k, st.phi, st._cap = dev, k, None, 0
    st.policy = UNIFIED64 if fdt == torch.float64 else MIXED32_64
    st.breakdown_factor = 0.0  # tol = 0: only an exactly zero column "breaks down"
    st.cdt = st.fdt = fdt
    st.ccode = st.fcode = _lib.dtype_code(fdt)
    st.ldq = st.n_local = 32
    with torch.cuda.device(dev):
        st.status = _lib.Status(dev)
        st._alloc(i + 2)
        st._P[0].copy_(cols[0])  # the first finalize takes s'_1 = p_1 (RGS step i == 0)
        # An LS launch reads the LS state (T, alpha, R_S^-1, status) before its
        # programmatic-dependent-launch wait: in the factorizer a column or
        # sketch kernel always separates two LS launches.  Back to back, a
        # plain (non-PDL) kernel in between keeps the next launch from
        # starting before the previous one has finished.
        fence = torch.zeros(1, dtype=torch.int32, device=dev)
        for j in range(i):
            st._ls(fin=j, s_parts=cols[j].data_ptr(), s_nparts=1, s_scale=1.0)
            fence.add_(1)
        st._ls(sol=i, p_parts=pd.data_ptr(), p_nparts=1, p_scale=1.0)
        res = st.status.read()
    if res["code"] in (_lib.ST_RANK, _lib.ST_BREAKDOWN):
        raise np.linalg.LinAlgError("sketched basis numerically rank deficient")
    R = st._R  # column c of R is row c of the tensor
    y = (R[i, :i] / torch.diagonal(R)[:i]).to(fdt)
    return y if on_dev else y.cpu().numpy()


def certificates(factors: QrFactors) -> StabilityCertificate:
    """Delta_m, Delta~_m and cond(S) in binary64 (gram_schmidt.py:474-487)."""
    if factors.S is None or factors.P is None:
        raise ValueError("certificates need the sketches S and P (randomized factors)")
    if isinstance(factors.S, torch.Tensor):
        S = factors.S.to(torch.float64)
        P = factors.P.to(torch.float64)
        R = factors.R.to(torch.float64)
        m = S.shape[1]
        eye = torch.eye(m, dtype=torch.float64, device=S.device)
        delta_m = float(torch.linalg.norm(eye - S.t() @ S))
        delta_tilde = float(torch.linalg.norm(P - S @ R) / torch.linalg.norm(P))
        sv = torch.linalg.svdvals(S)
        cond_s = float(sv[0] / sv[-1]) if float(sv[-1]) > 0 else math.inf
        return StabilityCertificate(delta_m, delta_tilde, cond_s)
    S = np.asarray(factors.S, dtype=np.float64)
    P = np.asarray(factors.P, dtype=np.float64)
    R = np.asarray(factors.R)
    m = S.shape[1]
    delta_m = float(np.linalg.norm(np.eye(m) - S.T @ S))
    delta_tilde = float(np.linalg.norm(P - S @ R) / np.linalg.norm(P))
    sv = np.linalg.svd(S, compute_uv=False)
    cond_s = float(sv[0] / sv[-1]) if sv[-1] > 0 else np.inf
    return StabilityCertificate(delta_m=delta_m, delta_tilde_m=delta_tilde, cond_S=cond_s)


def loss_of_orthogonality(Q) -> float:
    """||I - Q^T Q||_F in binary64 (gram_schmidt.py:490-494)."""
    if isinstance(Q, torch.Tensor):
        Qd = Q.to(torch.float64)
        m = Qd.shape[1]
        return float(torch.linalg.norm(torch.eye(m, dtype=torch.float64, device=Qd.device)
                                       - Qd.t() @ Qd))
    Qn = np.asarray(Q, dtype=np.float64)
    m = Qn.shape[1]
    return float(np.linalg.norm(np.eye(m) - Qn.T @ Qn))
