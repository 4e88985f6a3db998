"""Oblivious subspace embeddings Theta applied on the B200.

Interface mirror of the reference's ``sketch.py`` (SketchKind,
SketchOperator(kind, k, n, seed), make_sketch, fwht; ``sketch.py:39-210``):
``apply(x)`` / ``apply_block(X, col_range)`` return numpy arrays for numpy
inputs (so the operator drops into the reference's own ``RgsState``, which
calls ``.astype`` on the result, ``gram_schmidt.py:303``) and CUDA tensors for
CUDA-tensor inputs.  Shape errors raise ``ValueError`` as ``sketch.py:171-172``.

Kinds:

* ``PSRHT`` - the reference's partial subsampled randomized Hadamard
  transform.  Signs and sorted row samples are drawn exactly as the reference
  constructor does (numpy Philox keyed ``(seed << 64) | stream`` with streams
  0x5149 / 0xFA7E, ``sketch.py:116-145``), then uploaded once: signs as a
  packed bitmask, samples as int32.  Applied by one tile-FWHT kernel.
* ``RADEMACHER`` - the reference's +-1/sqrt(k) kind.  Its per-column Philox
  streams (``sketch.py:153-166``) are regenerated on the device bit for bit
  (``sgs_rademacher_bits``: numpy's Philox4x64-10, top bit of each 32-bit
  draw) and kept packed, 1 bit per entry; applied by
  ``sgs_rademacher_partials`` with the dense kernels' chunking and chains.
* ``GAUSSIAN`` (absent from the reference; BASELINE config 0) - Theta_ij
  = g_ij / sqrt(k), g ~ N(0, 1) from ``Philox((seed << 64) | 0x6A55)`` drawn as
  an (n, k) array (Theta column-major), applied by the dense kernel.
* ``BLOCK_SRHT`` (absent; BASELINE configs 2 and 4) - Theta = [Theta_1 ...
  Theta_B] / sqrt(B) over B contiguous 2^L-row blocks, Theta_j the reference
  P-SRHT (k, 2^L, seed_j) with ``seed_j = block_seed(seed, j)``.  Note that
  every Theta_j already carries 1/sqrt(k), so the literal 1/sqrt(B) scales the
  sketched norm by 1/sqrt(B) (and Q by sqrt(B)); implemented literally.
"""

from __future__ import annotations

import math
import warnings
from enum import Enum

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream_ptr

__all__ = ["SketchKind", "SketchOperator", "make_sketch", "fwht", "block_seed",
           "as_device_sketch", "next_pow2"]

_PSRHT_SIGN_STREAM = 0x5149
_PSRHT_SAMPLE_STREAM = 0xFA7E
_GAUSSIAN_STREAM = 0x6A55


class SketchKind(Enum):
    RADEMACHER = "rademacher"
    PSRHT = "psrht"
    GAUSSIAN = "gaussian"
    BLOCK_SRHT = "block_srht"


def next_pow2(n: int) -> int:
    return 1 << (int(n) - 1).bit_length()


def _philox(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=(int(seed) << 64) | int(stream)))


def block_seed(seed: int, j: int) -> int:
    """Seed of block j of a block-SRHT (documented, shared with the oracle)."""
    return int(seed) * 1_000_003 + int(j)


def _psrht_arrays(k: int, n: int, seed: int):
    """Signs (fp64 +-1, length n) and sorted samples (int64, length k) of the
    reference P-SRHT constructor (sketch.py:134-143)."""
    s = next_pow2(n)
    bits = _philox(seed, _PSRHT_SIGN_STREAM).integers(0, 2, size=n)
    signs = 2.0 * bits - 1.0
    perm = _philox(seed, _PSRHT_SAMPLE_STREAM).permutation(s)
    return s, signs, np.sort(perm[:k])


def _pack_signs(signs: np.ndarray) -> np.ndarray:
    bits = np.packbits(np.asarray(signs) > 0, bitorder="little")
    pad = (-bits.size) % 4
    if pad:
        bits = np.concatenate([bits, np.zeros(pad, dtype=np.uint8)])
    return bits.view("<u4").astype(np.uint32)


MAX_SRHT_ROWS = 8192  # shared-memory bound of the SRHT kernels (BASELINE uses k <= 3000)


class SketchOperator:
    """A seeded k x n embedding applied on the GPU without forming it when
    structured (P-SRHT kinds) or as a dense fp64 stream (Gaussian/Rademacher)."""

    def __init__(self, kind: SketchKind, k: int, n: int, seed: int, block_log2: int = 20):
        if k < 1 or n < 1:
            raise ValueError("k and n must be positive")
        if k > n:
            warnings.warn(f"sketch dimension k={k} exceeds ambient dimension n={n}",
                          stacklevel=3)
        if not isinstance(kind, SketchKind):
            raise TypeError(f"unknown sketch kind {kind!r}")
        if kind in (SketchKind.PSRHT, SketchKind.BLOCK_SRHT) and k > MAX_SRHT_ROWS:
            # each CTA keeps the k-vector and the sample rows in shared memory
            raise ValueError(f"P-SRHT sketches support k <= {MAX_SRHT_ROWS} rows on the "
                             f"B200 kernels (got k={k})")
        self.kind = kind
        self.k = int(k)
        self.n = int(n)
        self.seed = int(seed)
        self._dev = {}
        if kind is SketchKind.PSRHT:
            s = next_pow2(n)
            if s >= 1 << 62:
                raise OverflowError("padded Hadamard size overflows")
            self.s, self.signs, self.sample_indices = _psrht_arrays(k, n, seed)
            self.nblocks = 1
            self.log2_block = s.bit_length() - 1
            self.scale = 1.0 / math.sqrt(self.k)
        elif kind is SketchKind.BLOCK_SRHT:
            bs = 1 << int(block_log2)
            if n % bs != 0:
                raise ValueError(f"block-SRHT needs n a multiple of the block size {bs}")
            self.nblocks = n // bs
            self.log2_block = int(block_log2)
            self.s = bs
            signs, samples = [], []
            for j in range(self.nblocks):
                _, sg, sm = _psrht_arrays(k, bs, block_seed(seed, j))
                signs.append(sg)
                samples.append(sm)
            self.signs = np.concatenate(signs)
            self.sample_indices = np.stack(samples)  # (B, k)
            self.scale = 1.0 / math.sqrt(self.k) / math.sqrt(self.nblocks)
        elif kind in (SketchKind.GAUSSIAN, SketchKind.RADEMACHER):
            self.scale = 1.0 / math.sqrt(self.k)
        else:  # pragma: no cover - enum exhausted
            raise TypeError(f"unknown sketch kind {kind!r}")

    def __repr__(self):
        return (f"SketchOperator({self.kind.value}, k={self.k}, n={self.n}, "
                f"seed={self.seed})")

    # ---- host construction of dense kinds --------------------------------------
    def _dense_host(self) -> np.ndarray:
        """Unscaled Theta^T (n x k) of the Gaussian kind: N(0,1) entries."""
        return _philox(self.seed, _GAUSSIAN_STREAM).standard_normal((self.n, self.k))

    @property
    def is_dense(self) -> bool:
        """Applied by the dense chunking (Gaussian fp64 stream or Rademacher bits)."""
        return self.kind in (SketchKind.GAUSSIAN, SketchKind.RADEMACHER)

    @property
    def is_gaussian(self) -> bool:
        """Dense fp64 Theta^T in HBM (the fused dense column kernel)."""
        return self.kind is SketchKind.GAUSSIAN

    # ---- device resources -------------------------------------------------------
    def device_data(self, device=None) -> dict:
        _lib.require_cuda()
        dev = torch.device("cuda") if device is None else torch.device(device)
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        key = str(dev)
        d = self._dev.get(key)
        if d is not None:
            return d
        if self.kind is SketchKind.RADEMACHER:
            kw = (self.k + 31) // 32
            bits = torch.empty((self.n, kw), dtype=torch.int32, device=dev)
            with torch.cuda.device(dev):
                call("sgs_rademacher_bits", self.seed & (2**64 - 1), 0, self.n, self.k,
                     bits.data_ptr(), stream_ptr())
            d = {"rbits": bits, "kw": kw}
        elif self.is_dense:
            ldt = self.k + (self.k & 1)
            host = self._dense_host()
            t = torch.zeros((self.n, ldt), dtype=torch.float64, device=dev)
            t[:, :self.k] = torch.from_numpy(host).to(dev)
            d = {"thetaT": t, "ldt": ldt}
        else:
            samples = np.asarray(self.sample_indices, dtype=np.int64).reshape(self.nblocks, self.k)
            d = {"bits": torch.from_numpy(_pack_signs(self.signs).view(np.int32)).to(dev),
                 "samples": torch.from_numpy(samples.astype(np.int32)).to(dev)}
        self._dev[key] = d
        return d

    def nparts(self, n_local: int | None = None) -> int:
        n_local = self.n if n_local is None else int(n_local)
        lib = _lib.load()
        if self.kind is SketchKind.GAUSSIAN:
            return int(lib.sgs_gaussian_nparts(n_local))
        if self.is_dense:
            return int(lib.sgs_dense_nparts(n_local))
        return int(lib.sgs_srht_nparts(n_local, self.log2_block))

    def row_align(self) -> int:
        """Row granularity a shard boundary must respect."""
        if self.is_dense:
            return 1
        return 1 << min(self.log2_block, 12)

    def partials_into(self, X: torch.Tensor | int, x_dtype: int, ldx: int, ncols: int,
                      out: torch.Tensor, *, n_local: int | None = None, row0: int = 0,
                      status=None, stream=None, small_grid: bool = False) -> int:
        """Launch the partial sketches of ncols columns of X (device pointer or
        tensor, column-major with leading dimension ldx) into ``out``.  Returns
        the number of parts per column."""
        d = self.device_data(out.device)
        n_local = self.n if n_local is None else int(n_local)
        xp = X if isinstance(X, int) else X.data_ptr()
        sp = stream_ptr(stream)
        st = status.ptr if status is not None else None
        if self.kind is SketchKind.RADEMACHER:
            np_ = self.nparts(n_local)
            bp = d["rbits"].data_ptr() + row0 * d["kw"] * 4
            call("sgs_rademacher_partials", bp, self.k, xp, x_dtype, ldx, ncols, n_local,
                 out.data_ptr(), st, sp)
            return np_
        if self.is_dense:
            np_ = self.nparts(n_local)
            thetaT = d["thetaT"]
            tp = thetaT.data_ptr() + row0 * d["ldt"] * 8
            call("sgs_dense_partials", tp, d["ldt"], self.k, xp, x_dtype, ldx, ncols,
                 n_local, out.data_ptr(), st, sp)
            return np_
        np_ = self.nparts(n_local)
        if row0 % 32:
            raise ValueError("shard row offset must be a multiple of 32")
        bp = d["bits"].data_ptr() + (row0 // 32) * 4
        # small_grid: one CTA per 4 tiles (same partials) so that a cluster
        # launch queued behind finds free SMs (sgs_srht_partials_geom)
        call("sgs_srht_partials_geom", xp, x_dtype, ldx, ncols, n_local, row0, self.log2_block,
             bp, d["samples"].data_ptr(), self.k, out.data_ptr(), 1 if small_grid else 0, st, sp)
        return np_

    # ---- reference-facing application ------------------------------------------
    def _apply_device(self, X: torch.Tensor) -> torch.Tensor:
        """X: CUDA tensor (n,) or (n, c), fp32/fp64 -> fp64 (k,) / (k, c)."""
        vec = X.dim() == 1
        Xc = X.reshape(self.n, -1)
        if Xc.dtype not in (torch.float32, torch.float64):
            Xc = Xc.to(torch.float64)
        ncols = Xc.shape[1]
        Xcm = Xc.t().contiguous()  # (ncols, n): column-major, ld = n (no copy if already so)
        ldx = self.n
        nparts = self.nparts()
        parts = torch.empty((ncols, nparts, self.k), dtype=torch.float64, device=X.device)
        self.partials_into(Xcm, _lib.dtype_code(Xc.dtype), ldx, ncols, parts)
        Y = torch.empty((ncols, self.k), dtype=torch.float64, device=X.device)
        call("sgs_partials_reduce", parts.data_ptr(), nparts, self.k, ncols, self.scale,
             Y.data_ptr(), _lib.SGS_F64, self.k, None, stream_ptr())
        return Y[0] if vec else Y.t()

    def apply(self, x):
        """Return Theta @ x for an n-vector (fp64 result)."""
        if isinstance(x, torch.Tensor) and x.is_cuda:
            if tuple(x.shape) != (self.n,):
                raise ValueError(f"expected vector of length {self.n}, got {tuple(x.shape)}")
            return self._apply_device(x)
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ValueError(f"expected vector of length {self.n}, got {x.shape}")
        _lib.require_cuda()
        return self._apply_device(torch.from_numpy(x).cuda()).cpu().numpy()

    def apply_block(self, X, col_range: slice | None = None):
        """Columnwise Theta @ X; bit-identical to per-column ``apply``."""
        if isinstance(X, torch.Tensor) and X.is_cuda:
            if X.dim() == 1:
                X = X[:, None]
            if X.shape[0] != self.n:
                raise ValueError(f"expected {self.n} rows, got {X.shape[0]}")
            if col_range is not None:
                X = X[:, col_range]
            return self._apply_device(X)
        X = np.asarray(X, dtype=np.float64)
        if X.ndim == 1:
            X = X[:, None]
        if X.shape[0] != self.n:
            raise ValueError(f"expected {self.n} rows, got {X.shape[0]}")
        if col_range is not None:
            X = X[:, col_range]
        _lib.require_cuda()
        Xt = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()  # (c, n) = column-major X
        return self._apply_device(Xt.t()).cpu().numpy()

    def materialize(self) -> np.ndarray:
        """Dense k x n matrix; for small-n diagnostics and tests."""
        return self.apply_block(np.eye(self.n))

    def frobenius_norm(self) -> float:
        if self.kind in (SketchKind.PSRHT, SketchKind.RADEMACHER):
            return math.sqrt(self.n)  # every entry is +-1/sqrt(k)
        if self.kind is SketchKind.BLOCK_SRHT:
            return math.sqrt(self.n / self.nblocks)
        return float(np.linalg.norm(self._dense_host())) * self.scale


def make_sketch(kind: SketchKind, k: int, n: int, seed: int, **kw) -> SketchOperator:
    return SketchOperator(kind, k, n, seed, **kw)


def as_device_sketch(theta) -> SketchOperator:
    """Accept this package's operator, or adopt a reference ``sketchgs``
    P-SRHT / Rademacher operator (same kind, k, n, seed and, for P-SRHT, the
    very sign/sample arrays it holds)."""
    if isinstance(theta, SketchOperator):
        return theta
    kind = getattr(getattr(theta, "kind", None), "value", None)
    if kind == "psrht" and hasattr(theta, "signs") and hasattr(theta, "sample_indices"):
        op = SketchOperator.__new__(SketchOperator)
        op.kind, op.k, op.n, op.seed = SketchKind.PSRHT, int(theta.k), int(theta.n), int(theta.seed)
        op._dev = {}
        op.s = next_pow2(op.n)
        op.signs = np.asarray(theta.signs, dtype=np.float64)
        op.sample_indices = np.asarray(theta.sample_indices)
        op.nblocks, op.log2_block = 1, op.s.bit_length() - 1
        op.scale = 1.0 / math.sqrt(op.k)
        return op
    if kind == "rademacher":
        return SketchOperator(SketchKind.RADEMACHER, theta.k, theta.n, theta.seed)
    raise TypeError("the device factorizer needs a paper_2011_05090_b200 SketchOperator "
                    f"(or a reference P-SRHT/Rademacher operator); got {type(theta)!r}")


def fwht(v):
    """Unnormalised Sylvester FWHT along axis 0 (sketch.py:90-109), on the GPU.

    Float inputs are transformed in binary64 and returned in their dtype."""
    is_t = isinstance(v, torch.Tensor) and v.is_cuda
    a = v if is_t else np.array(v, copy=True)
    s = a.shape[0]
    if s < 1 or (s & (s - 1)) != 0:
        raise ValueError(f"leading dimension {s} is not a power of two")
    shape = tuple(a.shape)
    _lib.require_cuda()
    if is_t:
        out_dtype = a.dtype
        X = a.reshape(s, -1).to(torch.float64)
    else:
        out_dtype = a.dtype
        X = torch.from_numpy(np.asarray(a, dtype=np.float64).reshape(s, -1)).cuda()
    ncols = X.shape[1]
    Xc = X.t().contiguous()  # (ncols, s): column-major
    call("sgs_fwht", Xc.data_ptr(), s, ncols, s, stream_ptr())
    Y = Xc.t().reshape(shape)
    if is_t:
        return Y.to(out_dtype)
    return Y.cpu().numpy().astype(out_dtype, copy=False)
