"""Oracle sketch operators (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Restates reference sketch.py: P-SRHT construction (sketch.py:123-145), the
unnormalised Sylvester FWHT (sketch.py:90-109) and apply (sketch.py:168-184);
Rademacher columns (sketch.py:153-166).  Gaussian and block-SRHT are the
BASELINE additions defined in paper_2011_05090_b200/sketch.py docstring.
"""

from __future__ import annotations

import math

import numpy as np


def _gen(seed: int, stream: int) -> np.random.Generator:
    # sketch.py:116-117
    return np.random.Generator(np.random.Philox(key=(int(seed) << 64) | int(stream)))


def psrht_setup(k: int, n: int, seed: int):
    """(s, signs fp64 +-1, sorted samples) as sketch.py:134-143 draws them."""
    s = 1 << (int(n) - 1).bit_length()
    signs = 2.0 * _gen(seed, 0x5149).integers(0, 2, size=n) - 1.0
    order = _gen(seed, 0xFA7E).permutation(s)
    return s, signs, np.sort(order[:k])


def fwht_ref(v):
    """Radix-2 Sylvester FWHT along axis 0, stages h = 1, 2, 4, ... (sketch.py:100-108)."""
    a = np.array(v, copy=True)
    s = a.shape[0]
    if s < 1 or s & (s - 1):
        raise ValueError(f"leading dimension {s} is not a power of two")
    shape = a.shape
    cols = a.reshape(s, -1)
    h = 1
    while h < s:
        blk = cols.reshape(s // (2 * h), 2, h, -1)
        lo, hi = blk[:, 0], blk[:, 1]
        cols = np.stack((lo + hi, lo - hi), axis=1).reshape(s, -1)
        h <<= 1
    return cols.reshape(shape)


# numpy's Philox is Random123 Philox4x64-10 (numpy/random/src/philox/philox.h):
# multipliers, Weyl key increments, and the counter incremented before each
# block of four 64-bit outputs.
_PH_M = (0xD2E7470EE14C6C93, 0xCA5A826395121157)
_PH_W = (0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B)
_M64 = (1 << 64) - 1


def philox4x64_10(ctr, key):
    c, k = list(ctr), list(key)
    for r in range(10):
        if r:
            k = [(k[0] + _PH_W[0]) & _M64, (k[1] + _PH_W[1]) & _M64]
        p0, p1 = _PH_M[0] * c[0], _PH_M[1] * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k[0], p1 & _M64, (p0 >> 64) ^ c[3] ^ k[1], p0 & _M64]
    return c


def rademacher_column_bits(seed: int, j: int, k: int) -> np.ndarray:
    """Philox(key=(seed << 64) | j).integers(0, 2, size=k) (sketch.py:153-158)
    restated from the bit generator: next_uint32 returns the low then the high
    half of each 64-bit output, and the bounded draw over {0, 1} (Lemire,
    numpy's default for Generator.integers) is the top bit of one uint32.  This
    is the algorithm the device generator sgs_rademacher_bits implements;
    pinned against numpy by tests/test_oracle_golden.py."""
    key = [int(j) & _M64, int(seed) & _M64]
    out, ctr = [], 0
    while len(out) < k:
        ctr += 1
        for v in philox4x64_10([ctr, 0, 0, 0], key):
            out.append((v & 0xFFFFFFFF) >> 31)
            out.append(v >> 63)
    return np.asarray(out[:k], dtype=np.int64)


def block_seed(seed: int, j: int) -> int:
    return int(seed) * 1_000_003 + int(j)


class OracleSketch:
    """Duck-typed k x n operator (.k, .n, .apply, .apply_block) on the host."""

    def __init__(self, kind: str, k: int, n: int, seed: int, block_log2: int = 20,
                 threads: int = 1):
        self.kind, self.k, self.n, self.seed = kind, int(k), int(n), int(seed)
        # block-SRHT only: transform the blocks on `threads` host threads (numpy
        # releases the GIL); the block sums are still added in block order, so
        # the result is bit-identical to threads=1
        self.threads = int(threads)
        if kind == "psrht":
            self.s, self.signs, self.samples = psrht_setup(k, n, seed)
        elif kind == "block_srht":
            bs = 1 << block_log2
            if n % bs:
                raise ValueError("block-SRHT needs n a multiple of the block size")
            self.bs = bs
            self.blocks = [psrht_setup(k, bs, block_seed(seed, j)) for j in range(n // bs)]
        elif kind == "gaussian":
            # unscaled Theta (k x n, C order); drawn as Theta^T (n, k)
            self.D = np.ascontiguousarray(_gen(seed, 0x6A55).standard_normal((n, k)).T)
        elif kind == "rademacher":
            self.D = np.empty((k, n))  # sketch.py:153-158, column j from stream j
            for j in range(n):
                self.D[:, j] = 2.0 * _gen(seed, j).integers(0, 2, size=k) - 1.0
        else:
            raise TypeError(kind)

    def _psrht(self, s, signs, samples, x):
        # sketch.py:182-184: scale * fwht(pad(signs * x))[samples]
        buf = np.zeros(s)
        buf[:x.shape[0]] = signs * x
        return (1.0 / math.sqrt(self.k)) * fwht_ref(buf)[samples]

    def apply(self, x) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ValueError(f"expected vector of length {self.n}, got {x.shape}")
        if self.kind == "psrht":
            return self._psrht(self.s, self.signs, self.samples, x)
        if self.kind == "block_srht":
            acc = np.zeros(self.k)
            one = lambda j: self._psrht(*self.blocks[j], x[j * self.bs:(j + 1) * self.bs])  # noqa: E731
            if self.threads > 1:
                from concurrent.futures import ThreadPoolExecutor
                with ThreadPoolExecutor(min(self.threads, len(self.blocks))) as ex:
                    parts = list(ex.map(one, range(len(self.blocks))))
            else:
                parts = map(one, range(len(self.blocks)))
            for y in parts:
                acc += y
            return acc / math.sqrt(len(self.blocks))
        return (1.0 / math.sqrt(self.k)) * (self.D @ x)   # sketch.py:174-175

    def apply_block(self, X) -> np.ndarray:
        X = np.asarray(X, dtype=np.float64)
        if X.ndim == 1:
            X = X[:, None]
        return np.stack([self.apply(X[:, j]) for j in range(X.shape[1])], axis=1)
