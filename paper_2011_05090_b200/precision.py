"""Two-roundoff arithmetic model (u_crs, u_fine) realised as device dtypes.

Mirrors the reference's ``precision.py:19-52``: the coarse format stores Q and
runs the n-dimensional projection update (step 3), the fine format holds the
sketches S, P, the least-squares work and R.  On the device the coarse format
is the element type of the Q stream (fp32 halves its HBM bytes), the fine
format the type of the k-dimensional cluster kernel.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

U_BINARY32 = 2.0**-24
U_BINARY64 = 2.0**-53


@dataclass(frozen=True)
class PrecisionPolicy:
    """A (u_crs, u_fine) pair realised as dtypes per operation class."""

    mode: str  # "f32" | "f64" | "mixed"
    coarse_dtype: np.dtype
    fine_dtype: np.dtype
    u_crs: float
    u_fine: float

    def __post_init__(self):
        if self.u_fine > self.u_crs:
            raise ValueError("u_fine must not exceed u_crs")

    def __repr__(self):
        return f"PrecisionPolicy({self.mode!r})"


UNIFIED32 = PrecisionPolicy("f32", np.dtype(np.float32), np.dtype(np.float32),
                            U_BINARY32, U_BINARY32)
UNIFIED64 = PrecisionPolicy("f64", np.dtype(np.float64), np.dtype(np.float64),
                            U_BINARY64, U_BINARY64)
MIXED32_64 = PrecisionPolicy("mixed", np.dtype(np.float32), np.dtype(np.float64),
                             U_BINARY32, U_BINARY64)

_BY_NAME = {"f32": UNIFIED32, "f64": UNIFIED64, "mixed": MIXED32_64}


def policy_from_name(name: str) -> PrecisionPolicy:
    """Look a policy up by name; ValueError on an unknown name (precision.py:47-52)."""
    if name not in _BY_NAME:
        raise ValueError(f"unknown precision policy {name!r}; "
                         f"expected one of {sorted(_BY_NAME)}")
    return _BY_NAME[name]
