"""ctypes binding of the C ABI in include/sketchgs_b200.h.

The shared library is built in-tree (``paper_2011_05090_b200/_lib/``) by
``__graft_entry__.build()`` / ``make -C paper_2011_05090_b200/csrc``.  There is
no fallback: every compute entry point of the package goes through this
library, and using one without the library (or without a CUDA device) raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int64, c_uint64, c_void_p

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# SGS_LIB_CHECKED=1: the checked build (device-side bound checks, `make checked`)
LIB_PATH = os.path.join(_HERE, "_lib", "libsketchgs_b200_checked.so"
                        if os.environ.get("SGS_LIB_CHECKED", "0") == "1" else "libsketchgs_b200.so")

SGS_F32 = 0
SGS_F64 = 1

ST_OK = 0
ST_BREAKDOWN = 1
ST_RANK = 2
ST_CONVERGED = 3
ST_TIMEOUT = 4


class LsArgs(ctypes.Structure):
    """Mirror of ``sgs_ls_args``."""

    _fields_ = [
        ("k", c_int), ("cap", c_int), ("fine_dtype", c_int), ("coarse_dtype", c_int),
        ("do_finalize", c_int), ("col_fin", c_int),
        ("s_partials", c_void_p), ("s_nparts", c_int), ("s_scale", c_double),
        ("do_solve", c_int), ("col_sol", c_int),
        ("p_partials", c_void_p), ("p_nparts", c_int), ("p_scale", c_double),
        ("bf_ucrs", c_double),
        ("S", c_void_p), ("P", c_void_p), ("R", c_void_p),
        ("Qs", c_void_p), ("Rinv", c_void_p), ("alpha", c_void_p), ("scratch", c_void_p),
        ("r_crs", c_void_p), ("st", c_void_p), ("trace", c_void_p), ("cache_cols", c_int),
        ("timeline", c_void_p), ("t_pend", c_void_p), ("t_coef", c_void_p),
        ("p_lag", c_int),
        ("giv_on", c_int), ("giv_cs", c_void_p), ("giv_sn", c_void_p), ("giv_g", c_void_p),
        ("giv_T", c_void_p), ("giv_ldt", ctypes.c_longlong), ("giv_hist", c_void_p),
        ("giv_tol", c_double),
        ("peer", c_void_p),
    ]


# name -> (restype, argtypes)
_SIGS = {
    "sgs_abi_version": (c_int, []),
    "sgs_debug_timeline": (None, [c_void_p]),
    "sgs_debug_timeline_col": (None, [c_int64]),
    "sgs_last_error": (ctypes.c_char_p, []),
    "sgs_launch_count": (c_uint64, []),
    "sgs_device_sm_count": (c_int, [c_int]),
    "sgs_status_init": (c_int, [c_void_p, c_void_p]),
    "sgs_srht_nparts": (c_int, [c_int64, c_int]),
    "sgs_srht_partials": (c_int, [c_void_p, c_int, c_int64, c_int, c_int64, c_int64, c_int,
                                  c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "sgs_dense_nparts": (c_int, [c_int64]),
    "sgs_gaussian_nparts": (c_int, [c_int64]),
    "sgs_dense_column_nparts": (c_int, [c_int64, c_int]),
    "sgs_dense_partials": (c_int, [c_void_p, c_int64, c_int, c_void_p, c_int, c_int64, c_int,
                                   c_int64, c_void_p, c_void_p, c_void_p]),
    "sgs_mm_read_header": (c_int, [ctypes.c_char_p, POINTER(c_int64), POINTER(c_int64),
                                   POINTER(c_int64), POINTER(c_int)]),
    "sgs_mm_read_entries": (c_int, [ctypes.c_char_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "sgs_rademacher_bits": (c_int, [c_uint64, c_int64, c_int64, c_int, c_void_p, c_void_p]),
    "sgs_rademacher_partials": (c_int, [c_void_p, c_int, c_void_p, c_int, c_int64, c_int,
                                        c_int64, c_void_p, c_void_p, c_void_p]),
    "sgs_partials_reduce": (c_int, [c_void_p, c_int, c_int, c_int, c_double, c_void_p, c_int,
                                    c_int64, c_void_p, c_void_p]),
    "sgs_partials_reduce_div": (c_int, [c_void_p, c_int, c_int, c_int, c_double, c_void_p,
                                        c_void_p, c_int, c_int64, c_void_p, c_void_p]),
    "sgs_fwht": (c_int, [c_void_p, c_int64, c_int, c_int64, c_void_p]),
    "sgs_rgs_update": (c_int, [c_void_p, c_int, c_int64, c_int64, c_int, c_void_p, c_int,
                               c_void_p, c_int, c_void_p, c_int64, c_void_p, c_void_p]),
    "sgs_column_nparts": (c_int, [c_int64]),
    "sgs_rgs_update_srht": (c_int, [c_void_p, c_int, c_int64, c_int64, c_int, c_void_p, c_int,
                                    c_void_p, c_void_p, c_int, c_void_p, c_int64, c_int, c_int64, c_int,
                                    c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "sgs_srht_partials_geom": (c_int, [c_void_p, c_int, c_int64, c_int, c_int64, c_int64, c_int,
                                       c_void_p, c_void_p, c_int, c_void_p, c_int, c_void_p,
                                       c_void_p]),
    "sgs_srht_partials_pair": (c_int, [c_void_p, c_int, c_int64, c_int, c_int64, c_int64, c_int,
                                       c_void_p, c_void_p, c_int, c_void_p, c_int, c_void_p,
                                       c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "sgs_rgs_update_srht_phi": (c_int, [c_void_p, c_int, c_int64, c_int64, c_int, c_void_p, c_int,
                                        c_void_p, c_void_p, c_int, c_void_p, c_int64, c_int,
                                        c_int64, c_int, c_void_p, c_void_p, c_int, c_void_p,
                                        c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p,
                                        c_void_p]),
    "sgs_rgs_update_dense": (c_int, [c_void_p, c_int, c_int64, c_int64, c_int, c_void_p, c_int,
                                     c_void_p, c_int, c_void_p, c_int64, c_int, c_void_p,
                                     c_int64, c_int, c_void_p, c_void_p, c_void_p]),
    "sgs_rgs_update_rademacher": (c_int, [c_void_p, c_int, c_int64, c_int64, c_int, c_void_p,
                                          c_int, c_void_p, c_int, c_void_p, c_int64, c_int,
                                          c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "sgs_normalize_column": (c_int, [c_void_p, c_int, c_int64, c_int64, c_int, c_void_p,
                                     c_int64, c_void_p, c_void_p]),
    "sgs_gemv_f64": (c_int, [c_void_p, c_int, c_int64, c_int64, c_int, c_void_p, c_void_p,
                             c_void_p]),
    "sgs_ls_scratch_elems": (c_int64, [c_int, c_int]),
    "sgs_ls_cluster_size": (c_int, [c_int]),
    "sgs_ls_step": (c_int, [POINTER(LsArgs), c_void_p]),
    "sgs_peer_bytes": (c_int64, [c_int, c_int, c_int]),
    "sgs_peer_alloc": (c_int, [c_int64, POINTER(c_void_p)]),
    "sgs_peer_free": (c_int, [c_void_p]),
    "sgs_peer_export": (c_int, [c_void_p, ctypes.c_char_p]),
    "sgs_peer_import": (c_int, [ctypes.c_char_p, POINTER(c_void_p)]),
    "sgs_peer_unimport": (c_int, [c_void_p]),
    "sgs_peer_desc_create": (c_int, [c_int, c_int, c_int, POINTER(c_void_p), POINTER(c_void_p)]),
    "sgs_peer_desc_free": (c_int, [c_void_p]),
    "sgs_peer_begin": (c_int, [c_void_p, c_void_p]),
    "sgs_csr_spmv": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p,
                             c_void_p, c_void_p, c_void_p, c_void_p]),
    "sgs_csr_spmv_srht": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                                  c_void_p, c_void_p, c_void_p, c_int64, c_int, c_void_p,
                                  c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                                  c_void_p]),
    "sgs_spmv_srht_tilevec_elems": (c_int64, [c_int64, c_int]),
    "sgs_spmv_srht_counter_elems": (c_int64, [c_int64]),
    "sgs_norm2": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_void_p, c_void_p]),
    "sgs_norm2_work_elems": (c_int64, [c_int64]),
    "sgs_scale": (c_int, [c_void_p, c_double, c_void_p, c_int, c_void_p, c_int64, c_void_p]),
    "sgs_rsub": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "sgs_cast_div": (c_int, [c_void_p, c_int, c_void_p, c_int, c_void_p, c_int64, c_void_p]),
    "sgs_cos_init": (c_int, [c_void_p, c_int64, c_void_p]),
    "sgs_cos_init_at": (c_int, [c_void_p, c_int64, c_int64, c_void_p]),
    "sgs_power_step": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    "sgs_givens_step": (c_int, [c_void_p, c_int64, c_int, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_int64, c_void_p, c_double, c_void_p, c_void_p]),
    "sgs_arnoldi_head": (c_int, [c_void_p, c_int, c_int64, c_int64, c_int, c_void_p, c_int64,
                                 c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                                 c_int64, c_void_p, c_double, c_void_p, c_void_p]),
    "sgs_transpose": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int,
                              c_void_p]),
    "sgs_ilu0_analysis_work_elems": (c_int64, [c_int64]),
    "sgs_ilu0_analyse": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                 c_void_p, c_void_p]),
    "sgs_ilu0_factor": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_void_p]),
    "sgs_ilu0_pending_fill": (c_int, [c_void_p, c_int64, c_void_p]),
    "sgs_ilu0_solve": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                               c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                               c_void_p]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


class LibraryMissing(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load (once) and return the ctypes library; raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LibraryMissing(
            f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_2011_05090_b200/csrc`")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.sgs_abi_version() != 1:
        raise LibraryMissing("ABI version mismatch")
    _lib = lib
    return lib


def lib():
    return load()


def srht_legacy() -> bool:
    """SGS_SRHT_LEGACY=1: the library's three-pass SRHT kernel (no pair kernel)."""
    return os.environ.get("SGS_SRHT_LEGACY", "0") not in ("", "0")


def require_cuda():
    load()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2011_05090_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = _lib.sgs_last_error().decode(errors="replace") if _lib else ""
        raise RuntimeError(f"sketchgs_b200 {what} failed (rc={rc}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def dtype_code(dt) -> int:
    if dt in (torch.float32, "float32"):
        return SGS_F32
    if dt in (torch.float64, "float64"):
        return SGS_F64
    import numpy as np
    d = np.dtype(dt)
    if d == np.float32:
        return SGS_F32
    if d == np.float64:
        return SGS_F64
    raise TypeError(f"unsupported dtype {dt!r}")


def torch_dtype(np_dtype) -> torch.dtype:
    import numpy as np
    d = np.dtype(np_dtype)
    if d == np.float32:
        return torch.float32
    if d == np.float64:
        return torch.float64
    raise TypeError(f"unsupported dtype {np_dtype!r}")


def launch_count() -> int:
    return int(load().sgs_launch_count())


class Status:
    """Device-resident ``sgs_status`` block (8 x int64 / double)."""

    def __init__(self, device):
        self.buf = torch.zeros(8, dtype=torch.int64, device=device)
        self.reset()

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()

    def reset(self) -> None:
        call("sgs_status_init", self.ptr, stream_ptr())

    def read(self) -> dict:
        h = self.buf.cpu()
        f = h.view(torch.float64)
        return {"code": int(h[0]), "column": int(h[1]), "ncols": int(h[2]),
                "iters": int(h[3]), "r_ii": float(f[4]), "tol": float(f[5]),
                "diag_max": float(f[6]), "diag_min": float(f[7])}

    def clear_code(self) -> None:
        """Forget a recorded outcome (keeps counters and diag stats)."""
        self.buf[0:2].zero_()
