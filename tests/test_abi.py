"""The C-ABI library builds for sm_100a, loads, and exports every entry point
declared in include/sketchgs_b200.h (no compute calls: no GPU here)."""

import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "sketchgs_b200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sgs_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = _declared()
    assert "sgs_rgs_update" in names and "sgs_ls_step" in names and "sgs_srht_partials" in names
    assert len(names) >= 25


def test_library_loads_and_exports_all_declared_symbols():
    from paper_2011_05090_b200 import _lib
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.sgs_abi_version() == 1
    # the ctypes binding covers every declared symbol
    assert set(_declared()) <= set(_lib.EXPORTED_SYMBOLS)


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_2011_05090_b200", "_lib", "libsketchgs_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_pure_host_queries_without_gpu():
    from paper_2011_05090_b200 import _lib
    lib = _lib.load()
    # deterministic partitioning is a pure function of the sizes
    assert lib.sgs_srht_nparts(1_000_000, 20) == lib.sgs_srht_nparts(1_000_000, 20) > 0
    assert lib.sgs_srht_nparts(24, 5) == 1
    assert lib.sgs_dense_nparts(100_000) == 296
    # Gaussian: 152 DMMA sub-chunks summed in clusters of 8 -> 19 partials
    assert lib.sgs_gaussian_nparts(100_000) == 19
    assert lib.sgs_gaussian_nparts(50) == 1
    assert 1 <= lib.sgs_ls_cluster_size(1500) <= 16
    if "SGS_LS_ROWS" not in os.environ and "SGS_LS_MAX_CLUSTER" not in os.environ:
        # ceil(k / 64) CTAs, at most 16 (the non-portable cluster limit)
        assert [lib.sgs_ls_cluster_size(k) for k in (1, 64, 65, 600, 1500, 3000)] == [1, 1, 2, 10, 16, 16]
    assert lib.sgs_ls_scratch_elems(1500, 501) > 0


def test_error_convention_without_gpu():
    # argument validation happens before any CUDA call: negative code + message
    from paper_2011_05090_b200 import _lib
    lib = _lib.load()
    rc = lib.sgs_srht_partials(None, 1, 10, 1, 10, 0, 4, None, None, 4, None, None, None)
    assert rc == -1
    assert b"null pointer" in lib.sgs_last_error()
    rc = lib.sgs_fwht(None, 6, 1, 6, None)
    assert rc == -1
    rc = lib.sgs_rgs_update(None, 0, 8, 8, 0, None, 0, None, 0, None, 8, None, None)
    assert rc == -1 and b"update" in lib.sgs_last_error()
    a = _lib.LsArgs()
    assert lib.sgs_ls_step(ctypes_byref(a), None) == -1
    assert b"ls_step" in lib.sgs_last_error()


def ctypes_byref(x):
    import ctypes
    return ctypes.byref(x)
