"""The checked build (compute-sanitizer memcheck stand-in: this GPU pool does
not run compute-sanitizer).  `make checked` compiles every kernel with
SGS_DEVICE_CHECKS: shared-memory carve-ups against the launch's dynamic
shared-memory size, sample rows against their block, CSR ranges, LS slices
and column indices (SGS_DCHECK traps with its location).  A workload that
runs every kernel family (tools/sanitize_small.py: the fused SRHT column
kernel with its TMA ring and DSMEM sum, the LS cluster kernel, the tile /
DMMA / Rademacher sketches, the dense ring kernel, SpMV, standard and
one-synchronisation Arnoldi, ILU(0)) must finish without a trap, in a fresh
process that loads the checked library."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

CHECKED = os.path.join(ROOT, "paper_2011_05090_b200", "_lib", "libsketchgs_b200_checked.so")


def test_checked_build_runs_every_kernel_family_without_a_trap(cuda):
    assert os.path.exists(CHECKED), "checked build missing: make -C paper_2011_05090_b200/csrc checked"
    env = dict(os.environ, SGS_LIB_CHECKED="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_small.py")],
                         env=env, capture_output=True, text=True, timeout=900)
    log = out.stdout + out.stderr
    assert "SGS_DCHECK failed" not in log, log[-4000:]
    assert out.returncode == 0, log[-4000:]
    assert "SANITIZE_WORKLOAD_DONE" in out.stdout
    assert "libsketchgs_b200_checked.so" in out.stdout  # the checked library ran it
