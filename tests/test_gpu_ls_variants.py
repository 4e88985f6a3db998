"""The LS kernel's compiled-out variants and the column kernels' prefetch
switches must not change a bit of the factors.

`ls_step_kernel<T, PLAIN, MODE>` (csrc/sgs_rgs.cu) is the same code with the
one-synchronisation / peer / Givens branches compiled out (PLAIN) and the
launch mode fixed at compile time (MODE: fused, finalize-only, solve-only; no
stamps); which one runs is a per-launch choice (SGS_LS_PLAIN=0: always the
full kernel, 1: PLAIN only, default: all specialisations).  The column kernels'
pre-wait L2 prefetch (SGS_COL_PF_MB / SGS_DENSE_PF_MB = 0: off, SGS_COL_PF_PACE
= 0: one burst) only moves bytes.  The switches are read once per process, so
each setting runs tools/ls_variant_probe.py in a fresh process; the probe
prints SHA-256 digests of Q, R, S for batch and streaming factorisations
(reference path: gram_schmidt.py:283-375)."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _probe(**env):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ls_variant_probe.py")],
                         env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, (out.stdout + out.stderr)[-3000:]
    assert "LS_VARIANT_PROBE_DONE" in out.stdout
    return [ln for ln in out.stdout.splitlines() if ln.startswith(("batch", "push"))]


def test_ls_variants_and_prefetch_switches_are_bit_identical(cuda):
    base = _probe()
    assert len(base) == 8
    assert _probe(SGS_LS_PLAIN="0") == base          # full kernel everywhere
    assert _probe(SGS_LS_PLAIN="1") == base          # PLAIN without the MODE variants
    assert _probe(SGS_COL_PF_MB="0", SGS_DENSE_PF_MB="0") == base   # no prefetch
    assert _probe(SGS_COL_PF_PACE="0") == base       # burst prefetch
