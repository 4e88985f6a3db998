"""CPU oracle for the RGS / RGMRES hot path -- TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference package ``sketchgs``
(/root/reference/pkg/src/sketchgs, pure Python) for the functions on the hot
path, each citing the reference file:line it follows.  It is pinned against
golden vectors produced by running the reference itself in the build
container (``oracle/make_golden.py`` -> ``tests/golden/*.npz``) and against
the reference's own known-answer tests.

Only ``tests/``, ``__graft_entry__.smoke()`` and the CPU-baseline leg of
``bench.py`` may import this package, and only as the checker / the timed
CPU reference arm.  The product (``paper_2011_05090_b200``) never imports it.

Third-party arithmetic the reference relies on (not vendored, unpinned in
pkg/pyproject.toml:10-13): numpy Generator(Philox) for the sketch draws,
OpenBLAS ddot/dgemv, LAPACK dtrtrs via scipy.linalg.solve_triangular and
scipy's CSR matvec.  The oracle calls the same library functions in the same
order, so with single-threaded BLAS it reproduces the reference bit for bit
(checked by tests/test_oracle_golden.py).
"""

from .ref_sketch import OracleSketch, fwht_ref, psrht_setup
from .ref_rgs import OracleRgs, householder_lsq, oracle_certificates, oracle_rgs_factorize
from .ref_krylov import (OracleIlu0, csr_matvec, oracle_arnoldi, oracle_gmres, oracle_gmres_lagged,
                         oracle_gmres_restarted,
                         power_norm_estimate)
from .metrics import factor_metrics, factor_metrics_blocked, rel_diff
from .ref_cert import oracle_certify, oracle_epsilon_of, oracle_omega_bar
