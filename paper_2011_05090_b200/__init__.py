"""B200-native randomized Gram-Schmidt (RGS) and randomized GMRES.

Drop-in for the hot path of the reference package ``sketchgs``
(Balabanov & Grigori, arXiv 2011.05090): the same entry points and
sketch-operator interface (``sketchgs/__init__.py:5-26``), executed by
hand-written sm_100a kernels behind the C ABI of ``include/sketchgs_b200.h``.
There is no CPU fallback: compute entry points raise without the built
library and a CUDA device.
"""

from .precision import (MIXED32_64, U_BINARY32, U_BINARY64, UNIFIED32, UNIFIED64,
                        PrecisionPolicy, policy_from_name)
from .sketch import SketchKind, SketchOperator, as_device_sketch, block_seed, fwht, make_sketch
from .gram_schmidt import (BREAKDOWN_FACTOR, HOUSEHOLDER_QR, BreakdownError, GsVariant,
                           LsqSolver, QrFactors, RgsState, StabilityCertificate, certificates,
                           loss_of_orthogonality, rgs_factorize, sketched_lsq)
from .krylov import (ArnoldiDecomposition, GmresResult, Ilu0Preconditioner, RestartedResult,
                     SparseMatrix, arnoldi, gmres, gmres_restarted, ilu0)
from .mmio import MatrixMarketError, read_matrix_market, write_matrix_market
from .certification import (CertificationParams, CertificationResult, EmbeddingParams,
                            certify_factorization, epsilon_of, eps_star_for_dim,
                            make_certification_sketch, omega_bar, omega_bar_sharpness,
                            required_sketch_dim, rounding_sketch_trial, vector_certificate_dim)

__version__ = "0.1.0"

__all__ = [
    "MIXED32_64", "U_BINARY32", "U_BINARY64", "UNIFIED32", "UNIFIED64", "PrecisionPolicy",
    "policy_from_name", "SketchKind", "SketchOperator", "as_device_sketch", "block_seed", "fwht",
    "make_sketch", "BREAKDOWN_FACTOR", "HOUSEHOLDER_QR", "BreakdownError", "GsVariant",
    "LsqSolver", "QrFactors", "RgsState", "StabilityCertificate", "certificates",
    "loss_of_orthogonality", "rgs_factorize", "sketched_lsq", "ArnoldiDecomposition", "GmresResult",
    "RestartedResult", "SparseMatrix", "Ilu0Preconditioner", "ilu0", "arnoldi", "gmres",
    "gmres_restarted", "CertificationParams", "CertificationResult", "EmbeddingParams",
    "certify_factorization", "epsilon_of", "eps_star_for_dim", "make_certification_sketch",
    "omega_bar", "omega_bar_sharpness", "required_sketch_dim", "rounding_sketch_trial",
    "vector_certificate_dim", "MatrixMarketError", "read_matrix_market", "write_matrix_market",
]
