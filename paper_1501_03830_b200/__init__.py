"""B200-native (sm_100a) structure-preserving Bethe-Salpeter eigensolver.

Drop-in for the solver path of the reference package ``bse`` (bse-solver
0.1.0, pkg/src/bse/__init__.py:11-40): the same names and signatures for the
types, the structural transforms and the solvers, with the numerical core in
the CUDA library libbse_b200.so (C ABI: include/bse_b200.h).
"""
from .solvers import (hermitian_eigvals, real_embedding, solve_complex, solve_complex_device,
                      solve_oracle, solve_pair_device, solve_real, syevd_values_device,
                      tda_gap_report, validate)
from .spectra import absorption_device, absorption_spectrum
from .verify import PairResidualReport, pair_residual_report, pair_residuals_device
from .types import (BseOperator, ConvergenceError, DipoleData, FullEigensystem,
                    NotPositiveDefinite, PositiveEigensystem, SpectrumCurve, TdaGapReport,
                    ValidationReport,
                    assemble_h, build_m, conditioning_warnings, default_grid, dos_dominance,
                    expand_full, make_operator, residual_metrics)

__version__ = "0.1.0"

__all__ = [
    "BseOperator", "FullEigensystem", "PositiveEigensystem", "ValidationReport",
    "assemble_h", "make_operator", "residual_metrics", "build_m", "expand_full",
    "ConvergenceError", "NotPositiveDefinite", "solve_complex", "solve_real",
    "DipoleData", "SpectrumCurve", "absorption_spectrum", "default_grid", "dos_dominance",
    "conditioning_warnings", "real_embedding", "solve_complex_device", "solve_oracle",
    "solve_pair_device",
    "absorption_device", "hermitian_eigvals", "tda_gap_report", "TdaGapReport",
    "syevd_values_device", "PairResidualReport", "pair_residual_report",
    "pair_residuals_device", "validate", "__version__",
]
