"""Containers and structural transforms of the drop-in API.

Field-compatible with the reference's types (pkg/src/bse/core.py:45-200,
embeddings.py:62-149, spectra.py:25-70): frozen dataclasses holding read-only
numpy arrays, with the same validation rules and error messages.  These are
host-side plumbing; the eigensolve itself runs in the CUDA library.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

EPS = float(np.finfo(np.float64).eps)
SYM_RTOL = 100.0 * EPS          # core.py:23
CONDITION_WARN_RATIO = 1e-8     # solvers.py:24
DEFAULT_SIGMA = 5e-4            # spectra.py:17
DEFAULT_GRID_POINTS = 2001      # spectra.py:20


class NotPositiveDefinite(ArithmeticError):
    """Cholesky pivot breakdown (kernels.py:25-32)."""

    def __init__(self, pivot_index: int, pivot_value: float, what: str = "matrix"):
        super().__init__(f"{what} is not positive definite: "
                         f"pivot {pivot_value:.6e} at index {pivot_index}")
        self.pivot_index = pivot_index
        self.pivot_value = pivot_value


class ConvergenceError(RuntimeError):
    """An iterative kernel exhausted its retry budget (kernels.py:35-36)."""


def _frob(x) -> float:
    return float(np.linalg.norm(x))


def _readonly(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x)
    x.setflags(write=False)
    return x


@dataclass(frozen=True)
class BseOperator:
    """(A, B), A Hermitian, B symmetric; complex128, read-only (core.py:45-75)."""

    a: np.ndarray
    b: np.ndarray
    kind: str

    def __post_init__(self):
        a = np.asarray(self.a, dtype=np.complex128)
        b = np.asarray(self.b, dtype=np.complex128)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ValueError(f"A must be square, got shape {a.shape}")
        if b.shape != a.shape:
            raise ValueError(f"A and B shapes differ: {a.shape} vs {b.shape}")
        if self.kind not in ("real", "complex"):
            raise ValueError(f"kind must be 'real' or 'complex', got {self.kind!r}")
        if not (np.isfinite(a).all() and np.isfinite(b).all()):
            raise ValueError("A and B must contain only finite entries")
        if self.kind == "real" and (np.any(a.imag != 0.0) or np.any(b.imag != 0.0)):
            raise ValueError("kind='real' requires exactly zero imaginary parts")
        object.__setattr__(self, "a", _readonly(a))
        object.__setattr__(self, "b", _readonly(b))

    @property
    def n(self) -> int:
        return self.a.shape[0]


def make_operator(a, b, kind: str | None = None, symmetrize: bool = False,
                  tol: float | None = None) -> BseOperator:
    """Validated BseOperator (core.py:78-120)."""
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    if not (np.isfinite(a).all() and np.isfinite(b).all()):
        raise ValueError("A and B must contain only finite entries")
    if symmetrize:
        a = 0.5 * (a + a.conj().T)
        b = 0.5 * (b + b.T)
    rtol = SYM_RTOL if tol is None else float(tol)
    for name, mat, conj in (("A", a, True), ("B", b, False)):
        nrm = _frob(mat)
        defect = _frob(mat - (mat.conj().T if conj else mat.T))
        if defect > rtol * max(1.0, nrm):
            raise ValueError(
                f"{name} violates {'Hermitian' if conj else 'symmetric'} structure: "
                f"defect {defect:.3e} exceeds tolerance {rtol * max(1.0, nrm):.3e}; "
                f"pass symmetrize=True to average it away")
    if kind is None:
        kind = "real" if (np.all(a.imag == 0.0) and np.all(b.imag == 0.0)) else "complex"
    if kind == "real" and (np.any(a.imag != 0.0) or np.any(b.imag != 0.0)):
        raise ValueError("kind='real' requested but inputs have nonzero imaginary parts")
    return BseOperator(a=a, b=b, kind=kind)


@dataclass(frozen=True)
class ValidationReport:
    """core.py:123-139."""

    symmetry_ok: bool
    definiteness_ok: bool
    sym_defects: tuple[float, float]
    margin: float

    @property
    def ok(self) -> bool:
        return self.symmetry_ok and self.definiteness_ok


@dataclass(frozen=True)
class PositiveEigensystem:
    """lambda_1 >= ... >= lambda_n > 0 with X1^H X1 - X2^H X2 = I (core.py:142-169)."""

    lambda_plus: np.ndarray
    x1: np.ndarray
    x2: np.ndarray
    warnings: tuple[str, ...] = ()

    def __post_init__(self):
        lam = np.asarray(self.lambda_plus, dtype=np.float64)
        x1 = np.asarray(self.x1, dtype=np.complex128)
        x2 = np.asarray(self.x2, dtype=np.complex128)
        n = lam.shape[0]
        if x1.shape != (n, n) or x2.shape != (n, n):
            raise ValueError("eigenvector blocks must be n x n")
        if n and not np.all(lam > 0.0):
            raise ValueError("all eigenvalues must be strictly positive")
        if n > 1 and np.any(np.diff(lam) > 0.0):
            raise ValueError("eigenvalues must be sorted in descending order")
        object.__setattr__(self, "lambda_plus", _readonly(lam))
        object.__setattr__(self, "x1", _readonly(x1))
        object.__setattr__(self, "x2", _readonly(x2))

    @property
    def n(self) -> int:
        return self.lambda_plus.shape[0]


@dataclass(frozen=True)
class FullEigensystem:
    """All 2n eigenpairs; lam[n:] is the bitwise negation of lam[:n] (core.py:172-200)."""

    x: np.ndarray
    y: np.ndarray
    lam: np.ndarray

    def __post_init__(self):
        x = np.asarray(self.x, dtype=np.complex128)
        y = np.asarray(self.y, dtype=np.complex128)
        lam = np.asarray(self.lam, dtype=np.float64)
        m = lam.shape[0]
        if m % 2 != 0:
            raise ValueError("eigenvalue count must be even")
        if x.shape != (m, m) or y.shape != (m, m):
            raise ValueError("X and Y must be 2n x 2n")
        n = m // 2
        if m and not np.array_equal(lam[n:], -lam[:n]):
            raise ValueError("lambda[n:] must be the exact negation of lambda[:n]")
        object.__setattr__(self, "x", _readonly(x))
        object.__setattr__(self, "y", _readonly(y))
        object.__setattr__(self, "lam", _readonly(lam))

    @property
    def n(self) -> int:
        return self.lam.shape[0] // 2


@dataclass(frozen=True)
class TdaGapReport:
    """solvers.py:136-146."""

    gaps: np.ndarray
    max_relative_gap: float
    min_gap: float
    scale: float
    certified: bool


def build_m(op: BseOperator) -> np.ndarray:
    """M = [[Re(A+B), Im(A-B)], [-Im(A+B), Re(A-B)]], bitwise symmetric
    (embeddings.py:62-74)."""
    apb = op.a + op.b
    amb = op.a - op.b
    m = np.block([[apb.real, amb.imag], [-apb.imag, amb.real]])
    return 0.5 * (m + m.T)


def assemble_h(op: BseOperator) -> np.ndarray:
    """Dense H = [[A, B], [-conj B, -conj A]] (core.py:235-242); checks only."""
    return np.block([[op.a, op.b], [-op.b.conj(), -op.a.conj()]])


def expand_full(op: BseOperator, pos: PositiveEigensystem) -> FullEigensystem:
    """X = [[X1, conj X2], [X2, conj X1]], Y = [[X1, -conj X2], [-X2, conj X1]],
    lam = (lam+, -lam+) (embeddings.py:133-149)."""
    if pos.n != op.n:
        raise ValueError(f"dimension mismatch: operator n={op.n}, eigensystem n={pos.n}")
    x1, x2 = pos.x1, pos.x2
    x = np.block([[x1, x2.conj()], [x2, x1.conj()]])
    y = np.block([[x1, -x2.conj()], [-x2, x1.conj()]])
    lam = np.concatenate([pos.lambda_plus, -pos.lambda_plus])
    return FullEigensystem(x=x, y=y, lam=lam)


def residual_metrics(op: BseOperator, full: FullEigensystem) -> tuple[float, float]:
    """r1 = |Y^H H X - Lambda|_F/|H|_F, r2 = |Y^H X - I|_F/sqrt(2n) (core.py:281-294).
    Verification helper (host numpy); not on the solve path."""
    if full.n != op.n:
        raise ValueError(f"dimension mismatch: operator n={op.n}, eigensystem n={full.n}")
    h = assemble_h(op)
    m = 2 * op.n
    yh = full.y.conj().T
    r1 = _frob(yh @ (h @ full.x) - np.diag(full.lam)) / _frob(h)
    r2 = _frob(yh @ full.x - np.eye(m)) / np.sqrt(m)
    return float(r1), float(r2)


def conditioning_warnings(lam: np.ndarray) -> tuple[str, ...]:
    """solvers.py:163-168."""
    if lam.size and lam[-1] < CONDITION_WARN_RATIO * lam[0]:
        return (f"ill conditioned: smallest eigenvalue {lam[-1]:.3e} is below "
                f"{CONDITION_WARN_RATIO:g} of the largest {lam[0]:.3e}; the "
                f"Lambda^(-1/2) normalization amplifies rounding errors",)
    return ()


@dataclass(frozen=True)
class SpectrumCurve:
    """spectra.py:25-52."""

    omegas: np.ndarray
    values: np.ndarray
    sigma: float
    kind: str
    normalization_defect: float | None = None

    def __post_init__(self):
        omegas = np.asarray(self.omegas, dtype=np.float64)
        values = np.asarray(self.values, dtype=np.float64)
        if omegas.shape != values.shape or omegas.ndim != 1:
            raise ValueError("omegas and values must be 1-D of equal length")
        if omegas.size > 1 and not np.all(np.diff(omegas) > 0.0):
            raise ValueError("omegas must be strictly increasing")
        if not self.sigma > 0.0:
            raise ValueError("sigma must be positive")
        if self.kind not in ("dos", "absorption"):
            raise ValueError("kind must be 'dos' or 'absorption'")
        object.__setattr__(self, "omegas", _readonly(omegas))
        object.__setattr__(self, "values", _readonly(values))


@dataclass(frozen=True)
class DipoleData:
    """Right and left dipole vectors of length 2n (spectra.py:55-70)."""

    d_r: np.ndarray
    d_l: np.ndarray

    def __post_init__(self):
        d_r = np.asarray(self.d_r, dtype=np.complex128)
        d_l = np.asarray(self.d_l, dtype=np.complex128)
        if d_r.ndim != 1 or d_r.shape != d_l.shape:
            raise ValueError("dipole vectors must be 1-D of equal length")
        if not (np.isfinite(d_r).all() and np.isfinite(d_l).all()):
            raise ValueError("dipole vectors must be finite")
        object.__setattr__(self, "d_r", _readonly(d_r))
        object.__setattr__(self, "d_l", _readonly(d_l))


def default_grid(lam: np.ndarray, sigma: float, points: int = DEFAULT_GRID_POINTS) -> np.ndarray:
    """[min lam - 10 sigma, max lam + 10 sigma] (spectra.py:73-78)."""
    lam = np.asarray(lam, dtype=np.float64)
    return np.linspace(float(np.min(lam)) - 10.0 * sigma, float(np.max(lam)) + 10.0 * sigma,
                       points)


def dos_dominance(lambda_h: np.ndarray, lambda_a: np.ndarray) -> bool:
    """lambda_j(A) >= lambda_j(H) - 1e-12 scale, index by index (spectra.py:154-167)."""
    lambda_h = np.asarray(lambda_h, dtype=np.float64)
    lambda_a = np.asarray(lambda_a, dtype=np.float64)
    if lambda_h.shape != lambda_a.shape:
        raise ValueError("spectra must have equal length")
    if lambda_h.size == 0:
        return True
    scale = max(float(np.max(np.abs(lambda_h))), float(np.max(np.abs(lambda_a))))
    return bool(np.all(lambda_a >= lambda_h - 1e-12 * scale))
