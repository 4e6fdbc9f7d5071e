import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200, sm_100a) device")


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture
def dev():
    if not cuda_available():
        pytest.skip("no CUDA device")
    import torch
    return torch.device("cuda:0")


# Seeded generators with the same recipes as the reference suite's conftest
# (pkg/tests/conftest.py:5-32) -- restated here, not imported.
def random_hermitian(n, seed):
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    return 0.5 * (g + g.conj().T)


def random_symmetric(n, seed):
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, n))
    return 0.5 * (g + g.T)


def random_spd_real(n, seed):
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, n))
    return g @ g.T + n * np.eye(n)


def random_rotation(n, seed):
    q, r = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, n)))
    return q * np.sign(np.diagonal(r))


# ---------------------------------------------------------------------------
# SURVEY 8c parity procedure (steps 3-5): eigenvectors equal up to a unit
# phase for isolated eigenvalues, within n eps |W| / gap_j(lambda^2); for
# clusters, principal angles between the spans against the same bound with
# the gap to the rest of the spectrum.  |W| = lambda_1^2 (W = L^T M L).
EPS = float(np.finfo(np.float64).eps)


def principal_angle(x_new, x_ref):
    """Largest principal angle between span(x_new) and span(x_ref), from its
    sine |(I - Qa Qa^H) Qb|_2 (arccos of the cosines loses half the digits
    near 0: arccos(1 - eps) ~ 2e-8)."""
    qa, _ = np.linalg.qr(x_new)
    qb, _ = np.linalg.qr(x_ref)
    r = qb - qa @ (qa.conj().T @ qb)
    return float(np.arcsin(min(1.0, np.linalg.norm(r, 2))))


def vector_parity(lam, x_new, x_ref, n_scale, cluster_rtol=None, factor=1.0):
    """Assert the 8c(4)/(5) gates; returns (worst singleton ratio err/tol,
    worst cluster ratio) for reporting.  lam descending (positive); columns of
    x_* are the 2n-vectors [x1; x2]."""
    lam = np.asarray(lam, dtype=np.float64)
    l2 = lam ** 2
    wn = l2[0]
    if cluster_rtol is None:
        cluster_rtol = 1e3 * n_scale * EPS
    # clusters in lambda^2 (relative to |W|)
    groups, i = [], 0
    while i < l2.shape[0]:
        j = i + 1
        while j < l2.shape[0] and l2[j - 1] - l2[j] <= cluster_rtol * wn:
            j += 1
        groups.append((i, j))
        i = j
    worst_s = worst_c = 0.0
    for gi, (i, j) in enumerate(groups):
        left = l2[groups[gi - 1][1] - 1] - l2[i] if gi > 0 else np.inf
        right = l2[j - 1] - l2[groups[gi + 1][0]] if gi + 1 < len(groups) else np.inf
        gap = max(min(left, right), 1e-300)
        tol = factor * n_scale * EPS * wn / gap
        if j - i == 1:
            a, b = x_ref[:, i], x_new[:, i]
            c = np.vdot(a, b)
            c = c / abs(c) if abs(c) > 0 else 1.0
            err = np.linalg.norm(b - c * a) / np.linalg.norm(a)
            assert err <= max(tol, 1e-13), ("singleton", i, err, tol)
            worst_s = max(worst_s, err / tol)
        else:
            ang = principal_angle(x_new[:, i:j], x_ref[:, i:j])
            assert ang <= max(tol, 1e-13), ("cluster", i, j, ang, tol)
            worst_c = max(worst_c, ang / tol)
    return worst_s, worst_c


def lapack_solution(m, k):
    """Independent LAPACK route for a real pair (M, K): K = L L^T,
    W = L^T M L = Z Lam^2 Z^T, X1,2 = (L Z +- L^-T Z Lam) Lam^-1/2 / 2."""
    low = np.linalg.cholesky(k)
    w = low.T @ m @ low
    l2, z = np.linalg.eigh(0.5 * (w + w.T))
    l2, z = l2[::-1], z[:, ::-1]
    lam = np.sqrt(l2)
    u = low @ z
    v = np.linalg.solve(low.T, z * lam)
    sc = 0.5 / np.sqrt(lam)
    return lam, (u + v) * sc, (u - v) * sc
