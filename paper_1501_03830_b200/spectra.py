"""Absorption spectrum on the GPU (reference: spectra.py:120-151).

    eps+(omega) = sum_j Re[(d_r^H x_j)(y_j^H d_l) / (y_j^H x_j)] N(omega - lambda_j; sigma)

computed by bse_absorption_dev: one warp per eigenpair for the projections,
one thread per grid point for the truncated (8 sigma) Gaussians accumulated
in eigenvalue order.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .device import ptr, require_cuda, stream_ptr
from .types import (DEFAULT_SIGMA, DipoleData, PositiveEigensystem, SpectrumCurve,
                    default_grid)


def absorption_device(lam, X1c, X2c, d_r, d_l, grid, sigma):
    """Device call.  lam (n,) float64; X1c, X2c complex128 tensors of shape
    (n, ld) holding the COLUMNS of X1, X2 as rows; d_r, d_l complex128 (2n,);
    grid float64.  Returns (values, weights, defect, min|pairing|) tensors."""
    torch = require_cuda()
    n = lam.shape[0]
    dev = lam.device
    weights = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    values = torch.empty(max(grid.shape[0], 1), dtype=torch.float64, device=dev)
    scal = torch.empty(2, dtype=torch.float64, device=dev)
    st = _lib.load().bse_absorption_dev(n, ptr(lam), ptr(X1c), X1c.shape[1], ptr(X2c),
                                        X2c.shape[1], ptr(d_r), ptr(d_l), grid.shape[0], ptr(grid),
                                        float(sigma), ptr(weights), ptr(values), ptr(scal),
                                        ptr(scal) + 8, stream_ptr(dev))
    if st != _lib.BSE_OK:
        raise RuntimeError(f"bse_absorption_dev failed: {_lib.last_error()}")
    return values[:grid.shape[0]], weights[:n], scal[0], scal[1]


def absorption_spectrum(pos: PositiveEigensystem, dip: DipoleData, grid=None,
                        sigma: float = DEFAULT_SIGMA) -> SpectrumCurve:
    """Drop-in for spectra.absorption_spectrum (same checks and messages)."""
    if not sigma > 0.0:
        raise ValueError("sigma must be positive")
    n = pos.n
    if dip.d_r.shape[0] != 2 * n:
        raise ValueError(f"dipole vectors must have length {2 * n}")
    torch = require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    if grid is None:
        grid = default_grid(pos.lambda_plus, sigma)
    grid = np.asarray(grid, dtype=np.float64)
    lam = torch.from_numpy(np.array(pos.lambda_plus)).to(dev)
    X1c = torch.from_numpy(np.array(pos.x1.T, order="C")).to(dev)
    X2c = torch.from_numpy(np.array(pos.x2.T, order="C")).to(dev)
    dr = torch.from_numpy(np.array(dip.d_r)).to(dev)
    dl = torch.from_numpy(np.array(dip.d_l)).to(dev)
    g = torch.from_numpy(np.ascontiguousarray(grid)).to(dev)
    values, _, defect, minpair = absorption_device(lam, X1c, X2c, dr, dl, g, sigma)
    if n and float(minpair) < 1e-8:
        raise ValueError("invalid eigensystem: |y_j^H x_j| below 1e-8")
    return SpectrumCurve(omegas=grid, values=values.cpu().numpy(), sigma=float(sigma),
                         kind="absorption", normalization_defect=float(defect) if n else 0.0)


def spectral_density(lam, grid=None, sigma: float = DEFAULT_SIGMA) -> SpectrumCurve:
    """Broadened density of states phi(omega) = (1/N) sum_j N(omega -
    lambda_j; sigma) over all supplied eigenvalues (reference:
    spectra.spectral_density, spectra.py:99-117).  O(N x window) host
    post-processing of eigenvalues already on the host (no eigenvectors)."""
    lam = np.atleast_1d(np.asarray(lam, dtype=np.float64))
    if lam.size == 0:
        raise ValueError("empty spectrum")
    if not sigma > 0.0:
        raise ValueError("sigma must be positive")
    if grid is None:
        grid = default_grid(lam, sigma)
    grid = np.asarray(grid, dtype=np.float64)
    out = np.zeros(grid.shape[0])
    wpeak = (1.0 / lam.shape[0]) * (1.0 / (np.sqrt(2.0 * np.pi) * sigma))  # (w * peak)
    reach = 8.0 * sigma
    for c in lam:  # accumulated in eigenvalue order, truncated at 8 sigma (spectra.py:81-96)
        i0 = int(np.searchsorted(grid, c - reach, side="left"))
        i1 = int(np.searchsorted(grid, c + reach, side="right"))
        if i0 == i1:
            continue
        t = (grid[i0:i1] - c) / sigma
        out[i0:i1] += wpeak * np.exp(-0.5 * t * t)
    return SpectrumCurve(omegas=grid, values=out, sigma=float(sigma), kind="dos")
