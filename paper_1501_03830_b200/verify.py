"""Size-independent verification on the GPU.

The reference checks a solution with ``residual_metrics`` (core.py:281-294),
which materialises the 2n x 2n H and Y; at n >= 16384 that is 256 GB.  The
north-star gates are per pair instead:

    max_j ||H x_j - lam_j x_j|| / (||H|| ||x_j||) <= 1e-13 n
    ||X1^T X1 - X2^T X2 - I||_F                    <= 1e-12 n

``pair_residuals_device`` evaluates both with two SYMMs and one GEMM of the
sm_100a library (C ABI ``bse_pair_residuals_dev``).  ``||H||`` is the caller's
choice; ``lam_max`` (a lower bound of ||H||_2) makes the ratio conservative.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import ptr, require_cuda, stream_ptr, to_device_colmajor
from .types import BseOperator, PositiveEigensystem


@dataclass(frozen=True)
class PairResidualReport:
    """Per-pair residual ratios (res_j / (h_norm * ||x_j||)) and the
    biorthogonality defect ||X1^T X1 - X2^T X2 - I||_F."""
    ratios: np.ndarray
    biorthogonality: float
    h_norm: float

    @property
    def max_ratio(self) -> float:
        return float(self.ratios.max()) if self.ratios.size else 0.0

    def passes(self, n: int) -> bool:
        return self.max_ratio <= 1e-13 * max(n, 1) and self.biorthogonality <= 1e-12 * max(n, 1)


def pair_residuals_device(n: int, Mt, ldm: int, Kt, ldk: int, lam, X1, ldx1: int, X2, ldx2: int):
    """Device call.  Column-major FP64 buffers (M, K lower triangles read).
    Returns torch tensors (res (n,), xnorm (n,), bio ())."""
    torch = require_cuda()
    lib = _lib.load()
    dev = Mt.device
    res = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    xn = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    bio = torch.zeros(1, dtype=torch.float64, device=dev)
    wb = int(lib.bse_residual_workspace_bytes(n))
    work = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
    st = lib.bse_pair_residuals_dev(n, ptr(Mt), ldm, ptr(Kt), ldk, ptr(lam), ptr(X1), ldx1,
                                    ptr(X2), ldx2, ptr(res), ptr(xn), ptr(bio), ptr(work), wb,
                                    stream_ptr(dev))
    if st != _lib.BSE_OK:
        raise RuntimeError(f"bse_pair_residuals_dev failed ({st}): {_lib.last_error()}")
    return res[:n], xn[:n], bio[0]


def pair_residual_report(op: BseOperator, pos: PositiveEigensystem,
                         h_norm: float | None = None) -> PairResidualReport:
    """Host-array front end for a real operator (kind 'real').  ``h_norm``
    defaults to lam_max, a lower bound of ||H||_2 (conservative ratio)."""
    if op.kind != "real":
        raise ValueError("pair_residual_report requires an operator of kind 'real'")
    torch = require_cuda()
    n = op.n
    dev = torch.device("cuda", torch.cuda.current_device())
    a, b = op.a.real, op.b.real
    Mt, ldm = to_device_colmajor(a + b, dev)
    Kt, ldk = to_device_colmajor(a - b, dev)
    X1, ld1 = to_device_colmajor(np.real(pos.x1), dev)
    X2, ld2 = to_device_colmajor(np.real(pos.x2), dev)
    lam = torch.from_numpy(np.array(pos.lambda_plus, dtype=np.float64)).to(dev)
    res, xn, bio = pair_residuals_device(n, Mt, ldm, Kt, ldk, lam, X1, ld1, X2, ld2)
    hn = float(pos.lambda_plus[0]) if h_norm is None else float(h_norm)
    ratios = (res / (hn * xn)).cpu().numpy()
    return PairResidualReport(ratios=ratios, biorthogonality=float(bio), h_norm=hn)


def complex_pair_residuals(A, B, lam, X1, X2):
    """Per-pair gates for a complex solution on the device (torch complex
    GEMMs; verification, not the solve path): returns (max_j |H x_j -
    lam_j x_j| / (lam_max |x_j|), |X1^H X1 - X2^H X2 - I|_F) with
    H = [[A, B], [-conj B, -conj A]] (core.py:235-242)."""
    torch = require_cuda()
    lamc = lam.to(torch.complex128)
    rt = A @ X1 + B @ X2 - X1 * lamc
    rb = -(B.conj() @ X1) - A.conj() @ X2 - X2 * lamc
    res = torch.sqrt((rt.abs() ** 2).sum(0) + (rb.abs() ** 2).sum(0))
    del rt, rb
    xn = torch.sqrt((X1.abs() ** 2).sum(0) + (X2.abs() ** 2).sum(0))
    G = X1.conj().T @ X1 - X2.conj().T @ X2
    G.diagonal().sub_(1.0)
    return float((res / (lam[0] * xn)).max()), float(torch.linalg.matrix_norm(G))


def solution_report(op: BseOperator, pos: PositiveEigensystem):
    """(max pair residual ratio, biorthogonality defect) of a host solution,
    for either kind (the per-pair form of core.residual_metrics)."""
    if op.kind == "real":
        rep = pair_residual_report(op, pos)
        return rep.max_ratio, rep.biorthogonality
    torch = require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    up = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
    return complex_pair_residuals(up(op.a), up(op.b), up(pos.lambda_plus), up(pos.x1),
                                  up(pos.x2))
