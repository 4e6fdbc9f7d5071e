"""Drop-in solver API: ``solve_real`` / ``solve_complex`` with the reference's
signatures (pkg/src/bse/solvers.py:29, :80), backed by the sm_100a library.

Both run the north-star product form on the GPU: M = A+B, K = A-B (or their
2n x 2n real embedding for complex operators, D3), K = L L^T,
W = L^T M L = Z Lam^2 Z^T, X1,2 = (L Z +- L^{-T} Z Lam) Lam^{-1/2} / 2.
Torch is used for device memory, streams and index plumbing only; every
floating-point stage (Cholesky, congruence, eigensolver, back-transforms,
recovery, complex extraction, absorption) is a kernel of libbse_b200.so.  There is no CPU fallback: without a CUDA device these raise.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .device import (colmajor_empty, download_complex, ptr, require_cuda, stream_ptr,
                     to_device_colmajor, upload_rowmajor, view_colmajor)
from .types import (BseOperator, ConvergenceError, NotPositiveDefinite,
                    PositiveEigensystem, conditioning_warnings)

_WHAT_M = "the definiteness embedding M"


def _gemm(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, Cm, ldc):
    st = _lib.load().bse_gemm_dev(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, Cm, ldc, None,
                                  stream_ptr())
    if st != _lib.BSE_OK:
        raise RuntimeError(f"bse_gemm_dev failed: {_lib.last_error()}")


def solve_pair_device(Mt, ldm: int, Kt, ldk: int, n: int, flags: int = 0):
    """Core device call (C ABI bse_solve_spd_pair_dev).  Mt, Kt: column-major
    FP64 device buffers (lower triangles read).  Returns torch tensors
    (lam descending (n,), X1 buffer, X2 buffer, ld) or raises
    NotPositiveDefinite with (pivot_index, pivot_value, failed_factor)."""
    torch = require_cuda()
    lib = _lib.load()
    dev = Mt.device
    X1, ld = colmajor_empty(n, n, dev)
    X2, _ = colmajor_empty(n, n, dev)
    lam = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    wb = lib.bse_solve_workspace_bytes(n, flags)
    work = torch.empty(max(int(wb), 1), dtype=torch.uint8, device=dev)
    info = _lib.BseInfo()
    st = lib.bse_solve_spd_pair_dev(n, ptr(Mt), ldm, ptr(Kt), ldk, ptr(lam), ptr(X1), ld,
                                    ptr(X2), ld, ptr(work), wb, flags, stream_ptr(dev),
                                    C.byref(info))
    raise_for_status(st, info, "bse_solve_spd_pair_dev")
    return lam[:n], X1, X2, ld


def raise_for_status(st: int, info, where: str) -> None:
    """Map a C-ABI status to the reference's exceptions (kernels.py:25-36,
    core.py:159-160): 1 -> NotPositiveDefinite("A+B" | "A-B"), 2 ->
    ConvergenceError, 3 and 5 -> ValueError, 4 -> RuntimeError."""
    if st == _lib.BSE_OK:
        return
    if st == _lib.BSE_NOT_POSITIVE_DEFINITE:
        err = NotPositiveDefinite(int(info.pivot_index), float(info.pivot_value),
                                  "A+B" if info.failed_factor == 1 else "A-B")
        err.failed_factor = int(info.failed_factor)
        raise err
    if st == _lib.BSE_NO_CONVERGENCE:
        raise ConvergenceError(f"{where}: {_lib.last_error()}")
    if st == _lib.BSE_SPECTRUM_NOT_POSITIVE:
        raise ValueError("all eigenvalues must be strictly positive")
    if st == _lib.BSE_BAD_ARGUMENT:
        raise ValueError(f"{where}: {_lib.last_error()}")
    raise RuntimeError(f"{where} failed ({st}): {_lib.last_error()}")


def _device():
    torch = require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _real_pair(op: BseOperator):
    a = op.a.real
    b = op.b.real
    return a + b, a - b


def solve_real(op: BseOperator) -> PositiveEigensystem:
    """Real product-form solve (reference: solvers.py:80-109).  Raises
    NotPositiveDefinite naming "A+B" or "A-B" like the reference."""
    if op.kind != "real":
        raise ValueError("solve_real requires an operator of kind 'real'")
    n = op.n
    if n == 0:
        return PositiveEigensystem(lambda_plus=np.zeros(0), x1=np.zeros((0, 0)), x2=np.zeros((0, 0)))
    lam_h, x1, x2 = _solve_real_pair(op)
    return PositiveEigensystem(lambda_plus=lam_h, x1=x1, x2=x2,
                               warnings=conditioning_warnings(lam_h))


def _solve_real_pair(op: BseOperator):
    """(lam, X1, X2 complex128 C-order) of the real product form: M = A+B,
    K = A-B uploaded through the staging ring (lower triangles read, as the
    reference's cholesky), the device solve, X transposed and widened to
    complex128 on the device and downloaded through the staging ring."""
    torch = require_cuda()
    n = op.n
    dev = _device()
    # the operator's complex128 blocks go up as stored (staging ring); the real
    # parts, A+B / A-B and the column-major layout are formed on the device
    A = upload_rowmajor(op.a, dev)
    B = upload_rowmajor(op.b, dev)
    ar, br = torch.view_as_real(A)[..., 0], torch.view_as_real(B)[..., 0]
    Mt, ldm = colmajor_empty(n, n, dev, zero=True)
    Kt, ldk = colmajor_empty(n, n, dev, zero=True)
    view_colmajor(Mt, n, n).copy_(ar + br)
    view_colmajor(Kt, n, n).copy_(ar - br)
    del A, B, ar, br
    lam, X1, X2, _ = solve_pair_device(Mt, ldm, Kt, ldk, n)
    del Mt, Kt
    lam_h = lam.cpu().numpy()
    return lam_h, download_complex(X1, n, n), download_complex(X2, n, n)


def real_embedding(op: BseOperator):
    """Real 2n x 2n BSE pair of a complex operator (D3):
    A' = [[Ar, -Ai], [Ai, Ar]], B' = [[Br, Bi], [Bi, -Br]];
    M' = A'+B' = S build_m S, K' = A'-B' = S P build_m P S (S = diag(I,-I),
    P the block swap), so definiteness pivots coincide with build_m's."""
    ar, ai = op.a.real, op.a.imag
    br, bi = op.b.real, op.b.imag
    ap = np.block([[ar, -ai], [ai, ar]])
    bp = np.block([[br, bi], [bi, -br]])
    m = ap + bp
    k = ap - bp
    return 0.5 * (m + m.T), 0.5 * (k + k.T)


def solve_complex_device(A, B, n: int, flags: int = 0):
    """Core device call (C ABI bse_solve_complex_dev) on torch complex128
    tensors A, B (n x n, row-major = torch's layout).  Returns torch tensors
    (lam descending (n,), X1, X2 (n x n complex128)) or raises like the
    reference (NotPositiveDefinite names the definiteness embedding M)."""
    torch = require_cuda()
    lib = _lib.load()
    dev = A.device
    A = A.contiguous()
    B = B.contiguous()
    X1 = torch.empty((n, n), dtype=torch.complex128, device=dev)
    X2 = torch.empty((n, n), dtype=torch.complex128, device=dev)
    lam = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    wb = lib.bse_solve_complex_workspace_bytes(n, flags)
    work = torch.empty(max(int(wb), 1), dtype=torch.uint8, device=dev)
    info = _lib.BseInfo()
    st = lib.bse_solve_complex_dev(n, ptr(A), n, ptr(B), n, ptr(lam), ptr(X1), n, ptr(X2), n,
                                   ptr(work), wb, flags, stream_ptr(dev), C.byref(info))
    if st == _lib.BSE_NOT_POSITIVE_DEFINITE:
        raise NotPositiveDefinite(int(info.pivot_index), float(info.pivot_value), _WHAT_M)
    raise_for_status(st, info, "bse_solve_complex_dev")
    return lam[:n], X1, X2


def _solve_complex_host(a: np.ndarray, b: np.ndarray, n: int, flags: int = 0):
    """Host entry (bse_solve_complex_host): numpy complex128 in, numpy out;
    uploads, the solve and the downloads happen inside the library."""
    require_cuda()
    lib = _lib.load()
    a = np.ascontiguousarray(a, dtype=np.complex128)
    b = np.ascontiguousarray(b, dtype=np.complex128)
    lam = np.empty(n)
    x1 = np.empty((n, n), dtype=np.complex128)
    x2 = np.empty((n, n), dtype=np.complex128)
    info = _lib.BseInfo()
    st = lib.bse_solve_complex_host(n, a.ctypes.data, n, b.ctypes.data, n, lam.ctypes.data,
                                    x1.ctypes.data, n, x2.ctypes.data, n, flags, C.byref(info))
    if st == _lib.BSE_NOT_POSITIVE_DEFINITE:
        raise NotPositiveDefinite(int(info.pivot_index), float(info.pivot_value), _WHAT_M)
    raise_for_status(st, info, "bse_solve_complex_host")
    return lam, x1, x2


def syevd_values_device(At, lda: int, n: int):
    """Ascending eigenvalues of the symmetric matrix in At (lower triangle,
    destroyed) via bse_syevd_dev(BSE_FLAG_VALUES_ONLY): SY2SB + SB2ST + Sturm
    bisection, no back-transforms."""
    torch = require_cuda()
    lib = _lib.load()
    dev = At.device
    w = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    wb = lib.bse_syevd_workspace_bytes(n, _lib.FLAG_VALUES_ONLY)
    work = torch.empty(max(int(wb), 1), dtype=torch.uint8, device=dev)
    st = lib.bse_syevd_dev(n, ptr(At), lda, ptr(w), 0, n, ptr(work), wb, _lib.FLAG_VALUES_ONLY,
                           stream_ptr(dev))
    raise_for_status(st, None, "bse_syevd_dev")
    return w[:n]


def hermitian_eigvals(a) -> np.ndarray:
    """Eigenvalues (descending) of a Hermitian matrix on the GPU.  Complex
    input goes through the real doubling embedding [[Re A, Im A], [-Im A, Re A]]
    whose spectrum is A's with every eigenvalue doubled (reference:
    kernels.hermitian_eig, kernels.py:616-641, values only)."""
    a = np.asarray(a, dtype=np.complex128)
    n = a.shape[0]
    if n == 0:
        return np.zeros(0)
    dev = _device()
    if np.all(a.imag == 0.0):
        At, lda = to_device_colmajor(0.5 * (a.real + a.real.T), dev)
        w = syevd_values_device(At, lda, n).cpu().numpy()
        return w[::-1].copy()
    t = np.block([[a.real, a.imag], [-a.imag, a.real]])
    At, lda = to_device_colmajor(0.5 * (t + t.T), dev)
    w2 = syevd_values_device(At, lda, 2 * n).cpu().numpy()[::-1]
    return 0.5 * (w2[0::2] + w2[1::2])


def tda_gap_report(op: BseOperator, workers: int = 1):
    """Tamm-Dancoff overestimation gaps g_j = lambda_j(A) - lambda_j(H)
    (reference: solvers.tda_gap_report, solvers.py:149-160); both spectra on
    the GPU."""
    from .types import TdaGapReport
    lam_a = hermitian_eigvals(op.a)
    lam_h = solve_complex(op, workers=workers).lambda_plus
    gaps = lam_a - lam_h
    scale = float(np.max(np.abs(lam_a))) if lam_a.size else 0.0
    min_gap = float(np.min(gaps)) if gaps.size else 0.0
    max_rel = float(np.max(gaps / lam_h)) if gaps.size else 0.0
    return TdaGapReport(gaps=gaps, max_relative_gap=max_rel, min_gap=min_gap, scale=scale,
                        certified=bool(min_gap >= -1e-12 * scale))


def solve_complex(op: BseOperator, workers: int = 1) -> PositiveEigensystem:
    """Structure-preserving solve (reference: solvers.py:29-77).  ``workers``
    is accepted for signature compatibility; the output is independent of it.
    Real operators run the n x n product form directly (SURVEY 8b routing);
    complex ones go through bse_solve_complex_host (real 2n embedding, one
    eigenvector per doubled eigenvalue, complex extraction on the device)."""
    del workers
    n = op.n
    if n == 0:
        return PositiveEigensystem(lambda_plus=np.zeros(0), x1=np.zeros((0, 0)), x2=np.zeros((0, 0)))
    dev = _device()
    if op.kind == "real":
        try:
            lam_h, x1, x2 = _solve_real_pair(op)
        except NotPositiveDefinite as err:
            # build_m = diag(A+B, A-B): A-B pivots are offset by n
            idx = err.pivot_index if err.failed_factor == 1 else n + err.pivot_index
            raise NotPositiveDefinite(idx, err.pivot_value, _WHAT_M) from None
        return PositiveEigensystem(lambda_plus=lam_h, x1=x1, x2=x2,
                                   warnings=conditioning_warnings(lam_h))
    lam, x1, x2 = _solve_complex_host(op.a, op.b, n)
    return PositiveEigensystem(lambda_plus=lam, x1=x1, x2=x2, warnings=conditioning_warnings(lam))


def solve_oracle(op: BseOperator) -> np.ndarray:
    """Cross-check solver through the generalized Hermitian-definite route
    (reference: solvers.solve_oracle, solvers.py:116-133): Omega =
    [[A, B], [conj B, conj A]] = L L^H, eigenvalues of L^H diag(I, -I) L
    (similar to H), all 2n, descending; the +- pairing is not enforced.  On
    the GPU: Omega's interleaved real embedding (each entry z -> [[Re z,
    -Im z], [Im z, Re z]], so Cholesky pivot 2j is Omega's pivot j), the
    library's Cholesky, one DMMA GEMM for L^T S L and the values-only
    two-stage eigensolver; every eigenvalue comes out twice."""
    torch = require_cuda()
    n = op.n
    if n == 0:
        return np.zeros(0)
    dev = _device()
    A = torch.from_numpy(np.array(op.a)).to(dev)
    B = torch.from_numpy(np.array(op.b)).to(dev)
    om = torch.cat([torch.cat([A, B], 1), torch.cat([B.conj(), A.conj()], 1)], 0)
    om = 0.5 * (om + om.conj().T)
    m = 2 * n
    N = 2 * m
    emb = torch.empty((m, 2, m, 2), dtype=torch.float64, device=dev)
    emb[:, 0, :, 0] = om.real
    emb[:, 0, :, 1] = -om.imag
    emb[:, 1, :, 0] = om.imag
    emb[:, 1, :, 1] = om.real
    Lt, ld = colmajor_empty(N, N, dev)
    Lt[:N, :N].copy_(emb.reshape(N, N).T)  # column-major buffer of the (symmetric) embedding
    del emb, om, A, B
    lib = _lib.load()
    info = _lib.BseInfo()
    st = lib.bse_potrf_dev(N, ptr(Lt), ld, stream_ptr(dev), C.byref(info))
    if st == _lib.BSE_NOT_POSITIVE_DEFINITE:
        raise NotPositiveDefinite(int(info.pivot_index) // 2, float(info.pivot_value), "Omega")
    raise_for_status(st, info, "bse_potrf_dev")
    # T = S L (S = -1 on the rows of Omega's second block), K = L^T T
    T, _ = colmajor_empty(N, N, dev)
    T.copy_(Lt)
    view_colmajor(T, N, N)[m:, :] *= -1.0
    K, _ = colmajor_empty(N, N, dev)
    _gemm(1, 0, N, N, N, 1.0, ptr(Lt), ld, ptr(T), ld, 0.0, ptr(K), ld)
    del T, Lt
    w = syevd_values_device(K, ld, N).cpu().numpy()[::-1]
    return 0.5 * (w[0::2] + w[1::2])


def _potrf_margin(m: np.ndarray, dev):
    """GPU Cholesky probe of one symmetric block: (ok, margin, pivot_index)
    with margin = min(diag L)^2 or the failing pivot value."""
    n = m.shape[0]
    At, lda = to_device_colmajor(m, dev)
    info = _lib.BseInfo()
    st = _lib.load().bse_potrf_dev(n, ptr(At), lda, stream_ptr(dev), C.byref(info))
    if st == _lib.BSE_NOT_POSITIVE_DEFINITE:
        return False, float(info.pivot_value), int(info.pivot_index)
    if st != _lib.BSE_OK:
        raise RuntimeError(f"bse_potrf_dev failed ({st}): {_lib.last_error()}")
    d = view_colmajor(At, n, n).diagonal()
    return True, float(d.min().item()) ** 2, -1


def validate(op: BseOperator, tol: float | None = None):
    """Structural pre-check (reference: core.validate, core.py:203-232):
    (A Hermitian, B symmetric) within ``tol`` (default SYM_RTOL) and positive
    definiteness of the real embedding build_m, probed by the GPU Cholesky.
    ``margin`` is min(diag L)^2 on success, else the failing pivot value.
    For a real operator build_m = diag(A+B, A-B) exactly, so the two blocks
    are factored separately (A+B first, as the reference's column order)."""
    from .types import SYM_RTOL, ValidationReport, _frob, build_m
    rtol = SYM_RTOL if tol is None else float(tol)

    def defect(x, conj):
        nrm = _frob(x)
        return 0.0 if nrm == 0.0 else _frob(x - (x.conj().T if conj else x.T)) / nrm

    defects = (defect(op.a, True), defect(op.b, False))
    sym_ok = (_frob(op.a - op.a.conj().T) <= rtol * max(1.0, _frob(op.a))
              and _frob(op.b - op.b.T) <= rtol * max(1.0, _frob(op.b)))
    m = build_m(op)
    N = m.shape[0]
    if N == 0:
        return ValidationReport(symmetry_ok=bool(sym_ok), definiteness_ok=True,
                                sym_defects=defects, margin=0.0)
    dev = _device()
    n = op.n
    blocks = [m[:n, :n], m[n:, n:]] if op.kind == "real" else [m]
    margin = np.inf
    pd_ok = True
    for blk in blocks:
        ok, mg, _ = _potrf_margin(np.ascontiguousarray(blk), dev)
        if not ok:
            pd_ok, margin = False, mg
            break
        margin = min(margin, mg)
    return ValidationReport(symmetry_ok=bool(sym_ok), definiteness_ok=pd_ok,
                            sym_defects=defects, margin=float(margin))
