"""Drop-in solver API: ``solve_real`` / ``solve_complex`` with the reference's
signatures (pkg/src/bse/solvers.py:29, :80), backed by the sm_100a library.

Both run the north-star product form on the GPU: M = A+B, K = A-B (or their
2n x 2n real embedding for complex operators, D3), K = L L^T,
W = L^T M L = Z Lam^2 Z^T, X1,2 = (L Z +- L^{-T} Z Lam) Lam^{-1/2} / 2.
Torch is used for device memory, streams and index plumbing only; every
floating-point stage (Cholesky, congruence, eigensolver, back-transforms,
recovery, biorthogonality polish GEMMs, absorption) is a kernel of
libbse_b200.so.  There is no CPU fallback: without a CUDA device these raise.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .device import (colmajor_empty, from_device_colmajor, ptr, require_cuda, stream_ptr,
                     to_device_colmajor, view_colmajor)
from .types import (EPS, BseOperator, ConvergenceError, NotPositiveDefinite,
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
    dev = _device()
    m, k = _real_pair(op)
    Mt, ldm = to_device_colmajor(m, dev)
    Kt, ldk = to_device_colmajor(k, dev)
    lam, X1, X2, _ = solve_pair_device(Mt, ldm, Kt, ldk, n)
    lam_h = lam.cpu().numpy()
    x1 = from_device_colmajor(X1, n, n)
    x2 = from_device_colmajor(X2, n, n)
    return PositiveEigensystem(lambda_plus=lam_h, x1=x1.astype(np.complex128),
                               x2=x2.astype(np.complex128), warnings=conditioning_warnings(lam_h))


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


def _real_embedding_device(op: BseOperator, dev):
    """real_embedding() formed on the device from one upload of A and B:
    the same IEEE operations as the host version (bitwise equal), without
    host-side block assembly and transposes of 2n x 2n arrays.  M', K' are
    exactly symmetric, so their row-major tensors are their column-major
    buffers."""
    torch = require_cuda()
    n = op.n
    N = 2 * n

    def up(x):
        x = np.asarray(x)
        return torch.from_numpy(x if x.flags.writeable else x.copy()).to(dev)

    A, B = up(op.a), up(op.b)
    ar, ai, br, bi = A.real, A.imag, B.real, B.imag
    out = []
    for sgn in (1.0, -1.0):  # M' = A' + B', K' = A' - B'
        T = torch.empty((N, N), dtype=torch.float64, device=dev)
        T[:n, :n] = ar + sgn * br
        T[:n, n:] = -ai + sgn * bi
        T[n:, :n] = ai + sgn * bi
        T[n:, n:] = ar - sgn * br
        T = 0.5 * (T + T.T)
        buf, ld = colmajor_empty(N, N, dev)
        buf[:N, :N].copy_(T)
        del T
        out.append((buf, ld))
    del A, B
    return out


def _select_and_polish(lam2, X1, X2, ld, n, dev):
    """Complex eigenvectors from the doubled real spectrum of the 2n-embedding.

    Every complex eigenvalue appears twice; one real vector per pair maps to
    x = r1[:n] + i r1[n:], y = r2[:n] - i r2[n:].  Within clusters of
    (nearly) equal complex eigenvalues, k independent vectors are chosen by
    pivoted Gram-Schmidt in the indefinite product <x, y> = x1^H y1 - x2^H y2
    (positive definite on the positive-lambda subspace), mirroring the
    reference's _pivoted_orthonormal (kernels.py:644-674).  A GEMM-only
    biorthogonality polish X <- X (1.5 I - G / 2), G = X1^H X1 - X2^H X2, then
    restores Y^H X = I to O(eps) (D3)."""
    torch = require_cuda()
    N = 2 * n
    lam2_h = lam2.cpu().numpy()
    x1 = view_colmajor(X1, N, N)  # (N x N) torch views, columns = eigenvectors
    x2 = view_colmajor(X2, N, N)
    # cluster detection on the host (O(N) scalars)
    scale = max(1.0, float(np.max(np.abs(lam2_h))))
    dtol = 20.0 * N * EPS * scale
    sel = []
    lam = []
    start = 0
    while start < N:
        stop = start + 1
        while stop < N and lam2_h[stop - 1] - lam2_h[stop] <= dtol:
            stop += 1
        size = stop - start
        k = size // 2
        if size == 2:
            sel.append(start)
            lam.append(0.5 * (lam2_h[start] + lam2_h[start + 1]))
        else:
            # pivoted Gram-Schmidt in the indefinite product (device tensors)
            cand1 = torch.complex(x1[:n, start:stop], x1[n:, start:stop])
            cand2 = torch.complex(x2[:n, start:stop], -x2[n:, start:stop])
            chosen1, chosen2 = [], []
            w1, w2 = cand1.clone(), cand2.clone()
            for _ in range(max(k, 1)):
                nrm = (w1.abs() ** 2).sum(0) - (w2.abs() ** 2).sum(0)
                j = int(torch.argmax(nrm))
                s = torch.sqrt(torch.clamp(nrm[j], min=1e-300))
                u1, u2 = w1[:, j] / s, w2[:, j] / s
                chosen1.append(u1)
                chosen2.append(u2)
                coef = (u1.conj() @ w1) - (u2.conj() @ w2)
                w1 = w1 - torch.outer(u1, coef)
                w2 = w2 - torch.outer(u2, coef)
            sel.append((start, stop, torch.stack(chosen1, 1), torch.stack(chosen2, 1)))
            vals = lam2_h[start:stop]
            for t in range(max(k, 1)):
                lam.append(float(np.mean(vals[2 * t:2 * t + 2])) if 2 * t + 1 < size else float(vals[-1]))
        start = stop
    # assemble planar complex X1c, X2c (n x n) on device: one gather for all
    # simple pairs, cluster blocks copied in place
    X1c = torch.empty((n, n), dtype=torch.complex128, device=dev)
    X2c = torch.empty((n, n), dtype=torch.complex128, device=dev)
    simple_out, simple_src, col = [], [], 0
    blocks = []
    for s in sel:
        if isinstance(s, int):
            simple_out.append(col)
            simple_src.append(s)
            col += 1
        else:
            k = s[2].shape[1]
            blocks.append((col, s[2], s[3]))
            col += k
    if simple_src:
        src = torch.tensor(simple_src, device=dev)
        dst = torch.tensor(simple_out, device=dev)
        X1c[:, dst] = torch.complex(x1[:n, src], x1[n:, src])
        X2c[:, dst] = torch.complex(x2[:n, src], -x2[n:, src])
    for c0, b1, b2 in blocks:
        k = min(b1.shape[1], n - c0)
        if k > 0:
            X1c[:, c0:c0 + k] = b1[:, :k]
            X2c[:, c0:c0 + k] = b2[:, :k]
    lam = np.array(lam[:n])
    X1c, X2c = polish(X1c, X2c)
    return lam, X1c, X2c


def polish(X1c, X2c):
    """Biorthogonality polish with the library's DMMA GEMM (complex products
    as stacked real GEMMs): G = X1^H X1 - X2^H X2; X <- X (1.5 I - 0.5 G)."""
    torch = require_cuda()
    n = X1c.shape[0]
    dev = X1c.device
    # column-major planar stacks: P = [X1r; X1i; X2r; X2i] (4n x n)
    P, ldp = colmajor_empty(4 * n, n, dev)
    Q, _ = colmajor_empty(4 * n, n, dev)
    R, _ = colmajor_empty(4 * n, n, dev)
    pv, qv, rv = view_colmajor(P, 4 * n, n), view_colmajor(Q, 4 * n, n), view_colmajor(R, 4 * n, n)
    parts = (X1c.real, X1c.imag, X2c.real, X2c.imag)
    for i, blk in enumerate(parts):
        pv[i * n:(i + 1) * n] = blk
    qv[:2 * n] = pv[:2 * n]
    qv[2 * n:] = -pv[2 * n:]
    rv[0:n], rv[n:2 * n], rv[2 * n:3 * n], rv[3 * n:] = parts[1], -parts[0], -parts[3], parts[2]
    # Gr = P^T Q, Gi = P^T R  (n x n)
    Gr, ldg = colmajor_empty(n, n, dev)
    Gi, _ = colmajor_empty(n, n, dev)
    _gemm(1, 0, n, n, 4 * n, 1.0, ptr(P), ldp, ptr(Q), ldp, 0.0, ptr(Gr), ldg)
    _gemm(1, 0, n, n, 4 * n, 1.0, ptr(P), ldp, ptr(R), ldp, 0.0, ptr(Gi), ldg)
    # F_big = [[Fr, Fi], [-Fi, Fr]] with F = 1.5 I - 0.5 G
    Fb, ldf = colmajor_empty(2 * n, 2 * n, dev)
    fv = view_colmajor(Fb, 2 * n, 2 * n)
    gr, gi = view_colmajor(Gr, n, n), view_colmajor(Gi, n, n)
    eye = torch.eye(n, dtype=torch.float64, device=dev)
    fr = 1.5 * eye - 0.5 * gr
    fi = -0.5 * gi
    fv[:n, :n] = fr
    fv[:n, n:] = fi
    fv[n:, :n] = -fi
    fv[n:, n:] = fr
    # Xs = [X1r X1i; X2r X2i] (2n x 2n) ; Xs_new = Xs F_big
    Xs, ldx = colmajor_empty(2 * n, 2 * n, dev)
    xv = view_colmajor(Xs, 2 * n, 2 * n)
    xv[:n, :n], xv[:n, n:], xv[n:, :n], xv[n:, n:] = parts[0], parts[1], parts[2], parts[3]
    Out, _ = colmajor_empty(2 * n, 2 * n, dev)
    _gemm(0, 0, 2 * n, 2 * n, 2 * n, 1.0, ptr(Xs), ldx, ptr(Fb), ldf, 0.0, ptr(Out), ldx)
    ov = view_colmajor(Out, 2 * n, 2 * n)
    return torch.complex(ov[:n, :n], ov[:n, n:]), torch.complex(ov[n:, :n], ov[n:, n:])


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
    Real operators run the n x n product form directly (SURVEY 8b routing)."""
    del workers
    n = op.n
    if n == 0:
        return PositiveEigensystem(lambda_plus=np.zeros(0), x1=np.zeros((0, 0)), x2=np.zeros((0, 0)))
    dev = _device()
    if op.kind == "real":
        m, k = _real_pair(op)
        Mt, ldm = to_device_colmajor(m, dev)
        Kt, ldk = to_device_colmajor(k, dev)
        try:
            lam, X1, X2, _ = solve_pair_device(Mt, ldm, Kt, ldk, n)
        except NotPositiveDefinite as err:
            # build_m = diag(A+B, A-B): A-B pivots are offset by n
            idx = err.pivot_index if err.failed_factor == 1 else n + err.pivot_index
            raise NotPositiveDefinite(idx, err.pivot_value, _WHAT_M) from None
        lam_h = lam.cpu().numpy()
        x1 = from_device_colmajor(X1, n, n)
        x2 = from_device_colmajor(X2, n, n)
        return PositiveEigensystem(lambda_plus=lam_h, x1=x1.astype(np.complex128),
                                   x2=x2.astype(np.complex128),
                                   warnings=conditioning_warnings(lam_h))
    N = 2 * n
    (Mt, ldm), (Kt, ldk) = _real_embedding_device(op, dev)
    try:
        lam2, X1, X2, ld = solve_pair_device(Mt, ldm, Kt, ldk, N)
    except NotPositiveDefinite as err:
        raise NotPositiveDefinite(err.pivot_index, err.pivot_value, _WHAT_M) from None
    lam, X1c, X2c = _select_and_polish(lam2, X1, X2, ld, n, dev)
    return PositiveEigensystem(lambda_plus=lam, x1=X1c.cpu().numpy(), x2=X2c.cpu().numpy(),
                               warnings=conditioning_warnings(lam))


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
