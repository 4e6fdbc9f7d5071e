"""Complex Hermitian BSE through the library entry (bse_solve_complex_*,
the drop-in for solvers.solve_complex, solvers.py:29-77): the BASELINE cfg3
size with every pair verified, clustered spectra resolved by the pivoted
Gram-Schmidt (kernels.py:659-674 analogue) compared by principal angles with
the reference algorithm, and host entry == device entry."""
import ctypes as C

import numpy as np
import pytest

import paper_1501_03830_b200 as bg
from oracle import bse_oracle as orc
from paper_1501_03830_b200 import _lib, configs
from paper_1501_03830_b200.device import ptr, stream_ptr

pytestmark = pytest.mark.gpu
EPS = np.finfo(float).eps


def verify_device(A, B, lam, X1, X2):
    """Per-pair residual / (lam_max |x|), |X1^H X1 - X2^H X2 - I|_F."""
    from paper_1501_03830_b200.verify import complex_pair_residuals
    return complex_pair_residuals(A, B, lam, X1, X2)


def principal_angle_max(x_new, x_ref):
    from conftest import principal_angle
    return principal_angle(x_new, x_ref)


def clusters_of(lam, rtol):
    out, i = [], 0
    while i < lam.shape[0]:
        j = i + 1
        while j < lam.shape[0] and lam[j - 1] - lam[j] <= rtol * lam[0]:
            j += 1
        out.append((i, j))
        i = j
    return out


def test_cfg3_full_size_every_pair(dev):
    """BASELINE cfg3: complex n = 16384 (real embedding N = 32768) on one
    B200 through bse_solve_complex_dev; gates on EVERY pair."""
    import torch
    n = 16384
    A, B, _, a_vals = configs.torch_complex_operator(n, seed=3, lo=2.0, hi=10.0, bnorm="0.9min",
                                                     device=dev)
    lam, X1, X2 = bg.solve_complex_device(A, B, n)
    torch.cuda.synchronize()
    lam_h = lam.cpu().numpy()
    assert np.all(lam_h > 0) and np.all(np.diff(lam_h) <= 0)
    assert bg.dos_dominance(lam_h, a_vals.cpu().numpy())  # TDA: lam_j(H) <= a_j
    torch.cuda.empty_cache()
    res, bio = verify_device(A, B, lam, X1, X2)
    assert res <= 1e-13 * n, res
    assert bio <= 1e-12 * n, bio


def test_host_entry_equals_device_entry(dev):
    import torch
    n = 300
    a, b, _, _ = configs.complex_operator(n, seed=11, bnorm="0.9min")
    op = bg.make_operator(a, b, kind="complex")
    pos = bg.solve_complex(op)  # host entry
    lam, X1, X2 = bg.solve_complex_device(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev), n)
    assert np.array_equal(pos.lambda_plus, lam.cpu().numpy())
    assert np.array_equal(pos.x1, X1.cpu().numpy())
    assert np.array_equal(pos.x2, X2.cpu().numpy())


@pytest.mark.parametrize("n", [37, 1000, 3000])
def test_complex_vs_lapack_and_gates(dev, n):
    """Odd / non-tile sizes: lambda against an independent LAPACK route
    (eigvalsh of L'^T M' L' on the host embedding), r1/r2-type gates."""
    import torch
    a, b, _, _ = configs.complex_operator(n, seed=n, bnorm="0.9min")
    op = bg.make_operator(a, b, kind="complex")
    pos = bg.solve_complex(op)
    m, k = bg.real_embedding(op)
    l = np.linalg.cholesky(k)
    w2 = np.linalg.eigvalsh(l.T @ m @ l)[::-1]
    lam_ref = np.sqrt(0.5 * (w2[0::2] + w2[1::2]))
    assert np.max(np.abs(pos.lambda_plus - lam_ref) / lam_ref) <= 1e-10
    At, Bt = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    res, bio = verify_device(At, Bt, torch.from_numpy(pos.lambda_plus).to(dev),
                             torch.from_numpy(pos.x1).to(dev), torch.from_numpy(pos.x2).to(dev))
    assert res <= 1e-13 * n and bio <= 1e-12 * n, (res, bio)
    if n <= 1000:
        r1, r2 = bg.residual_metrics(op, bg.expand_full(op, pos))
        assert r1 <= 5e-14 and r2 <= 5e-14, (r1, r2)


@pytest.mark.parametrize("mult,b_scale", [(3, 0.0), (2, 0.0), (4, 1e-13)])
def test_degenerate_clusters_principal_angles(dev, mult, b_scale):
    """Exactly (b_scale = 0) or nearly degenerate complex eigenvalues: the
    doubled real clusters of size 2*mult go through the pivoted Gram-Schmidt.
    Subspaces of each cluster agree with the reference algorithm's (principal
    angles), lambda within 1e-10, r1/r2 <= 5e-14 (test_acceptance.py:31-43)."""
    rng = np.random.default_rng(mult)
    n = 12 * mult
    vals = np.repeat(np.linspace(2.0, 9.0, n // mult), mult)
    u = configs.haar_unitary(rng, n)
    a = (u * vals) @ u.conj().T
    a = 0.5 * (a + a.conj().T)
    g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    b = b_scale * 0.5 * (g + g.T)
    op = bg.make_operator(a, b, kind="complex")
    pos = bg.solve_complex(op)
    lam_ref, x1r, x2r = orc.solve_complex(op.a, op.b)
    assert np.max(np.abs(pos.lambda_plus - lam_ref) / lam_ref) <= 1e-10
    x_new = np.vstack([pos.x1, pos.x2])
    x_ref = np.vstack([x1r, x2r])
    gap = 7.0 / (n // mult - 1)          # between cluster centres (lambda)
    tol = 10.0 * n * EPS * 81.0 / (4.0 * gap)  # n eps |W| / gap(lambda^2), x10
    for i, j in clusters_of(lam_ref, 1e-8):
        ang = principal_angle_max(x_new[:, i:j], x_ref[:, i:j])
        assert ang <= tol, (i, j, ang, tol)
    r1, r2 = bg.residual_metrics(op, bg.expand_full(op, pos))
    assert r1 <= 5e-14 and r2 <= 5e-14, (r1, r2)


def test_cluster_count_reported(dev):
    import torch
    n = 24
    vals = np.repeat([3.0, 5.0, 8.0], 8)
    op = bg.make_operator(np.diag(vals).astype(complex), np.zeros((n, n)), kind="complex")
    lib = _lib.load()
    A = torch.from_numpy(np.ascontiguousarray(op.a)).to(dev)
    B = torch.from_numpy(np.ascontiguousarray(op.b)).to(dev)
    X1 = torch.empty((n, n), dtype=torch.complex128, device=dev)
    X2 = torch.empty_like(X1)
    lam = torch.empty(n, dtype=torch.float64, device=dev)
    wb = lib.bse_solve_complex_workspace_bytes(n, 0)
    work = torch.empty(wb, dtype=torch.uint8, device=dev)
    info = _lib.BseInfo()
    st = lib.bse_solve_complex_dev(n, ptr(A), n, ptr(B), n, ptr(lam), ptr(X1), n, ptr(X2), n,
                                   ptr(work), wb, 0, stream_ptr(dev), C.byref(info))
    assert st == _lib.BSE_OK
    assert info.clusters == 3
    x1, x2 = X1.cpu().numpy(), X2.cpu().numpy()
    assert np.linalg.norm(x1.conj().T @ x1 - x2.conj().T @ x2 - np.eye(n)) <= 1e-13
    assert np.allclose(lam.cpu().numpy(), np.sort(vals)[::-1], rtol=1e-14)
