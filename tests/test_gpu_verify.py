"""Device verification (bse_pair_residuals_dev) against numpy, then the
BASELINE cfg2 solve at its FULL size (real n = 16384) checked through the
size-independent properties of SURVEY 8c(8): per-pair residual <= 1e-13 n,
||X1^T X1 - X2^T X2 - I||_F <= 1e-12 n, lam > 0 descending, and the spectral
moment identities sum lam^2 = tr(M K), sum lam^4 = tr((M K)^2) (independent
of every stage of the eigensolver)."""
import numpy as np
import pytest

import paper_1501_03830_b200 as bg
from paper_1501_03830_b200 import configs
from paper_1501_03830_b200.device import to_device_colmajor

from conftest import random_spd_real

pytestmark = pytest.mark.gpu


def numpy_pair_residuals(m, k, lam, x1, x2):
    a, b = 0.5 * (m + k), 0.5 * (m - k)
    top = a @ x1 + b @ x2 - x1 * lam
    bot = -(b @ x1) - a @ x2 - x2 * lam
    res = np.sqrt(np.sum(top ** 2, 0) + np.sum(bot ** 2, 0))
    xn = np.sqrt(np.sum(x1 ** 2, 0) + np.sum(x2 ** 2, 0))
    bio = np.linalg.norm(x1.T @ x1 - x2.T @ x2 - np.eye(x1.shape[1]))
    return res, xn, bio


@pytest.mark.parametrize("n", [1, 2, 7, 64, 65, 300])
def test_pair_residuals_vs_numpy(dev, n):
    import torch
    rng = np.random.default_rng(n)
    m, k = random_spd_real(n, n), random_spd_real(n, n + 1)
    x1 = rng.standard_normal((n, n))
    x2 = 0.3 * rng.standard_normal((n, n))
    lam = np.sort(rng.uniform(1, 5, n))[::-1].copy()
    # only the lower triangles of M, K may be read
    Mt, ldm = to_device_colmajor(np.tril(m), dev)
    Kt, ldk = to_device_colmajor(np.tril(k), dev)
    X1, l1 = to_device_colmajor(x1, dev)
    X2, l2 = to_device_colmajor(x2, dev)
    lt = torch.from_numpy(lam).to(dev)
    res, xn, bio = bg.pair_residuals_device(n, Mt, ldm, Kt, ldk, lt, X1, l1, X2, l2)
    r_ref, x_ref, b_ref = numpy_pair_residuals(m, k, lam, x1, x2)
    np.testing.assert_allclose(res.cpu().numpy(), r_ref, rtol=1e-12)
    np.testing.assert_allclose(xn.cpu().numpy(), x_ref, rtol=1e-13)
    assert abs(float(bio) - b_ref) <= 1e-12 * b_ref


def test_pair_residual_report_on_solution(dev):
    n = 200
    a, b, _ = configs.config_operator(0, n=n)
    op = bg.make_operator(a, b, kind="real")
    pos = bg.solve_real(op)
    rep = bg.pair_residual_report(op, pos)
    assert rep.passes(n)
    # conservative lam_max normalisation is >= the ||H||_2 one
    hn = np.linalg.norm(np.block([[a, b], [-b, -a]]), 2)
    res, xn, bio = numpy_pair_residuals(a + b, a - b, pos.lambda_plus, pos.x1.real, pos.x2.real)
    assert rep.max_ratio >= 0.999 * np.max(res / (hn * xn))
    assert rep.biorthogonality == pytest.approx(bio, rel=1e-6, abs=1e-14)


def test_cfg2_full_size_properties(dev):
    """BASELINE config 2 at its full size: real n = 16384 (the bench workload)."""
    import torch
    n = 16384
    S, D, _ = configs.torch_real_operator(n, seed=2, device=dev)
    lam, X1, X2, ld = bg.solve_pair_device(S, n, D, n, n)
    lam_h = lam.cpu().numpy()
    assert np.all(lam_h > 0) and np.all(np.diff(lam_h) <= 0)
    res, xn, bio = bg.pair_residuals_device(n, S, n, D, n, lam, X1, ld, X2, ld)
    ratio = (res / (lam[0] * xn)).max().item()
    assert ratio <= 1e-13 * n, ratio
    assert bio.item() <= 1e-12 * n, bio.item()
    # spectral moments of W = L^T M L ~ M K (test-side cuBLAS as the checker)
    G = S @ D
    m2 = torch.sum(S * D).item()            # tr(M K)
    m4 = torch.sum(G * G.T).item()          # tr((M K)^2)
    l2 = lam.double() ** 2
    assert abs(torch.sum(l2).item() - m2) <= 1e-12 * n * m2
    assert abs(torch.sum(l2 * l2).item() - m4) <= 1e-12 * n * m4


def test_cfg4_recipe_n16384_properties(dev):
    """BASELINE config 4's clustered spectrum (256 clusters, 1e-6 relative
    spread: heavy D&C deflation, near-degenerate eigenvectors) at n = 16384
    on one GPU: positivity/order, per-pair residual and biorthogonality
    gates, and the spectral moments tr(MK), tr((MK)^2)."""
    import torch
    n = 16384
    S, D, _ = configs.torch_real_operator(n, seed=4, spectrum="clustered", lo=1.0, hi=10.0,
                                          device=dev)
    lam, X1, X2, ld = bg.solve_pair_device(S, n, D, n, n)
    lam_h = lam.cpu().numpy()
    assert np.all(lam_h > 0) and np.all(np.diff(lam_h) <= 0)
    res, xn, bio = bg.pair_residuals_device(n, S, n, D, n, lam, X1, ld, X2, ld)
    ratio = (res / (lam[0] * xn)).max().item()
    assert ratio <= 1e-13 * n, ratio
    assert bio.item() <= 1e-12 * n, bio.item()
    G = S @ D
    m2 = torch.sum(S * D).item()
    m4 = torch.sum(G * G.T).item()
    l2 = lam.double() ** 2
    assert abs(torch.sum(l2).item() - m2) <= 1e-12 * n * m2
    assert abs(torch.sum(l2 * l2).item() - m4) <= 1e-12 * n * m4
