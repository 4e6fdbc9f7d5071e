"""GPU parity at BASELINE sizes the host can still check: cfg1 at full size
(complex n = 2048, real embedding N = 4096) and cfg0/cfg2-recipe real
problems at n = 2048, against an independent LAPACK route (numpy Cholesky +
eigvalsh of W = L^T M L) and the size-independent properties of SURVEY 8c(8):
per-pair residual <= 1e-13 n, ||Y^H X - I|| <= 1e-12 n, lambda > 0,
descending, TDA overestimation.  Also the values-only eigensolver
(SY2SB + SB2ST + Sturm bisection) against LAPACK."""
import numpy as np
import pytest

import paper_1501_03830_b200 as bg
from paper_1501_03830_b200 import configs

from conftest import random_symmetric

pytestmark = pytest.mark.gpu


def lapack_lambda(m, k):
    """Independent route: K = L L^T (LAPACK), eig(L^T M L) (LAPACK)."""
    low = np.linalg.cholesky(k)
    w = low.T @ m @ low
    lam2 = np.linalg.eigvalsh(0.5 * (w + w.T))
    return np.sqrt(lam2)[::-1]


def check_properties(op, pos, n):
    lam = pos.lambda_plus
    assert np.all(lam > 0) and np.all(np.diff(lam) <= 0)
    a, b = op.a, op.b
    x1, x2 = pos.x1, pos.x2
    # H [x1; x2] = [A x1 + B x2; -conj(B) x1 - conj(A) x2]
    top = a @ x1 + b @ x2 - x1 * lam
    bot = -(b.conj() @ x1) - a.conj() @ x2 - x2 * lam
    hn = np.linalg.norm(np.block([[a, b], [-b.conj(), -a.conj()]]), 2)
    res = np.sqrt(np.sum(np.abs(top) ** 2, 0) + np.sum(np.abs(bot) ** 2, 0))
    xn = np.sqrt(np.sum(np.abs(x1) ** 2, 0) + np.sum(np.abs(x2) ** 2, 0))
    assert (res / (hn * xn)).max() <= 1e-13 * n
    # Y^H X - I with Y = [[X1, -conj X2], [-X2, conj X1]] blockwise:
    g11 = x1.conj().T @ x1 - x2.conj().T @ x2 - np.eye(n)
    g12 = x1.conj().T @ x2.conj() - x2.conj().T @ x1.conj()
    assert np.sqrt(2 * np.linalg.norm(g11) ** 2 + 2 * np.linalg.norm(g12) ** 2) <= 1e-12 * n
    return res / (hn * xn)


def test_cfg1_full_size(dev):
    """BASELINE config 1 at its full size (complex n = 2048)."""
    a, b, dip = configs.config_operator(1, n=2048)
    op = bg.make_operator(a, b, kind="complex")
    pos = bg.solve_complex(op)
    m, k = bg.real_embedding(op)
    lam_ref = lapack_lambda(m, k)[0::2]
    assert np.max(np.abs(pos.lambda_plus - lam_ref) / lam_ref) <= 1e-10
    check_properties(op, pos, 2048)
    # TDA: lambda_j(H) <= lambda_j(A); the TDA truth is sort(a) (U diag(a) U^H)
    _, _, _, a_vals = configs.complex_operator(2048, seed=1)
    assert bg.dos_dominance(pos.lambda_plus, a_vals)
    lam_a = bg.hermitian_eigvals(a)
    assert np.max(np.abs(lam_a - a_vals)) <= 1e-12 * a_vals[0]
    # absorption pairing defect
    curve = bg.absorption_spectrum(pos, bg.DipoleData(d_r=dip, d_l=dip), sigma=0.05)
    assert curve.normalization_defect <= 1e-11


@pytest.mark.parametrize("cfg", [0, 2])
def test_real_n2048(dev, cfg):
    a, b, _ = configs.config_operator(cfg, n=2048)
    op = bg.make_operator(a, b, kind="real")
    pos = bg.solve_real(op)
    lam_ref = lapack_lambda(a + b, a - b)
    assert np.max(np.abs(pos.lambda_plus - lam_ref) / lam_ref) <= 1e-10
    check_properties(op, pos, 2048)


@pytest.mark.parametrize("n", [1024, 6144])
def test_clustered_cfg4_recipe(dev, n):
    """cfg4 recipe (256 clusters of 1e-6 relative spread): heavy D&C
    deflation; n = 6144 runs the emulated-FP64 path (top merges, Q1, ...)."""
    a, b, _ = configs.config_operator(4, n=n)
    op = bg.make_operator(a, b, kind="real")
    pos = bg.solve_real(op)
    lam_ref = lapack_lambda(a + b, a - b)
    assert np.max(np.abs(pos.lambda_plus - lam_ref) / lam_ref) <= 1e-10
    check_properties(op, pos, n)


@pytest.mark.parametrize("n", [1, 2, 7, 64, 65, 1000, 2049])
def test_values_only_vs_lapack(dev, n):
    s = random_symmetric(n, n + 3)
    got = bg.hermitian_eigvals(s)
    ref = np.sort(np.linalg.eigvalsh(s))[::-1]
    assert np.max(np.abs(got - ref)) <= 1e-13 * max(1.0, np.abs(ref).max()) * max(1, np.log2(n))


def test_tda_gap_report_golden(dev):
    from pathlib import Path
    z = dict(np.load(Path(__file__).resolve().parent / "golden" / "tda_cfg1_n48.npz"))
    lam_a = bg.hermitian_eigvals(z["a"])
    assert np.max(np.abs(lam_a - z["lam_a"])) <= 1e-13 * np.max(np.abs(z["lam_a"]))
    a, b, _ = configs.config_operator(1, n=48)
    rep = bg.tda_gap_report(bg.make_operator(a, b))
    assert rep.certified and rep.min_gap >= -1e-12 * rep.scale


def test_tda_gap_1x1_analytic(dev):
    rep = bg.tda_gap_report(bg.make_operator([[2.0]], [[1j]]))
    assert rep.gaps[0] == pytest.approx(2.0 - np.sqrt(3.0), abs=1e-14)
    assert rep.certified


def test_emulated_fp64_path_n4608(dev):
    """n >= 4096 routes the congruence, the top D&C merges, Q1, the recovery
    TRMM and the top TRSM updates through the emulated-FP64 INT8 engine:
    the solve must meet the same gates as the all-DMMA path
    (BSE_FLAG_NATIVE_FP64) and agree with it and with LAPACK."""
    import torch
    from paper_1501_03830_b200 import _lib
    from paper_1501_03830_b200.device import from_device_colmajor, to_device_colmajor
    n = 4608
    a, b, _ = configs.config_operator(2, n=n)
    op = bg.make_operator(a, b, kind="real")
    pos = bg.solve_real(op)
    lam_ref = lapack_lambda(a + b, a - b)
    assert np.max(np.abs(pos.lambda_plus - lam_ref) / lam_ref) <= 1e-10
    check_properties(op, pos, n)
    Mt, ldm = to_device_colmajor(a + b, dev)
    Kt, ldk = to_device_colmajor(a - b, dev)
    lam_n, X1n, _, _ = bg.solve_pair_device(Mt, ldm, Kt, ldk, n, flags=_lib.FLAG_NATIVE_FP64)
    lam_n = lam_n.cpu().numpy()
    assert np.max(np.abs(lam_n - pos.lambda_plus) / lam_n) <= 1e-12
    x1n = from_device_colmajor(X1n, n, n)
    x1 = pos.x1.real
    # columns equal up to sign, tolerance n eps |W| / gap(lambda^2)
    l2 = lam_n ** 2
    d = -np.diff(l2)
    gap = np.minimum(np.r_[np.inf, d], np.r_[d, np.inf]) / l2[0]
    sgn = np.sign(np.sum(x1 * x1n, axis=0))
    err = np.linalg.norm(x1 * sgn - x1n, axis=0) / np.linalg.norm(x1n, axis=0)
    assert np.all(err <= n * np.finfo(float).eps / gap + 1e-12)
    torch.cuda.synchronize()


def test_repeat_solves_bitwise_identical(dev):
    """The solve overlaps work on auxiliary streams (SY2SB panel look-ahead,
    Q2/Q1 block builds under the D&C): repeated solves must be bitwise
    identical (no race, no order-dependent reduction)."""
    import torch
    from paper_1501_03830_b200.device import to_device_colmajor, view_colmajor
    n = 5000
    a, b, _ = configs.config_operator(2, n=n, seed=7)
    Mt, ldm = to_device_colmajor(a + b, dev)
    Kt, ldk = to_device_colmajor(a - b, dev)
    outs = []
    for _ in range(3):
        lam, X1, X2, _ = bg.solve_pair_device(Mt, ldm, Kt, ldk, n)
        outs.append((lam.clone(), view_colmajor(X1, n, n).clone(), view_colmajor(X2, n, n).clone()))
    torch.cuda.synchronize()
    for lam, X1, X2 in outs[1:]:
        assert torch.equal(lam, outs[0][0])
        assert torch.equal(X1, outs[0][1]) and torch.equal(X2, outs[0][2])
