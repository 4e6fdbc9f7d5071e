"""GPU parity of the drop-in solver against the reference's pins and the
numpy oracle: known-answer cases (test_solvers.py:20-76), golden vectors from
the reference itself (tests/golden), north-star gates (lambda 1e-10 rel,
residual 1e-13 n, Y^H X = I to 1e-12 n) and the acceptance r1/r2 gate."""
from pathlib import Path

import numpy as np
import pytest

import paper_1501_03830_b200 as bg
from oracle import bse_oracle as orc
from paper_1501_03830_b200 import configs

from conftest import vector_parity

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


def golden(name):
    return dict(np.load(G / f"{name}.npz", allow_pickle=False))


def x_full(pos):
    return np.vstack([pos.x1, pos.x2])


def assert_vectors_match(lam, x_new, x_ref, n_scale):
    """n eps |W| / gap(lambda^2) per isolated vector,
    principal angles inside clusters (conftest.vector_parity)."""
    vector_parity(lam, x_new, x_ref, n_scale)


def test_complex_1x1_analytic(dev):
    op = bg.make_operator([[2.0]], [[1j]])
    pos = bg.solve_complex(op)
    assert pos.lambda_plus == pytest.approx([np.sqrt(3.0)], abs=1e-15)
    r1, r2 = bg.residual_metrics(op, bg.expand_full(op, pos))
    assert r1 <= 1e-14 and r2 <= 1e-14


def test_real_1x1_analytic(dev):
    op = bg.make_operator([[2.0]], [[1.0]])
    pos = bg.solve_real(op)
    root = 3.0 ** 0.25
    assert pos.lambda_plus == pytest.approx([np.sqrt(3.0)], abs=1e-15)
    # sign convention: eigenvectors are defined up to sign; compare |.| and X1^2 - X2^2
    assert abs(pos.x1[0, 0]) == pytest.approx((1.0 + np.sqrt(3.0)) / (2.0 * root), abs=1e-14)
    assert abs(pos.x2[0, 0]) == pytest.approx(abs(1.0 - np.sqrt(3.0)) / (2.0 * root), abs=1e-14)
    assert (pos.x1[0, 0] ** 2 - pos.x2[0, 0] ** 2).real == pytest.approx(1.0, abs=1e-14)


def test_identity_case(dev):
    op = bg.make_operator(np.eye(4), np.zeros((4, 4)))
    pos = bg.solve_complex(op)
    assert np.allclose(pos.lambda_plus, np.ones(4), atol=1e-14)
    assert np.linalg.norm(pos.x1.conj().T @ pos.x1 - np.eye(4)) <= 1e-13
    assert np.linalg.norm(pos.x2) <= 1e-13


def test_identity_forced_complex(dev):
    # SURVEY D3 pitfall: degenerate complex cluster needs pivoted selection
    op = bg.make_operator(np.eye(4), np.zeros((4, 4)), kind="complex")
    pos = bg.solve_complex(op)
    assert np.allclose(pos.lambda_plus, np.ones(4), atol=1e-14)
    assert np.linalg.norm(pos.x1.conj().T @ pos.x1 - pos.x2.conj().T @ pos.x2 - np.eye(4)) <= 1e-13


def test_rejects_indefinite(dev):
    with pytest.raises(bg.NotPositiveDefinite):
        bg.solve_complex(bg.make_operator([[1.0]], [[2.0]]))


def test_real_identifies_failing_factor(dev):
    op = bg.make_operator(np.zeros((2, 2)), np.eye(2))  # A-B = -I
    with pytest.raises(bg.NotPositiveDefinite, match="A-B"):
        bg.solve_real(op)
    op = bg.make_operator(np.zeros((2, 2)), -np.eye(2))  # A+B = -I
    with pytest.raises(bg.NotPositiveDefinite, match="A\\+B"):
        bg.solve_real(op)


def test_pivot_matches_reference_embedding(dev):
    # complex: pivots of M' = S build_m S coincide with build_m's (D3)
    rng = np.random.default_rng(0)
    n = 6
    a = np.diag(rng.uniform(1, 2, n)).astype(complex)
    b = 3.0 * np.eye(n) * 1j
    op = bg.make_operator(a, b)
    with pytest.raises(bg.NotPositiveDefinite) as got:
        bg.solve_complex(op)
    with pytest.raises(orc.NotPositiveDefinite) as ref:
        orc.cholesky(orc.build_m(op.a, op.b))
    assert got.value.pivot_index == ref.value.pivot_index
    assert got.value.pivot_value == pytest.approx(ref.value.pivot_value, rel=1e-12)


def test_conditioning_warning(dev):
    op = bg.make_operator(np.diag([1e9, 1.0]), np.zeros((2, 2)))
    pos = bg.solve_complex(op)
    assert any("ill conditioned" in w for w in pos.warnings)


@pytest.mark.parametrize("name", ["real_1x1", "random_real_n24_s1", "cfg0_n64", "cfg2_n96"])
def test_real_golden(dev, name):
    z = golden(name)
    op = bg.make_operator(z["a"], z["b"], kind="real")
    pos = bg.solve_real(op)
    lam_ref = z["lam_real"] if "lam_real" in z else z["lam"]
    assert np.max(np.abs(pos.lambda_plus - lam_ref) / lam_ref) <= 1e-10
    xr = np.vstack([z["x1_real"], z["x2_real"]]) if "x1_real" in z else np.vstack([z["x1"], z["x2"]])
    assert_vectors_match(lam_ref, x_full(pos), xr, op.n)
    r1, r2 = bg.residual_metrics(op, bg.expand_full(op, pos))
    assert r1 <= 5e-14 and r2 <= 5e-14


@pytest.mark.parametrize("name", ["complex_1x1", "random_complex_n32_s0", "cfg1_n48", "cfg3_n40"])
def test_complex_golden(dev, name):
    z = golden(name)
    op = bg.make_operator(z["a"], z["b"], kind="complex")
    pos = bg.solve_complex(op)
    assert np.max(np.abs(pos.lambda_plus - z["lam"]) / z["lam"]) <= 1e-10
    assert_vectors_match(z["lam"], x_full(pos), np.vstack([z["x1"], z["x2"]]), 2 * op.n)
    r1, r2 = bg.residual_metrics(op, bg.expand_full(op, pos))
    assert r1 <= 5e-14 and r2 <= 5e-14


@pytest.mark.parametrize("n,seed", [(32, 0), (128, 3), (512, 7)])
def test_acceptance_residuals_random_bse(dev, n, seed):
    """test_acceptance.py:31-43 gate (r1, r2 <= 5e-14) on random_bse-style inputs."""
    rng = np.random.default_rng(seed)
    g = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
    a0 = 0.5 * (g + g.conj().T)
    g2 = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
    b0 = 0.5 * (g2 + g2.T)
    shift = np.linalg.norm(a0) + np.linalg.norm(b0) + 1.0
    op = bg.make_operator(a0 + shift * np.eye(n), b0)
    pos = bg.solve_complex(op)
    r1, r2 = bg.residual_metrics(op, bg.expand_full(op, pos))
    assert r1 <= 5e-14 and r2 <= 5e-14


@pytest.mark.parametrize("cfg,n", [(0, 512), (2, 256), (1, 128)])
def test_config_gates(dev, cfg, n):
    """North-star gates at reduced n with the BASELINE generators, checked
    against the numpy oracle's solve_complex (the reference algorithm)."""
    a, b, dip = configs.config_operator(cfg, n=n)
    op = bg.make_operator(a, b, kind=configs.CONFIGS[cfg]["kind"])
    pos = bg.solve_complex(op)
    lam_ref, x1r, x2r = orc.solve_complex(a, b)
    assert np.max(np.abs(pos.lambda_plus - lam_ref) / lam_ref) <= 1e-10
    h = bg.assemble_h(op)
    hn = np.linalg.norm(h, 2)
    x = x_full(pos)
    res = np.linalg.norm(h @ x - x * pos.lambda_plus, axis=0) / (hn * np.linalg.norm(x, axis=0))
    assert res.max() <= 1e-13 * n
    full = bg.expand_full(op, pos)
    assert np.linalg.norm(full.y.conj().T @ full.x - np.eye(2 * n)) <= 1e-12 * n
    assert np.all(pos.lambda_plus > 0)
    # absorption: basis-invariant curve vs the oracle
    sigma = 0.05
    grid = np.linspace(lam_ref.min() - 10 * sigma, lam_ref.max() + 10 * sigma, 2000)
    curve = bg.absorption_spectrum(pos, bg.DipoleData(d_r=dip, d_l=dip), grid=grid, sigma=sigma)
    _, ref_vals, _, _ = orc.absorption(lam_ref, x1r, x2r, dip, dip, grid=grid, sigma=sigma)
    assert np.max(np.abs(curve.values - ref_vals)) <= 1e-10 * np.max(np.abs(ref_vals))


def test_tda_overestimation(dev):
    """lambda_j(H) <= lambda_j(A) (Thm 2.5) on the complex config recipe."""
    a, b, _ = configs.config_operator(1, n=64)
    op = bg.make_operator(a, b)
    pos = bg.solve_complex(op)
    lam_a = np.sort(np.linalg.eigvalsh(a))[::-1]
    assert bg.dos_dominance(pos.lambda_plus, lam_a)


def test_absorption_1x1_direct_formula(dev):
    op = bg.make_operator([[2.0]], [[1j]])
    pos = bg.solve_complex(op)
    d = np.array([1.0, 0.0], dtype=complex)
    sigma = 0.05
    grid = np.linspace(1.0, 2.5, 301)
    curve = bg.absorption_spectrum(pos, bg.DipoleData(d_r=d, d_l=d), grid=grid, sigma=sigma)
    x = np.array([pos.x1[0, 0], pos.x2[0, 0]])
    y = np.array([pos.x1[0, 0], -pos.x2[0, 0]])
    weight = ((d.conj() @ x) * (y.conj() @ d) / (y.conj() @ x)).real
    direct = weight * np.exp(-0.5 * ((grid - pos.lambda_plus[0]) / sigma) ** 2) / (np.sqrt(2 * np.pi) * sigma)
    assert np.max(np.abs(curve.values - direct)) <= 1e-13 * np.max(np.abs(direct))


def test_absorption_rejects_degenerate_pairing(dev):
    pos = bg.PositiveEigensystem(lambda_plus=np.array([1.0]), x1=np.eye(1, dtype=complex),
                                 x2=np.eye(1, dtype=complex))
    with pytest.raises(ValueError, match="1e-8"):
        bg.absorption_spectrum(pos, bg.DipoleData(d_r=np.ones(2), d_l=np.ones(2)),
                               grid=np.linspace(0, 2, 5), sigma=0.1)


@pytest.mark.parametrize("n", [3, 300, 4500])
def test_host_entry_matches_device_entry(dev, n):
    """bse_solve_spd_pair_host (pinned-free host buffers, column-blocked D2H
    overlapped with the recovery) gives bit-identical results to the device
    entry used by the Python API."""
    import ctypes as C
    from paper_1501_03830_b200 import _lib
    a, b, _ = configs.config_operator(0, n=n)
    m = np.asfortranarray(a + b)
    k = np.asfortranarray(a - b)
    lam = np.empty(n)
    x1 = np.empty((n, n), order="F")
    x2 = np.empty((n, n), order="F")
    info = _lib.BseInfo()
    st = _lib.load().bse_solve_spd_pair_host(n, m.ctypes.data, n, k.ctypes.data, n,
                                             lam.ctypes.data, x1.ctypes.data, n, x2.ctypes.data, n,
                                             0, C.byref(info))
    assert st == 0, _lib.last_error()
    pos = bg.solve_real(bg.make_operator(a, b, kind="real"))
    assert np.array_equal(lam, pos.lambda_plus)
    assert np.array_equal(x1, pos.x1.real) and np.array_equal(x2, pos.x2.real)
