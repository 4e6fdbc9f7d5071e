"""Pin the CPU oracle (oracle/bse_oracle.py) against outputs of the reference
package itself (tests/golden/*.npz, made by tests/golden/make_golden.py)."""
from pathlib import Path

import numpy as np
import pytest

from oracle import bse_oracle as orc

G = Path(__file__).resolve().parent / "golden"


def load(name):
    return dict(np.load(G / f"{name}.npz", allow_pickle=False))


def test_cholesky_golden():
    z = load("cholesky")
    assert np.array_equal(orc.cholesky(np.array([[4.0, 2.0], [2.0, 5.0]])), z["hand"])
    assert np.max(np.abs(orc.cholesky(z["spd"]) - z["low"])) <= 1e-14 * np.max(np.abs(z["low"]))


def test_cholesky_pivot_report():
    with pytest.raises(orc.NotPositiveDefinite) as exc:
        orc.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert exc.value.pivot_index == 1 and exc.value.pivot_value == pytest.approx(-3.0)


def test_tridiag_golden():
    z = load("tridiag")
    vals, vecs = orc.tridiag_eig(z["d"], z["e"], which="all")
    assert np.max(np.abs(vals - z["vals"])) <= 1e-14 * np.max(np.abs(z["vals"]))
    assert np.max(np.abs(vecs - z["vecs"])) <= 1e-12
    pv, pvec = orc.tridiag_eig(np.zeros(40), z["alphas"], which="positive")
    assert np.max(np.abs(pv - z["pvals"])) <= 1e-14 * np.max(pv)
    assert np.max(np.abs(pvec - z["pvecs"])) <= 1e-12


def test_skew_golden():
    z = load("skew")
    _, sub, store, taus = orc.tridiagonalize(z["w"], skew=True)
    assert np.max(np.abs(-sub - z["alphas"])) <= 1e-13
    q = orc.apply_reflectors(store, taus, np.eye(24))
    assert np.max(np.abs(q - z["q"])) <= 1e-13


@pytest.mark.parametrize("name", ["complex_1x1", "real_1x1", "random_complex_n32_s0",
                                  "random_real_n24_s1", "cfg0_n64", "cfg2_n96", "cfg1_n48",
                                  "cfg3_n40"])
def test_solve_complex_golden(name):
    z = load(name)
    lam, x1, x2 = orc.solve_complex(z["a"], z["b"])
    assert np.max(np.abs(lam - z["lam"])) <= 1e-13 * z["lam"][0]
    scale = max(1.0, np.max(np.abs(z["x1"])))
    assert np.max(np.abs(x1 - z["x1"])) <= 1e-11 * scale
    assert np.max(np.abs(x2 - z["x2"])) <= 1e-11 * scale
    r1, r2 = orc.residual_metrics(z["a"], z["b"], x1, x2, lam)
    assert r1 == pytest.approx(float(z["r1"]), rel=0.5, abs=1e-15)
    assert r2 == pytest.approx(float(z["r2"]), rel=0.5, abs=1e-15)
    if "absorption" in z:
        grid, vals, _, defect = orc.absorption(lam, x1, x2, z["dip"], z["dip"], grid=z["grid"],
                                               sigma=float(z["sigma"]))
        ref = z["absorption"]
        assert np.max(np.abs(vals - ref)) <= 1e-11 * np.max(np.abs(ref))


@pytest.mark.parametrize("name", ["real_1x1", "random_real_n24_s1", "cfg0_n64"])
def test_solve_real_golden(name):
    z = load(name)
    lam, x1, x2 = orc.solve_real(z["a"].real, z["b"].real)
    assert np.max(np.abs(lam - z["lam_real"])) <= 1e-13 * z["lam_real"][0]
    assert np.max(np.abs(x1 - z["x1_real"].real)) <= 1e-10
    assert np.max(np.abs(x2 - z["x2_real"].real)) <= 1e-10


def test_tda_golden():
    z = load("tda_cfg1_n48")
    lam_a = orc.hermitian_eigvals(z["a"])
    assert np.max(np.abs(lam_a - z["lam_a"])) <= 1e-13 * np.max(np.abs(z["lam_a"]))


def test_real_1x1_closed_form():
    # test_solvers.py:69-76: X1 = (1+sqrt3)/(2*3^(1/4)), X2 = (1-sqrt3)/(2*3^(1/4))
    lam, x1, x2 = orc.solve_real(np.array([[2.0]]), np.array([[1.0]]))
    root = 3.0 ** 0.25
    assert lam[0] == pytest.approx(np.sqrt(3.0), abs=1e-15)
    assert x1[0, 0] == pytest.approx((1.0 + np.sqrt(3.0)) / (2.0 * root), abs=1e-14)
    assert x2[0, 0] == pytest.approx((1.0 - np.sqrt(3.0)) / (2.0 * root), abs=1e-14)
