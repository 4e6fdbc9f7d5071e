"""GPU `validate` (reference: core.validate, core.py:203-232) against the
reference's own pins (pkg/tests/test_core.py:15-42) and the numpy oracle's
left-looking Cholesky of build_m (oracle.bse_oracle.cholesky)."""
import numpy as np
import pytest

import paper_1501_03830_b200 as bg
from oracle import bse_oracle as orc
from paper_1501_03830_b200 import configs

pytestmark = pytest.mark.gpu


def test_validate_positive_1x1(dev):
    rep = bg.validate(bg.make_operator([[2.0]], [[1.0]]))
    assert rep.symmetry_ok and rep.definiteness_ok and rep.ok
    # M = diag(A+B, A-B) = diag(3, 1): smallest pivot is 1
    assert rep.margin == pytest.approx(1.0)


def test_validate_negative_1x1(dev):
    rep = bg.validate(bg.make_operator([[1.0]], [[2.0]]))
    assert rep.symmetry_ok and not rep.definiteness_ok and not rep.ok
    assert rep.margin < 0.0
    assert rep.margin == pytest.approx(-1.0)  # A-B = -1 is the failing pivot


def test_validate_non_hermitian(dev):
    op = bg.BseOperator(a=np.array([[0.0, 1.0], [0.0, 0.0]]), b=np.zeros((2, 2)), kind="real")
    rep = bg.validate(op)
    assert not rep.symmetry_ok
    assert rep.sym_defects[0] > 0.1


def test_validate_does_not_mutate(dev):
    op = bg.make_operator([[2.0]], [[1j]])
    a_before = op.a.copy()
    bg.validate(op)
    assert np.array_equal(op.a, a_before)


@pytest.mark.parametrize("kind,n", [("real", 64), ("real", 300), ("complex", 48), ("complex", 150)])
def test_validate_margin_matches_oracle(dev, kind, n):
    idx = 0 if kind == "real" else 1
    a, b, _ = configs.config_operator(idx, n=n)
    op = bg.make_operator(a, b, kind=kind)
    rep = bg.validate(op)
    low = orc.cholesky(orc.build_m(op.a, op.b))
    ref = float(np.min(np.diagonal(low)) ** 2)
    assert rep.ok
    assert abs(rep.margin - ref) <= 1e-12 * ref


@pytest.mark.parametrize("kind", ["real", "complex"])
def test_validate_indefinite_matches_oracle(dev, kind):
    n = 40
    idx = 0 if kind == "real" else 1
    a, b, _ = configs.config_operator(idx, n=n)
    # shift so that A-B (real) / the embedding (complex) loses definiteness
    if kind == "real":
        b = b + np.linalg.eigvalsh(a - b)[5] * np.eye(n)
    else:
        b = b * 40.0
    op = bg.make_operator(a, b, kind=kind)
    rep = bg.validate(op)
    with pytest.raises(orc.NotPositiveDefinite) as ei:
        orc.cholesky(orc.build_m(op.a, op.b))
    assert not rep.definiteness_ok
    assert rep.margin <= 0.0
    assert abs(rep.margin - ei.value.pivot_value) <= 1e-9 * max(1.0, abs(ei.value.pivot_value))
