"""CPU-only checks: the C-ABI library loads and exports every symbol declared
in include/bse_b200.h (no compute calls), the host-side types/transforms
mirror the reference's contracts (core.py, embeddings.py, spectra.py), and
the real 2n-embedding used for complex operators is exact."""
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1501_03830_b200 as bg
from oracle import bse_oracle as orc
from paper_1501_03830_b200 import _lib, configs

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "bse_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*|long long)\s+(bse_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    syms = header_symbols()
    assert "bse_solve_spd_pair_dev" in syms and "bse_potrf_dev" in syms and len(syms) >= 14


def test_library_exports_every_header_symbol():
    lib = _lib.load(strict=True)
    for s in header_symbols():
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} missing from the ctypes table"
    assert lib.bse_version() == 100


def test_workspace_query_is_pure_host():
    lib = _lib.load()
    assert lib.bse_solve_workspace_bytes(0, 0) == 0
    assert lib.bse_solve_workspace_bytes(512, 0) > 4 * 512 * 512 * 8
    assert lib.bse_syevd_workspace_bytes(1000, 0) > 0


def test_make_operator_contracts():
    with pytest.raises(ValueError, match="Hermitian"):
        bg.make_operator([[1.0, 2.0], [0.0, 1.0]], np.zeros((2, 2)))
    with pytest.raises(ValueError, match="symmetric"):
        bg.make_operator(np.eye(2), [[0.0, 1.0], [0.0, 0.0]])
    op = bg.make_operator([[1.0, 2.0], [0.0, 1.0]], np.zeros((2, 2)), symmetrize=True)
    assert op.kind == "real" and np.allclose(op.a, [[1, 1], [1, 1]])
    assert bg.make_operator([[2.0]], [[1j]]).kind == "complex"
    with pytest.raises(ValueError):
        bg.make_operator([[np.nan]], [[0.0]])
    assert not op.a.flags.writeable


def test_positive_eigensystem_contract():
    with pytest.raises(ValueError, match="positive"):
        bg.PositiveEigensystem(lambda_plus=np.array([1.0, -1.0]), x1=np.eye(2), x2=np.eye(2))
    with pytest.raises(ValueError, match="descending"):
        bg.PositiveEigensystem(lambda_plus=np.array([1.0, 2.0]), x1=np.eye(2), x2=np.eye(2))
    pos = bg.PositiveEigensystem(lambda_plus=np.array([2.0, 1.0]), x1=np.eye(2), x2=np.zeros((2, 2)))
    full = bg.expand_full(bg.make_operator(np.diag([2.0, 1.0]), np.zeros((2, 2))), pos)
    assert np.array_equal(full.lam[2:], -full.lam[:2])


def test_build_m_matches_reference_fixtures():
    assert np.array_equal(bg.build_m(bg.make_operator([[2.0]], [[1j]])), [[2.0, -1.0], [-1.0, 2.0]])
    assert np.array_equal(bg.build_m(bg.make_operator([[2.0]], [[1.0]])), np.diag([3.0, 1.0]))


@pytest.mark.parametrize("seed", range(3))
def test_real_embedding_exact(seed):
    """The 2n real BSE built from (A', B') has the spectrum of H with every
    eigenvalue doubled, and M' = S build_m S (same Cholesky pivots)."""
    n = 5
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    a = 0.5 * (g + g.conj().T) + 8 * np.eye(n)
    g2 = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    b = 0.5 * (g2 + g2.T)
    op = bg.make_operator(a, b)
    m, k = bg.real_embedding(op)
    s = np.diag(np.concatenate([np.ones(n), -np.ones(n)]))
    assert np.allclose(m, s @ bg.build_m(op) @ s, atol=1e-14)
    lam_h = np.sort(np.linalg.eigvals(bg.assemble_h(op)).real)[n:]
    lam2 = np.sort(np.sqrt(np.linalg.eigvals(k @ m).real))
    assert np.allclose(lam2[0::2], lam_h, rtol=1e-12) and np.allclose(lam2[1::2], lam_h, rtol=1e-12)


def test_config_generators_shapes():
    a, b, d = configs.config_operator(0, n=16)
    assert a.shape == (16, 16) and d.shape == (32,)
    assert np.all(np.linalg.eigvalsh(a + b) > 0) and np.all(np.linalg.eigvalsh(a - b) > 0)
    a, b, d = configs.config_operator(1, n=12)
    assert np.linalg.norm(b, 2) == pytest.approx(1.0, rel=1e-12)
    assert np.all(np.linalg.eigvalsh(orc.build_m(a, b)) > 0)
    a, b, d = configs.config_operator(4, n=64)
    assert a.shape == (64, 64)


def test_dos_dominance():
    lam = np.array([3.0, 2.0, 1.0])
    assert bg.dos_dominance(lam, lam + 0.1)
    assert not bg.dos_dominance(lam, np.array([3.0, 1.9, 1.0]))


def test_solvers_fail_loudly_without_gpu(monkeypatch):
    import torch
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        bg.solve_real(bg.make_operator([[2.0]], [[1.0]]))
