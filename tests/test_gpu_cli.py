"""The drop-in CLI (reference cli.py:63-295) end to end on the GPU: solve /
solve-real / compare / spectrum / check / oracle artefacts, metrics.json
fields and exit codes, Matrix Market and binary inputs."""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_1501_03830_b200 as bg
from paper_1501_03830_b200 import cli, configs, mmio

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden" / "io"


def test_solve_matrix_market(dev, tmp_path):
    assert cli.main(["solve", "--a", str(G / "complex_A.mtx"), "--b", str(G / "complex_B.mtx"),
                     "--out", str(tmp_path), "--emit-vectors"]) == cli.EXIT_OK
    m = json.loads((tmp_path / "metrics.json").read_text())
    assert m["command"] == "solve" and m["n"] == 5 and m["kind"] == "complex"
    assert m["r1"] <= 5e-14 and m["r2"] <= 5e-14
    lam = mmio.read_eigenvalues(tmp_path / "eigenvalues.csv")
    op = mmio.load_operator(G / "complex_A.mtx", G / "complex_B.mtx")
    pos = bg.solve_complex(op)
    assert np.array_equal(lam[:5], pos.lambda_plus) and np.array_equal(lam[5:], -pos.lambda_plus[::-1])
    x1, _, _ = mmio.read_matrix(tmp_path / "vectors_x1.mtx")
    assert np.array_equal(x1, pos.x1)


def test_solve_real_binary_inputs(dev, tmp_path):
    op = configs.random_bse(40, 9, kind="real")
    mmio.write_operator(tmp_path / "A.npy", tmp_path / "B.npy", op)
    out = tmp_path / "run"
    assert cli.main(["solve-real", "--a", str(tmp_path / "A.npy"), "--b", str(tmp_path / "B.npy"),
                     "--out", str(out), "--emit-vectors", "--format", "npy"]) == cli.EXIT_OK
    m = json.loads((out / "metrics.json").read_text())
    assert m["r1"] <= 5e-14 and m["r2"] <= 5e-14
    x2 = np.load(out / "vectors_x2.npy")
    assert np.array_equal(x2, bg.solve_real(op).x2)


def test_compare_and_oracle(dev, tmp_path):
    op = configs.random_bse(24, 5, kind="complex")
    mmio.write_operator(tmp_path / "A.mtx", tmp_path / "B.mtx", op)
    args = ["--a", str(tmp_path / "A.mtx"), "--b", str(tmp_path / "B.mtx")]
    assert cli.main(["compare", *args, "--out", str(tmp_path / "c")]) == cli.EXIT_OK
    s = json.loads((tmp_path / "c" / "summary.json").read_text())
    scale = float(np.max(np.abs(np.linalg.eigvals(bg.assemble_h(op)))))
    assert s["max_abs_deviation_solve_vs_oracle"] <= 1e-12 * scale
    assert s["tda_dominance"] and s["tda_min_gap"] >= -1e-12 * scale
    rows = (tmp_path / "c" / "comparison.csv").read_text().splitlines()
    assert rows[0] == "index,lambda_solve,lambda_oracle,lambda_tda,tda_gap" and len(rows) == 49
    assert cli.main(["oracle", *args, "--out", str(tmp_path / "o")]) == cli.EXIT_OK
    vals = mmio.read_eigenvalues(tmp_path / "o" / "eigenvalues.csv")
    ref = np.sort(np.linalg.eigvals(bg.assemble_h(op)).real)[::-1]
    assert np.max(np.abs(vals - ref)) <= 1e-11 * scale


def test_spectrum_with_dipoles(dev, tmp_path):
    op = configs.random_bse(5, 1, kind="complex")
    rng = np.random.default_rng(2)
    d = rng.standard_normal((10, 2)) + 1j * rng.standard_normal((10, 2))
    mmio.write_operator(tmp_path / "A.mtx", tmp_path / "B.mtx", op)
    mmio.write_matrix(tmp_path / "dip.mtx", d)
    rc = cli.main(["spectrum", "--a", str(tmp_path / "A.mtx"), "--b", str(tmp_path / "B.mtx"),
                   "--dipoles", str(tmp_path / "dip.mtx"), "--sigma", "0.1",
                   "--out", str(tmp_path / "s")])
    assert rc == cli.EXIT_OK
    om, val = mmio.read_spectrum(tmp_path / "s" / "absorption.csv")
    pos = bg.solve_complex(op)
    ref = bg.absorption_spectrum(pos, bg.DipoleData(d_r=d[:, 0], d_l=d[:, 1]), grid=om, sigma=0.1)
    assert np.allclose(val, ref.values, rtol=0, atol=1e-12 * np.max(np.abs(ref.values)))


def test_validation_exit_codes(dev, tmp_path):
    n = 4
    mmio.write_matrix(tmp_path / "A.mtx", np.eye(n), symmetry="symmetric")
    mmio.write_matrix(tmp_path / "B.mtx", 2.0 * np.eye(n), symmetry="symmetric")  # A-B = -I
    args = ["--a", str(tmp_path / "A.mtx"), "--b", str(tmp_path / "B.mtx"), "--out", str(tmp_path)]
    assert cli.main(["check", *args]) == cli.EXIT_VALIDATION
    assert cli.main(["solve", *args]) == cli.EXIT_VALIDATION
    assert cli.main(["solve-real", *args]) == cli.EXIT_VALIDATION


def test_tda_values(dev, tmp_path):
    op = configs.random_bse(30, 2, kind="complex")
    mmio.write_matrix(tmp_path / "A.mtx", op.a, symmetry="hermitian")
    assert cli.main(["tda", "--a", str(tmp_path / "A.mtx"), "--out", str(tmp_path)]) == 0
    vals = mmio.read_eigenvalues(tmp_path / "eigenvalues.csv")
    assert np.allclose(vals, np.linalg.eigvalsh(op.a)[::-1], rtol=0, atol=1e-12 * np.abs(vals).max())
