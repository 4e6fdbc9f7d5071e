"""CPU tests of the drop-in's I/O and CLI plumbing against
files written by the reference itself (tests/golden/io, made by
tests/golden/make_io_golden.py): byte-identical writers, readers that
accept the reference's files, the binary (.npy) format, random_bse, the
host DOS, and the CLI's I/O exit codes (no GPU needed for these)."""
from pathlib import Path

import numpy as np
import pytest

from paper_1501_03830_b200 import cli, configs, mmio
from paper_1501_03830_b200.spectra import spectral_density

G = Path(__file__).resolve().parent / "golden" / "io"
Z = np.load(G / "arrays.npz")


@pytest.mark.parametrize("kind", ["complex", "real"])
def test_random_bse_and_operator_files_match_reference(tmp_path, kind):
    n, seed = (5, 1) if kind == "complex" else (4, 2)
    op = configs.random_bse(n, seed, kind=kind)
    assert np.array_equal(op.a, Z[f"{kind}_a"]) and np.array_equal(op.b, Z[f"{kind}_b"])
    mmio.write_operator(tmp_path / "A.mtx", tmp_path / "B.mtx", op)
    assert (tmp_path / "A.mtx").read_bytes() == (G / f"{kind}_A.mtx").read_bytes()
    assert (tmp_path / "B.mtx").read_bytes() == (G / f"{kind}_B.mtx").read_bytes()
    back = mmio.load_operator(G / f"{kind}_A.mtx", G / f"{kind}_B.mtx")
    assert back.kind == kind
    assert np.array_equal(back.a, op.a) and np.array_equal(back.b, op.b)


def test_csv_writers_byte_identical(tmp_path):
    mmio.write_eigenvalues(tmp_path / "e.csv", Z["lam"])
    assert (tmp_path / "e.csv").read_bytes() == (G / "eigenvalues.csv").read_bytes()
    assert np.array_equal(mmio.read_eigenvalues(G / "eigenvalues.csv"), Z["lam"])
    mmio.write_spectrum(tmp_path / "s.csv", Z["om"], np.exp(Z["om"]) / 3.0)
    assert (tmp_path / "s.csv").read_bytes() == (G / "spectrum.csv").read_bytes()
    om, val = mmio.read_spectrum(G / "spectrum.csv")
    assert np.array_equal(om, Z["om"])


def test_dipoles_and_dos_match_reference():
    d_r, d_l = mmio.load_dipoles(G / "dipoles.mtx")
    assert np.array_equal(d_r, Z["dip"][:, 0]) and np.array_equal(d_l, Z["dip"][:, 1])
    dos = spectral_density(np.array([1.0, 1.1, -0.5, 2.0]), sigma=0.05)
    assert np.array_equal(dos.omegas, Z["dos_omegas"])
    assert np.array_equal(dos.values, Z["dos_values"])  # same accumulation order


def test_binary_roundtrip_is_memory_mapped(tmp_path):
    op = configs.random_bse(7, 3, kind="complex")
    mmio.write_operator(tmp_path / "A.npy", tmp_path / "B.npy", op)
    a, field, _ = mmio.read_binary(tmp_path / "A.npy")
    assert isinstance(a, np.memmap) and field == "complex"
    back = mmio.load_operator(tmp_path / "A.npy", tmp_path / "B.npy")
    assert np.array_equal(back.a, op.a) and np.array_equal(back.b, op.b)
    opr = configs.random_bse(6, 4, kind="real")
    mmio.write_operator(tmp_path / "Ar.npy", tmp_path / "Br.npy", opr)
    assert mmio.read_binary(tmp_path / "Ar.npy")[0].dtype == np.float64
    assert mmio.load_operator(tmp_path / "Ar.npy", tmp_path / "Br.npy").kind == "real"


def test_format_errors(tmp_path):
    bad = tmp_path / "bad.mtx"
    bad.write_text("not a header\n")
    with pytest.raises(mmio.FormatError):
        mmio.read_matrix(bad)
    np.save(tmp_path / "i.npy", np.zeros((3, 3), dtype=np.int32))
    with pytest.raises(mmio.FormatError):
        mmio.read_binary(tmp_path / "i.npy")
    with pytest.raises(mmio.FormatError):  # complex file requested as real
        mmio.load_operator(G / "complex_A.mtx", G / "complex_B.mtx", kind="real")


def test_cli_io_exit_codes(tmp_path):
    assert cli.main(["solve", "--a", str(tmp_path / "missing.mtx"), "--b",
                     str(tmp_path / "missing.mtx"), "--out", str(tmp_path)]) == cli.EXIT_IO
    assert cli.main(["solve", "--a", str(G / "real_A.mtx"), "--out", str(tmp_path)]) == cli.EXIT_IO
    assert cli.main(["spectrum", "--eigenvalues", str(G / "eigenvalues.csv"), "--dipoles",
                     str(G / "dipoles.mtx"), "--out", str(tmp_path)]) == cli.EXIT_IO


def test_cli_gen_and_dos_from_eigenvalues(tmp_path):
    assert cli.main(["gen", "--n", "5", "--seed", "1", "--out", str(tmp_path)]) == 0
    assert (tmp_path / "A.mtx").read_bytes() == (G / "complex_A.mtx").read_bytes()
    assert cli.main(["gen", "--config", "0", "--n", "16", "--format", "npy",
                     "--out", str(tmp_path / "c0")]) == 0
    op = mmio.load_operator(tmp_path / "c0" / "A.npy", tmp_path / "c0" / "B.npy")
    a, b, _ = configs.config_operator(0, n=16)
    assert np.array_equal(op.a.real, a) and op.kind == "real"
    assert mmio.read_binary(tmp_path / "c0" / "dipoles.npy")[0].shape == (32, 2)
    rc = cli.main(["spectrum", "--eigenvalues", str(G / "eigenvalues.csv"), "--grid=-3:4:11",
                   "--out", str(tmp_path / "s")])
    assert rc == 0
    om, val = mmio.read_spectrum(tmp_path / "s" / "dos.csv")
    assert om.shape == (11,) and np.all(val >= 0)
