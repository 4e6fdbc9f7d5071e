"""I/O fixtures from the REFERENCE package itself (build container only):

    python tests/golden/make_io_golden.py

Writes tests/golden/io/: the reference's Matrix Market files for small
random_bse operators (mmio.write_operator, mmio.py:127-135), its eigenvalue
and spectrum CSVs (mmio.py:155-180), a dipole file, and the random_bse
arrays (core.py:245-278) as .npz, so tests/test_cpu_io.py can check that the
drop-in writes byte-identical files and reads the reference's.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent / "io"
sys.path.insert(0, "/root/reference/pkg/src")

import bse  # noqa: E402  (the reference)
from bse import mmio  # noqa: E402


def main():
    HERE.mkdir(exist_ok=True)
    arrays = {}
    for kind, n, seed in (("complex", 5, 1), ("real", 4, 2)):
        op = bse.random_bse(n, seed, kind=kind)
        mmio.write_operator(HERE / f"{kind}_A.mtx", HERE / f"{kind}_B.mtx", op)
        arrays[f"{kind}_a"] = op.a
        arrays[f"{kind}_b"] = op.b
    lam = np.array([3.25, 1.0 / 3.0, -1e-17, -2.5])
    mmio.write_eigenvalues(HERE / "eigenvalues.csv", lam)
    om = np.linspace(-1.0, 1.0, 7)
    mmio.write_spectrum(HERE / "spectrum.csv", om, np.exp(om) / 3.0)
    rng = np.random.default_rng(4)
    d = rng.standard_normal((10, 2)) + 1j * rng.standard_normal((10, 2))
    mmio.write_matrix(HERE / "dipoles.mtx", d)
    dos = bse.spectral_density(np.array([1.0, 1.1, -0.5, 2.0]), sigma=0.05)
    np.savez(HERE / "arrays.npz", lam=lam, om=om, dip=d, dos_omegas=dos.omegas,
             dos_values=dos.values, **arrays)
    print("wrote", sorted(p.name for p in HERE.iterdir()))


if __name__ == "__main__":
    main()
