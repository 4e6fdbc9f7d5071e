"""Generate golden fixtures by running the REFERENCE package itself.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Only this script touches /root/reference (read-only import, build container
only).  Its outputs (tests/golden/*.npz) pin the numpy oracle
(oracle/bse_oracle.py) and the GPU path; nothing at test time reads the
reference tree.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parents[1]))

import bse  # noqa: E402  (the reference)
from paper_1501_03830_b200 import configs  # noqa: E402


def save(name, **arrays):
    np.savez_compressed(HERE / f"{name}.npz", **arrays)
    print("wrote", name, {k: getattr(v, "shape", None) for k, v in arrays.items()})


def solve_case(name, op, real_too=False, dip=None, sigma=0.05, points=2000):
    pos = bse.solve_complex(op)
    full = bse.expand_full(op, pos)
    r1, r2 = bse.residual_metrics(op, full)
    out = dict(a=op.a, b=op.b, kind=np.array(op.kind), lam=pos.lambda_plus, x1=pos.x1,
               x2=pos.x2, r1=np.array(r1), r2=np.array(r2))
    if real_too:
        rp = bse.solve_real(op)
        out.update(lam_real=rp.lambda_plus, x1_real=rp.x1, x2_real=rp.x2)
    if dip is not None:
        lam = pos.lambda_plus
        grid = np.linspace(lam.min() - 10 * sigma, lam.max() + 10 * sigma, points)
        curve = bse.absorption_spectrum(pos, bse.DipoleData(d_r=dip, d_l=dip), grid=grid,
                                        sigma=sigma)
        out.update(dip=dip, grid=grid, sigma=np.array(sigma), absorption=curve.values,
                   defect=np.array(curve.normalization_defect))
    save(name, **out)


def main():
    # Cholesky known answers + random SPD (kernels.py:43-65)
    rng = np.random.default_rng(7)
    g = rng.standard_normal((40, 40))
    spd = g @ g.T + 40 * np.eye(40)
    save("cholesky", spd=spd, low=bse.cholesky(spd), hand=bse.cholesky(np.array([[4.0, 2.0], [2.0, 5.0]])))

    # Tridiagonal eigensolver (kernels.py:460-535)
    rng = np.random.default_rng(8)
    d = rng.uniform(-2, 2, 60)
    e = rng.uniform(0.1, 1.5, 59)
    vals, vecs = bse.tridiag_eig(bse.SymTridiagonal(diag=d, offdiag=e), which="all")
    alphas = rng.uniform(0.2, 2.0, 39)
    pvals, pvecs = bse.tridiag_eig(bse.SymTridiagonal(diag=np.zeros(40), offdiag=alphas),
                                   which="positive")
    save("tridiag", d=d, e=e, vals=vals, vecs=vecs, alphas=alphas, pvals=pvals, pvecs=pvecs)

    # Skew tridiagonalization (kernels.py:194-213)
    rng = np.random.default_rng(9)
    g = rng.standard_normal((24, 24))
    w = 0.5 * (g - g.T)
    st = bse.skew_tridiagonalize(w)
    save("skew", w=w, alphas=st.alphas, taus=st.taus, q=st.q_matrix())

    # Analytic 1x1 cases (test_solvers.py:20-25, :69-76)
    solve_case("complex_1x1", bse.make_operator([[2.0]], [[1j]]), dip=np.array([1.0, 0.0], complex),
               sigma=0.05, points=301)
    solve_case("real_1x1", bse.make_operator([[2.0]], [[1.0]]), real_too=True)

    # random_bse instances (core.py:245-278)
    solve_case("random_complex_n32_s0", bse.random_bse(32, seed=0))
    solve_case("random_real_n24_s1", bse.random_bse(24, seed=1, kind="real"), real_too=True)

    # BASELINE config recipes at reduced n (same generators as bench/tests)
    a, b, dip = configs.config_operator(0, n=64)
    solve_case("cfg0_n64", bse.make_operator(a, b, kind="real"), real_too=True, dip=dip)
    a, b, dip = configs.config_operator(2, n=96)
    solve_case("cfg2_n96", bse.make_operator(a, b, kind="real"), dip=dip)
    a, b, dip = configs.config_operator(1, n=48)
    solve_case("cfg1_n48", bse.make_operator(a, b, kind="complex"), dip=dip)
    a, b, dip = configs.config_operator(3, n=40)
    solve_case("cfg3_n40", bse.make_operator(a, b, kind="complex"), dip=dip)

    # TDA values of A for the complex config (kernels.py:616-656)
    a, b, _ = configs.config_operator(1, n=48)
    lam_a, _ = bse.hermitian_eig(a, vectors=False)
    save("tda_cfg1_n48", a=a, lam_a=lam_a)


if __name__ == "__main__":
    main()
