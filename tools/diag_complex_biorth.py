"""Biorthogonality diagnostics of the complex extraction (one vector per
doubled eigenvalue + banded polish): per seed, r1/r2 of the reference's
residual_metrics, |G - I| split into the polished band and the rest, and the
r1/r2 after one extra full Newton-Schulz polish on the host."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_1501_03830_b200 as bg  # noqa: E402
from paper_1501_03830_b200 import configs  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    W = 16
    for seed in range(10):
        op = configs.random_bse(n, seed)
        pos = bg.solve_complex(op)
        r1, r2 = bg.residual_metrics(op, bg.expand_full(op, pos))
        x1, x2 = pos.x1, pos.x2
        g = x1.conj().T @ x1 - x2.conj().T @ x2 - np.eye(n)
        i, j = np.indices(g.shape)
        band = np.abs(i - j) <= W
        gb, go = np.linalg.norm(g[band]), np.linalg.norm(g[~band])
        f = 1.5 * np.eye(n) - 0.5 * (g + np.eye(n))
        pp = bg.PositiveEigensystem(lambda_plus=pos.lambda_plus, x1=x1 @ f, x2=x2 @ f)
        q1, q2 = bg.residual_metrics(op, bg.expand_full(op, pp))
        lam = pos.lambda_plus
        gap = np.min(-np.diff(lam)) / lam[0]
        print(f"seed {seed}: r1 {r1:.2e} r2 {r2:.2e} | G-I band {gb:.2e} off-band {go:.2e} "
              f"| full polish r1 {q1:.2e} r2 {q2:.2e} | min rel gap {gap:.2e}", flush=True)


if __name__ == "__main__":
    main()
