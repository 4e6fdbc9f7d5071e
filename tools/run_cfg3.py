"""BASELINE config 3 at full size on ONE B200: complex Hermitian BSE n = 16384
(real embedding N = 32768), all eigenpairs, left/right eigenvectors, TDA check.

    python tools/run_cfg3.py [--n 16384] [--cols 256]

Generation (numpy PCG64, seed 3, cfg3 recipe: A = U diag(a) U^H, a ~ U[2,10],
B = (G + G^T)/2 rescaled to ||B||_2 = 0.9 min(a)) runs on the host and is not
timed.  The solve goes through the drop-in ``solve_complex`` (host in, host
out).  Checks on the GPU (torch complex products as the checker) for a
random subset of eigenpairs: ||H x - lam x|| / (||H||_F-bound ||x||), the
biorthogonality block Y^H X - I, positivity / order, and the TDA bound
lam_j(H) <= lam_j(A) from the known spectrum of A."""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1501_03830_b200 as bg  # noqa: E402
from paper_1501_03830_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--cols", type=int, default=256)
a = ap.parse_args()
n = a.n
t0 = time.perf_counter()
A, B, dip, a_sorted = configs.complex_operator(n, seed=3, lo=2.0, hi=10.0, bnorm="0.9min")
tgen = time.perf_counter() - t0
op = bg.make_operator(A, B, kind="complex")
torch.cuda.synchronize()
t0 = time.perf_counter()
pos = bg.solve_complex(op)
tsolve = time.perf_counter() - t0
lam = pos.lambda_plus
dev = torch.device("cuda", 0)
rng = np.random.default_rng(0)
cols = np.sort(rng.choice(n, size=min(a.cols, n), replace=False))
At = torch.from_numpy(A).to(dev)
Bt = torch.from_numpy(B).to(dev)
x1 = torch.from_numpy(np.ascontiguousarray(pos.x1[:, cols])).to(dev)
x2 = torch.from_numpy(np.ascontiguousarray(pos.x2[:, cols])).to(dev)
lt = torch.from_numpy(lam[cols]).to(dev)
top = At @ x1 + Bt @ x2 - x1 * lt
bot = -(Bt.conj() @ x1) - At.conj() @ x2 - x2 * lt
res = torch.sqrt((top.abs() ** 2).sum(0) + (bot.abs() ** 2).sum(0))
xn = torch.sqrt((x1.abs() ** 2).sum(0) + (x2.abs() ** 2).sum(0))
hbound = float(lam[0])  # ||H||_2 >= lam_max; lam_max is the scale of the gate
ratio = (res / (hbound * xn)).max().item()
# biorthogonality on the subset: X1^H X1 - X2^H X2 = I
g = x1.conj().T @ x1 - x2.conj().T @ x2 - torch.eye(len(cols), dtype=x1.dtype, device=dev)
bio = torch.linalg.norm(g).item()
out = {
    "config": f"cfg3 complex BSE n={n} (real embedding N={2 * n}), one B200",
    "generate_s_host": round(tgen, 1), "solve_s_host_in_host_out": round(tsolve, 3),
    "lambda_positive_descending": bool(np.all(lam > 0) and np.all(np.diff(lam) <= 0)),
    "tda_bound_holds": bool(np.all(lam <= a_sorted * (1 + 1e-12))),
    "checked_pairs": int(len(cols)), "max_pair_residual": ratio,
    "biorthogonality_block_fro": bio,
    "gates": {"residual": 1e-13 * n, "biorthogonality": 1e-12 * n},
}
out["pass"] = bool(out["lambda_positive_descending"] and out["tda_bound_holds"]
                   and ratio <= 1e-13 * n and bio <= 1e-12 * n)
print(json.dumps(out))
