"""One warm-up solve then one profiled solve at size n (for ncu launch lists).

    python tools/profile_solve.py --n 8192
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1501_03830_b200 import _lib, configs  # noqa: E402
from paper_1501_03830_b200.device import ptr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--complex", action="store_true",
                help="complex BSE (cfg3 recipe) through bse_solve_complex_dev at block size n")
a = ap.parse_args()
n = a.n
dev = torch.device("cuda", 0)
lib = _lib.load()
if a.complex:
    A, B, _, _ = configs.torch_complex_operator(n, seed=3, device=dev)
    X1 = torch.empty((n, n), dtype=torch.complex128, device=dev)
    X2 = torch.empty_like(X1)
    lam = torch.empty(n, dtype=torch.float64, device=dev)
    wb = lib.bse_solve_complex_workspace_bytes(n, 0)
    work = torch.empty(wb, dtype=torch.uint8, device=dev)
    info = _lib.BseInfo()
    sp = torch.cuda.current_stream().cuda_stream
    torch.cuda.synchronize()
    c0 = lib.bse_launch_count()
    for _ in range(1 + a.reps):
        st = lib.bse_solve_complex_dev(n, ptr(A), n, ptr(B), n, ptr(lam), ptr(X1), n, ptr(X2), n,
                                       ptr(work), wb, 0, sp, C.byref(info))
        assert st == 0, _lib.last_error()
    torch.cuda.synchronize()
    print("launches per complex solve", (lib.bse_launch_count() - c0) // (1 + a.reps))
    sys.exit(0)
S, D, _ = configs.torch_real_operator(n, seed=2, device=dev)
ld = n + (n & 1)
M = torch.zeros((n, ld), dtype=torch.float64, device=dev); M[:, :n] = S
K = torch.zeros((n, ld), dtype=torch.float64, device=dev); K[:, :n] = D
X1 = torch.empty_like(M); X2 = torch.empty_like(M)
lam = torch.empty(n, dtype=torch.float64, device=dev)
wb = lib.bse_solve_workspace_bytes(n, 0)
work = torch.empty(wb, dtype=torch.uint8, device=dev)
info = _lib.BseInfo()
sp = torch.cuda.current_stream().cuda_stream
torch.cuda.synchronize()
c0 = lib.bse_launch_count()
for _ in range(1 + a.reps):
    st = lib.bse_solve_spd_pair_dev(n, ptr(M), ld, ptr(K), ld, ptr(lam), ptr(X1), ld, ptr(X2), ld,
                                    ptr(work), wb, 0, sp, C.byref(info))
    assert st == 0, _lib.last_error()
torch.cuda.synchronize()
print("launches per solve", (lib.bse_launch_count() - c0) // (1 + a.reps))
