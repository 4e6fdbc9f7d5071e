"""Per-rank cost of the column-sharded solve, measured on ONE GPU.

    python tools/dist_projection.py --n 16384 --worlds 1 2 4 8

For each world size P, runs the exact kernels rank 0 of a P-GPU solve
executes (bse_comm_create_solo: same column blocks, no exchange) and reports
the device time and stage breakdown.  The exchanges a real P-GPU run adds are
three column all-gathers (W, X1, X2: 3 n^2 doubles in total, each rank
receiving (P-1)/P of it over NVLink 5); their volume is printed beside the
compute time.  This is a measurement of per-rank compute, not a multi-GPU
number.
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1501_03830_b200 import _lib, configs  # noqa: E402
from paper_1501_03830_b200.device import ptr  # noqa: E402
from paper_1501_03830_b200.distributed import Communicator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--worlds", type=int, nargs="+", default=[1, 2, 4, 8])
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
n = a.n
dev = torch.device("cuda", 0)
lib = _lib.load()
S, D, _ = configs.torch_real_operator(n, seed=2, device=dev)
ld = n + (n & 1)
M = torch.zeros((n, ld), dtype=torch.float64, device=dev); M[:, :n] = S
K = torch.zeros((n, ld), dtype=torch.float64, device=dev); K[:, :n] = D
del S, D
X1 = torch.empty_like(M); X2 = torch.empty_like(M)
lam = torch.empty(n, dtype=torch.float64, device=dev)
wb = lib.bse_solve_workspace_bytes(n, 0)
work = torch.empty(wb, dtype=torch.uint8, device=dev)
info = _lib.BseInfo()
sp = torch.cuda.current_stream().cuda_stream
for P in a.worlds:
    comm = Communicator.solo(0, P)

    def solve():
        st = lib.bse_solve_spd_pair_dist_dev(comm.handle, n, ptr(M), ld, ptr(K), ld, ptr(lam),
                                             ptr(X1), ld, ptr(X2), ld, ptr(work), wb, 0, sp,
                                             C.byref(info))
        assert st == 0, _lib.last_error()
    solve()
    torch.cuda.synchronize()
    lib.bse_profile_enable(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        solve()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    msarr = (C.c_double * 4096)()
    names = C.create_string_buffer(32 * 4096)
    cnt = lib.bse_profile_read(4096, msarr, names)
    lib.bse_profile_enable(0)
    stages = {}
    for i in range(cnt):
        nm = names.raw[32 * i:32 * (i + 1)].split(b"\0")[0].decode()
        if nm != "end":
            stages[nm] = round(stages.get(nm, 0.0) + msarr[i] / a.reps, 2)
    gather_bytes = 3 * n * n * 8 * (P - 1) / P
    print(json.dumps({"world": P, "n": n, "rank0_compute_ms": round(ms, 1),
                      "allgather_bytes_received_per_rank": gather_bytes,
                      "stages_ms": stages}), flush=True)
    comm.close()
