"""Standalone POTRF timing: python tools/bench_potrf.py [--n 16384] [--reps 3]"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1501_03830_b200 import _lib  # noqa: E402
from paper_1501_03830_b200.device import ptr, stream_ptr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
n = a.n
lib = _lib.load()
dev = torch.device("cuda", 0)
G = torch.randn(n, n, dtype=torch.float64, device=dev)
S = G @ G.T + n * torch.eye(n, dtype=torch.float64, device=dev)
W = torch.empty_like(S)
info = _lib.BseInfo()
def run():
    W.copy_(S)
    assert lib.bse_potrf_dev(n, ptr(W), n, stream_ptr(), C.byref(info)) == 0
run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / max(a.reps, 1)
print(f"potrf n={n}: {ms:.2f} ms, {n**3 / 3 / ms / 1e9:.2f} TFLOP/s")
