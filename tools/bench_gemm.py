"""Standalone DMMA GEMM timing (CUDA events) for the engine in csrc/gemm.cu.

    python tools/bench_gemm.py [--n 8192] [--ta 0 --tb 0] [--k K] [--reps 5]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1501_03830_b200 import _lib  # noqa: E402
from paper_1501_03830_b200.device import ptr, stream_ptr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--m", type=int, default=0)
ap.add_argument("--k", type=int, default=0)
ap.add_argument("--ta", type=int, default=0)
ap.add_argument("--tb", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
n, k = a.n, (a.k or a.n)
mm = a.m or n
lib = _lib.load()
dev = torch.device("cuda", 0)
ld = max(n, k, mm)
A = torch.randn(ld, max(mm, k), dtype=torch.float64, device=dev)
B = torch.randn(ld, max(n, k), dtype=torch.float64, device=dev)
C = torch.zeros(n, mm, dtype=torch.float64, device=dev)
def run():
    st = lib.bse_gemm_dev(a.ta, a.tb, mm, n, k, 1.0, ptr(A), ld, ptr(B), ld, 1.0, ptr(C), mm, None,
                          stream_ptr())
    assert st == 0
run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
print(f"m={mm} n={n} k={k} ta={a.ta} tb={a.tb}: {ms:.3f} ms, {2 * mm * n * k / ms / 1e9:.2f} TFLOP/s")
