"""Emulated-FP64 (Ozaki II on tcgen05 int8) vs DMMA GEMM timing, CUDA events.

    python tools/bench_ozgemm.py [--m M --n N --k K] [--ta 0 --tb 0] [--chunk C]

The ozgemm time includes the slicing, the 16 batched int8 products and the
CRT reconstruction; its workspace is allocated once outside the timed loop
(bse_ozgemm_dev allocates per call from the stream-ordered pool)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1501_03830_b200 import _lib  # noqa: E402
from paper_1501_03830_b200.device import ptr, stream_ptr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=16384)
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--k", type=int, default=16384)
ap.add_argument("--ta", type=int, default=0)
ap.add_argument("--tb", type=int, default=0)
ap.add_argument("--chunk", type=int, default=4096)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--engines", default="2,1,0", help="emulated-engine kernels to time (bse_oz_set_engine)")
ap.add_argument("--no-dmma", action="store_true")
a = ap.parse_args()
m, n, k = a.m, a.n, a.k
lib = _lib.load()
dev = torch.device("cuda", 0)
# keep the pool's freed workspace mapped between calls
pool = torch.cuda.memory  # noqa: F841
A = torch.randn(max(m, k), max(m, k), dtype=torch.float64, device=dev) / k ** 0.5
B = torch.randn(max(n, k), max(n, k), dtype=torch.float64, device=dev)
lda = ldb = A.shape[0]
C0 = torch.zeros(n, m, dtype=torch.float64, device=dev)
C1 = torch.zeros(n, m, dtype=torch.float64, device=dev)


def dmma():
    assert lib.bse_gemm_dev(a.ta, a.tb, m, n, k, 1.0, ptr(A), lda, ptr(B), ldb, 0.0, ptr(C0), m,
                            None, stream_ptr()) == 0


def oz():
    assert lib.bse_ozgemm_dev(a.ta, a.tb, m, n, k, 1.0, ptr(A), lda, ptr(B), ldb, 0.0, ptr(C1), m,
                              None, a.chunk, stream_ptr()) == 0, _lib.last_error()


def timed(name, fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    print(f"{name:18s} m={m} n={n} k={k} ta={a.ta} tb={a.tb}: {ms:8.3f} ms, "
          f"{2 * m * n * k / ms / 1e9:7.2f} TFLOP/s (FP64-equivalent)", flush=True)


if not a.no_dmma:
    timed("dmma", dmma)
ref = None
for eng in [int(x) for x in a.engines.split(",")]:
    lib.bse_oz_set_engine(eng)
    timed(f"ozaki engine {eng}", oz)
    if ref is None:
        ref = C1.clone()
    else:
        print(f"  bitwise equal to the first engine: {bool(torch.equal(ref, C1))}")
if not a.no_dmma:
    d = (C0 - C1).abs().max().item()
    print(f"max |dmma - ozaki| = {d:.3e}  (max |C| = {C0.abs().max().item():.3e})")
