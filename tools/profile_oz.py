"""One emulated-FP64 product per engine, for ncu.

    python tools/profile_oz.py --m M --n N --k K --engine E [--tb 1] [--chunk C] [--lower]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1501_03830_b200 import _lib  # noqa: E402
from paper_1501_03830_b200.device import mask_array, ptr, stream_ptr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=16384)
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--k", type=int, default=16384)
ap.add_argument("--ta", type=int, default=0)
ap.add_argument("--tb", type=int, default=0)
ap.add_argument("--chunk", type=int, default=4096)
ap.add_argument("--engine", type=int, default=0)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--lower", action="store_true")
a = ap.parse_args()
lib = _lib.load()
dev = torch.device("cuda", 0)
m, n, k = a.m, a.n, a.k
A = torch.randn(max(m, k), max(m, k), dtype=torch.float64, device=dev)
B = torch.randn(max(n, k), max(n, k), dtype=torch.float64, device=dev)
C = torch.zeros(n, m, dtype=torch.float64, device=dev)
lib.bse_oz_set_engine(a.engine)
masks = mask_array(None, None, (None, 0, 0)) if a.lower else None
for _ in range(a.reps + 1):
    assert lib.bse_ozgemm_dev(a.ta, a.tb, m, n, k, 1.0, ptr(A), A.shape[0], ptr(B), B.shape[0], 0.0,
                              ptr(C), m, masks, a.chunk, stream_ptr()) == 0, _lib.last_error()
torch.cuda.synchronize()
print("done", float(C.abs().max()))
