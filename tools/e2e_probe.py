"""Where the e2e (host-buffer) solve spends its time beyond the device solve:
pinned H2D / D2H bandwidth, the device entry, and the host entry with its
stage events (bse_profile_enable records on the entry's internal stream).

    python tools/e2e_probe.py [--n 16384]
"""
import argparse
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1501_03830_b200 import _lib, configs  # noqa: E402
from paper_1501_03830_b200.device import ptr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
a = ap.parse_args()
n = a.n
dev = torch.device("cuda", 0)
lib = _lib.load()
S, D, _ = configs.torch_real_operator(n, seed=2, device=dev)
Mh = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
Kh = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
Mh.copy_(S)
Kh.copy_(D)
X1h = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
X2h = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
lamh = torch.empty(n, dtype=torch.float64, pin_memory=True)
dbuf = torch.empty((n, n), dtype=torch.float64, device=dev)
torch.cuda.synchronize()
for name, fn in (("h2d", lambda: dbuf.copy_(Mh, non_blocking=True)),
                 ("d2h", lambda: X1h.copy_(dbuf, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{name}: {dt * 1e3:.1f} ms for {n * n * 8 / 1e9:.2f} GB = {n * n * 8 / dt / 1e9:.1f} GB/s")
info = _lib.BseInfo()


def host():
    st = lib.bse_solve_spd_pair_host(n, ptr(Mh), n, ptr(Kh), n, ptr(lamh), ptr(X1h), n, ptr(X2h),
                                     n, 0, C.byref(info))
    assert st == 0, _lib.last_error()


host()
lib.bse_profile_enable(1)
t0 = time.perf_counter()
host()
dt = time.perf_counter() - t0
cap = 4096
ms = (C.c_double * cap)()
names = C.create_string_buffer(cap * 32)
k = lib.bse_profile_read(cap, ms, names)
print(f"host entry: {dt * 1e3:.1f} ms wall; {k} stage intervals")
raw = names.raw
agg = {}
for i in range(k):
    nm = raw[i * 32:(i + 1) * 32].split(b"\0")[0].decode()
    agg[nm] = agg.get(nm, 0.0) + ms[i]
for nm, v in agg.items():
    print(f"  {nm:16s} {v:8.2f} ms")
print(f"  {'sum':16s} {sum(agg.values()):8.2f} ms")
lib.bse_profile_enable(0)
