"""Bitwise repeatability of the symmetric eigensolver under contention: P
processes share cuda:0 and each runs bse_syevd_dev R times on the same matrix;
every (w, Z) must equal the first bit for bit.  A difference points at a
timing-dependent stage (the persistent SB2ST kernel, the cooperative panel QR).

    python tools/determinism_probe.py [--n 4608] [--procs 2] [--reps 6] [--native]
"""
import argparse
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np  # noqa: E402


def worker(rank, n, reps, flags, out):
    if flags == -1:
        return worker_stedc(rank, n, reps, out)
    import torch
    from paper_1501_03830_b200 import _lib
    from paper_1501_03830_b200.device import (check, colmajor_empty, ptr, stream_ptr,
                                              to_device_colmajor)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    lib = _lib.load()
    rng = np.random.default_rng(7)
    a = rng.standard_normal((n, n))
    a = a + a.T
    res = []
    wb = lib.bse_syevd_workspace_bytes(n, flags)
    work = torch.empty(wb, dtype=torch.uint8, device=dev)
    for _ in range(reps):
        da, lda = to_device_colmajor(a, dev)
        Z, ldz = colmajor_empty(n, n, dev)
        w = torch.empty(n, dtype=torch.float64, device=dev)
        check(lib.bse_syevd_dev(n, ptr(da), lda, ptr(w), ptr(Z), ldz, ptr(work), wb, flags,
                                stream_ptr()), "syevd")
        torch.cuda.synchronize()
        wh = w.cpu().numpy()
        res.append((hashlib.sha1(wh.tobytes()).hexdigest()[:12],
                    hashlib.sha1(Z.cpu().numpy().tobytes()).hexdigest()[:12], wh))
    out[rank] = res


def worker_stedc(rank, n, reps, out):
    import torch
    from paper_1501_03830_b200 import _lib
    from paper_1501_03830_b200.device import check, colmajor_empty, ptr, stream_ptr
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    lib = _lib.load()
    # the tridiagonal form of the same dense matrix the syevd probe uses
    from scipy.linalg import hessenberg
    rng = np.random.default_rng(7)
    a = rng.standard_normal((n, n))
    t = hessenberg(a + a.T)
    d, e = np.ascontiguousarray(np.diag(t)), np.concatenate([np.diag(t, -1), [0.0]])
    wb = lib.bse_stedc_workspace_bytes(n)
    work = torch.empty(wb, dtype=torch.uint8, device=dev)
    res = []
    for _ in range(reps):
        dd = torch.tensor(d, dtype=torch.float64, device=dev)
        de = torch.tensor(e, dtype=torch.float64, device=dev)
        Q, ldq = colmajor_empty(n, n, dev)
        check(lib.bse_stedc_dev(n, ptr(dd), ptr(de), ptr(Q), ldq, ptr(work), wb, stream_ptr()), "stedc")
        torch.cuda.synchronize()
        wh = dd.cpu().numpy()
        res.append((hashlib.sha1(wh.tobytes()).hexdigest()[:12],
                    hashlib.sha1(Q.cpu().numpy().tobytes()).hexdigest()[:12], wh))
    out[rank] = res


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4608)
    ap.add_argument("--procs", type=int, default=2)
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--native", action="store_true")
    ap.add_argument("--values", action="store_true", help="eigenvalues only: SY2SB + SB2ST + bisection")
    ap.add_argument("--stedc", action="store_true", help="the tridiagonal D&C alone")
    a = ap.parse_args()
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(worker, args=(a.n, a.reps, -1 if a.stedc else (1 if a.values else 0) | (4 if a.native else 0), out), nprocs=a.procs,
                           join=True, start_method="spawn")
        out = dict(out)
    ref = out[0][0]
    bad = 0
    for r in range(a.procs):
        for i, (hw, hz, w) in enumerate(out[r]):
            same = (hw == ref[0], hz == ref[1])
            if not all(same):
                bad += 1
                d = np.max(np.abs(w - ref[2]) / np.maximum(np.abs(ref[2]), 1e-300))
                print(f"proc {r} rep {i}: w equal {same[0]} Z equal {same[1]} max rel dw {d:.3e}")
    print(f"n={a.n} procs={a.procs} reps={a.reps}: {bad} of {a.procs * a.reps} runs differ from the first")
