"""GPU parity of the eigensolver stages: tridiagonal divide and conquer
(bse_stedc_dev) and the two-stage symmetric eigensolver (bse_syevd_dev),
against numpy's LAPACK (float64) and structural properties."""
import numpy as np
import pytest

from paper_1501_03830_b200 import _lib
from paper_1501_03830_b200.device import (check, colmajor_empty, from_device_colmajor, ptr,
                                          stream_ptr, to_device_colmajor)

from conftest import random_symmetric

pytestmark = pytest.mark.gpu


def run_stedc(d, e, dev):
    import torch
    lib = _lib.load()
    n = d.shape[0]
    dd = torch.tensor(d, dtype=torch.float64, device=dev)
    de = torch.tensor(np.concatenate([e, [0.0]]), dtype=torch.float64, device=dev)
    Q, ldq = colmajor_empty(n, n, dev)
    wb = lib.bse_stedc_workspace_bytes(n)
    work = torch.empty(wb, dtype=torch.uint8, device=dev)
    check(lib.bse_stedc_dev(n, ptr(dd), ptr(de), ptr(Q), ldq, ptr(work), wb, stream_ptr()), "stedc")
    return dd.cpu().numpy(), from_device_colmajor(Q, n, n)


def run_syevd(a, dev):
    import torch
    lib = _lib.load()
    n = a.shape[0]
    da, lda = to_device_colmajor(a, dev)
    Z, ldz = colmajor_empty(n, n, dev)
    w = torch.empty(n, dtype=torch.float64, device=dev)
    wb = lib.bse_syevd_workspace_bytes(n, 0)
    work = torch.empty(wb, dtype=torch.uint8, device=dev)
    check(lib.bse_syevd_dev(n, ptr(da), lda, ptr(w), ptr(Z), ldz, ptr(work), wb, 0, stream_ptr()),
          "syevd")
    return w.cpu().numpy(), from_device_colmajor(Z, n, n)


def tri_cases():
    rng = np.random.default_rng(3)
    out = []
    for n in (1, 2, 3, 7, 64, 100, 257, 1000, 2049):
        out.append((f"random{n}", rng.uniform(-2, 2, n), rng.uniform(-1, 1, max(n - 1, 0))))
    n = 300
    out.append(("toeplitz", np.zeros(n), np.ones(n - 1)))
    out.append(("identity", np.ones(n), np.zeros(n - 1)))
    out.append(("clustered", np.repeat(rng.uniform(1, 2, 30), 10), 1e-10 * rng.standard_normal(n - 1)))
    out.append(("wilkinson21", np.abs(np.arange(21) - 10.0), np.ones(20)))
    out.append(("zero_diag", np.zeros(n), rng.uniform(0.2, 2, n - 1)))
    out.append(("graded", np.arange(n) * 1.0, 1e-8 * np.ones(n - 1)))
    out.append(("glued_wilkinson", np.tile(np.abs(np.arange(21) - 10.0), 10),
                np.where(np.arange(209) % 21 == 20, 1e-9, 1.0)))
    return out


@pytest.mark.parametrize("name,d,e", tri_cases(), ids=[c[0] for c in tri_cases()])
def test_stedc(dev, name, d, e):
    n = d.shape[0]
    w, Q = run_stedc(d, e, dev)
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    w0 = np.linalg.eigvalsh(T)
    nrm = max(np.abs(w0).max(), 1e-300)
    assert np.all(np.diff(w) >= 0)
    assert np.abs(w - w0).max() <= 1e-13 * nrm * max(1.0, np.log2(n + 1))
    assert np.abs(T @ Q - Q * w).max() <= 1e-13 * nrm * max(1.0, np.log2(n + 1))
    assert np.abs(Q.T @ Q - np.eye(n)).max() <= 1e-13 * max(1.0, np.log2(n + 1))


@pytest.mark.parametrize("n", [1, 2, 3, 5, 63, 64, 65, 66, 67, 128, 130, 200, 513, 1000, 2000])
def test_syevd_random(dev, n):
    a = random_symmetric(n, n)
    w, Z = run_syevd(a, dev)
    w0 = np.linalg.eigvalsh(a)
    nrm = np.abs(w0).max()
    assert np.abs(w - w0).max() <= 2e-14 * n * nrm + 1e-300
    assert np.abs(a @ Z - Z * w).max() <= 2e-14 * n * nrm
    assert np.abs(Z.T @ Z - np.eye(n)).max() <= 1e-14 * n


def test_syevd_clustered(dev):
    # commuting-cluster stress: repeated eigenvalues
    n = 600
    rng = np.random.default_rng(4)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    vals = np.repeat(rng.uniform(1, 10, 20), 30) * (1 + 1e-12 * rng.uniform(-1, 1, n))
    a = (q * vals) @ q.T
    a = 0.5 * (a + a.T)
    w, Z = run_syevd(a, dev)
    assert np.abs(w - np.sort(vals)).max() <= 1e-12 * 10
    assert np.abs(a @ Z - Z * w).max() <= 1e-12 * 10
    assert np.abs(Z.T @ Z - np.eye(n)).max() <= 1e-12


_SB2ST_HASH_SCRIPT = r"""
import hashlib, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
from paper_1501_03830_b200 import _lib
from paper_1501_03830_b200.device import check, colmajor_empty, ptr, stream_ptr, to_device_colmajor
dev = torch.device("cuda", 0)
lib = _lib.load()
n = 2000
rng = np.random.default_rng(5)
a = rng.standard_normal((n, n)); a = a + a.T
out = []
for _ in range(3):
    da, lda = to_device_colmajor(a, dev)
    Z, ldz = colmajor_empty(n, n, dev)
    w = torch.empty(n, dtype=torch.float64, device=dev)
    wb = lib.bse_syevd_workspace_bytes(n, 1)
    work = torch.empty(wb, dtype=torch.uint8, device=dev)
    check(lib.bse_syevd_dev(n, ptr(da), lda, ptr(w), ptr(Z), ldz, ptr(work), wb, 1, stream_ptr()), "syevd")
    torch.cuda.synchronize()
    out.append(hashlib.sha1(w.cpu().numpy().tobytes()).hexdigest())
print("HASHES", *out)
"""


def test_sb2st_result_independent_of_handoff_timing(dev):
    """Regression for the cross-sweep race fixed in round 2:
    with pseudo-random delays of up to 16 us injected before the bulk stores of
    warps 1-7 (BSE_SB2ST_MODE=264) -- which made every run differ before the
    fix -- the band -> tridiagonal stage must give bit-identical eigenvalues,
    equal to the undisturbed run's.  (The mode is read once per process, hence
    the subprocesses.)"""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parents[1])
    script = _SB2ST_HASH_SCRIPT.format(root=root)

    def run(mode):
        env = dict(os.environ)
        env.pop("BSE_SB2ST_MODE", None)
        if mode:
            env["BSE_SB2ST_MODE"] = str(mode)
        res = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True,
                             timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        line = [ln for ln in res.stdout.splitlines() if ln.startswith("HASHES")][-1]
        return line.split()[1:]

    plain = run(0)
    delayed = run(264)
    uniform = run(72)
    assert len(set(plain)) == 1
    assert set(delayed) == set(plain) and set(uniform) == set(plain)
