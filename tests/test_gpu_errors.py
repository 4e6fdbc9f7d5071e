"""Error semantics through the C ABI (include/bse_b200.h status codes) and
their mapping to the reference's exceptions (kernels.py:25-36, core.py:159-160,
solvers.py:93-98)."""
import ctypes as C
import time

import numpy as np
import pytest

import paper_1501_03830_b200 as bg
from paper_1501_03830_b200 import _lib, configs, solvers
from paper_1501_03830_b200.device import colmajor_empty, ptr, stream_ptr, to_device_colmajor

pytestmark = pytest.mark.gpu


def _solve_status(m, k, flags=0):
    import torch
    dev = torch.device("cuda:0")
    lib = _lib.load()
    n = m.shape[0]
    Mt, ld = to_device_colmajor(m, dev)
    Kt, _ = to_device_colmajor(k, dev)
    X1, ldx = colmajor_empty(n, n, dev)
    X2, _ = colmajor_empty(n, n, dev)
    lam = torch.empty(n, dtype=torch.float64, device=dev)
    wb = lib.bse_solve_workspace_bytes(n, flags & _lib.FLAG_NATIVE_FP64)
    work = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
    info = _lib.BseInfo()
    st = lib.bse_solve_spd_pair_dev(n, ptr(Mt), ld, ptr(Kt), ld, ptr(lam), ptr(X1), ldx, ptr(X2),
                                    ldx, ptr(work), wb, flags, stream_ptr(dev), C.byref(info))
    torch.cuda.synchronize()
    return st, info, lam


def test_unsupported_flags_rejected(dev):
    a, b, _ = configs.config_operator(0, n=16)
    for flags in (0x1, 0x2, 0x8):
        st, _, _ = _solve_status(a + b, a - b, flags)
        assert st == _lib.BSE_BAD_ARGUMENT, flags
        assert "flag" in _lib.last_error()


def test_min_pivot_reported(dev):
    a, b, _ = configs.config_operator(0, n=64)
    st, info, _ = _solve_status(a + b, a - b)
    assert st == _lib.BSE_OK
    assert info.pivot_index == -1 and info.failed_factor == -1
    ref = np.min(np.diagonal(np.linalg.cholesky(a - b))) ** 2
    assert info.min_pivot == pytest.approx(ref, rel=1e-12)


def test_potrf_min_pivot(dev):
    rng = np.random.default_rng(3)
    g = rng.standard_normal((200, 200))
    s = g @ g.T + 200 * np.eye(200)
    At, lda = to_device_colmajor(s, dev)
    info = _lib.BseInfo()
    st = _lib.load().bse_potrf_dev(200, ptr(At), lda, stream_ptr(dev), C.byref(info))
    assert st == _lib.BSE_OK
    ref = np.min(np.diagonal(np.linalg.cholesky(s))) ** 2
    assert info.min_pivot == pytest.approx(ref, rel=1e-12)


def test_k_failure_returns_before_the_reduction(dev):
    """K = A - B indefinite: the status comes back right after the Cholesky
    (no SY2SB/SB2ST/D&C on a partial factor), with A+B probed first."""
    n = 4096
    a, b, _ = configs.config_operator(0, n=n, seed=5)
    m, k = a + b, a - b
    _solve_status(m, k)  # warm-up (workspace, kernels)
    t0 = time.perf_counter()
    _solve_status(m, k)
    t_ok = time.perf_counter() - t0
    k_bad = k.copy()
    k_bad[100, 100] = -5.0
    t0 = time.perf_counter()
    st, info, _ = _solve_status(m, k_bad)
    t_bad = time.perf_counter() - t0
    assert st == _lib.BSE_NOT_POSITIVE_DEFINITE
    assert info.failed_factor == 0 and info.pivot_index == 100
    assert t_bad < 0.6 * t_ok, (t_bad, t_ok)
    # A+B failing too: A+B is reported (the reference factors it first)
    m_bad = m.copy()
    m_bad[7, 7] = -1.0
    st, info, _ = _solve_status(m_bad, k_bad)
    assert st == _lib.BSE_NOT_POSITIVE_DEFINITE
    assert info.failed_factor == 1 and info.pivot_index == 7


def test_stedc_nonfinite_input_is_no_convergence(dev):
    import torch
    lib = _lib.load()
    n = 64
    d = torch.linspace(1.0, 2.0, n, dtype=torch.float64, device=dev)
    e = torch.full((n,), 0.1, dtype=torch.float64, device=dev)
    e[10] = float("nan")
    Q, ldq = colmajor_empty(n, n, dev)
    wb = lib.bse_stedc_workspace_bytes(n)
    work = torch.empty(wb, dtype=torch.uint8, device=dev)
    st = lib.bse_stedc_dev(n, ptr(d), ptr(e), ptr(Q), ldq, ptr(work), wb, stream_ptr(dev))
    assert st == _lib.BSE_NO_CONVERGENCE
    with pytest.raises(bg.ConvergenceError):
        solvers.raise_for_status(st, None, "bse_stedc_dev")


def test_stedc_ok_status(dev):
    import torch
    lib = _lib.load()
    n = 300
    rng = np.random.default_rng(0)
    d = torch.tensor(rng.standard_normal(n), device=dev)
    e = torch.tensor(rng.standard_normal(n), device=dev)
    Q, ldq = colmajor_empty(n, n, dev)
    wb = lib.bse_stedc_workspace_bytes(n)
    work = torch.empty(wb, dtype=torch.uint8, device=dev)
    assert lib.bse_stedc_dev(n, ptr(d), ptr(e), ptr(Q), ldq, ptr(work), wb,
                             stream_ptr(dev)) == _lib.BSE_OK


def test_status_mapping():
    info = _lib.BseInfo()
    info.pivot_index, info.pivot_value, info.failed_factor = 3, -1.5, 1
    with pytest.raises(bg.NotPositiveDefinite) as ei:
        solvers.raise_for_status(_lib.BSE_NOT_POSITIVE_DEFINITE, info, "x")
    assert ei.value.pivot_index == 3 and "A+B" in str(ei.value)
    with pytest.raises(ValueError, match="strictly positive"):
        solvers.raise_for_status(_lib.BSE_SPECTRUM_NOT_POSITIVE, info, "x")
    with pytest.raises(RuntimeError):
        solvers.raise_for_status(_lib.BSE_CUDA_ERROR, info, "x")


def test_host_entry_uses_a_private_pool(dev):
    """The host entry must not change the device's default mempool."""
    import torch
    lib = _lib.load()
    n = 256
    a, b, _ = configs.config_operator(0, n=n)
    from cuda.bindings import runtime as rt  # cuda-python
    err, p = rt.cudaDeviceGetDefaultMemPool(0)
    err, before = rt.cudaMemPoolGetAttribute(p, rt.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold)
    m = np.asfortranarray(a + b)
    k = np.asfortranarray(a - b)
    lam = np.empty(n)
    x1 = np.empty((n, n), order="F")
    x2 = np.empty((n, n), order="F")
    info = _lib.BseInfo()
    st = lib.bse_solve_spd_pair_host(n, m.ctypes.data, n, k.ctypes.data, n, lam.ctypes.data,
                                     x1.ctypes.data, n, x2.ctypes.data, n, 0, C.byref(info))
    assert st == _lib.BSE_OK
    err, after = rt.cudaMemPoolGetAttribute(p, rt.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold)
    assert int(after) == int(before)
    assert lib.bse_release_cached_memory() == _lib.BSE_OK
