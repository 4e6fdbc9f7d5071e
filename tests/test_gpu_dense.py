"""GPU parity of the dense building blocks (DMMA GEMM engine, POTRF, TRSM)
against float64 references (numpy / torch).  Cholesky pins follow the
reference's kernel tests (pkg/tests/test_kernels.py:20-47)."""
import ctypes as C

import numpy as np
import pytest

from paper_1501_03830_b200 import _lib
from paper_1501_03830_b200.device import (check, from_device_colmajor, mask_array, ptr,
                                          stream_ptr, to_device_colmajor)

from conftest import random_spd_real

pytestmark = pytest.mark.gpu


def _band(a, lo, hi, unit):
    r, c = np.indices(a.shape)
    d = c - r
    keep = np.ones(a.shape, bool)
    if lo is not None:
        keep &= d >= lo
    if hi is not None:
        keep &= d <= hi
    out = np.where(keep, a, 0.0)
    if unit:
        out = np.where(d == 0, 1.0, out)
    return out


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 5, 3), (64, 64, 64), (130, 257, 77),
                                   (300, 129, 1000), (513, 511, 256)])
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_gemm_plain(dev, M, N, K, ta, tb):
    lib = _lib.load()
    rng = np.random.default_rng(M * 7 + N * 3 + K + ta * 11 + tb * 13)
    a = rng.standard_normal((K, M) if ta else (M, K))
    b = rng.standard_normal((N, K) if tb else (K, N))
    c = rng.standard_normal((M, N))
    da, lda = to_device_colmajor(a, dev)
    db, ldb = to_device_colmajor(b, dev)
    dc, ldc = to_device_colmajor(c, dev)
    check(lib.bse_gemm_dev(ta, tb, M, N, K, 1.5, ptr(da), lda, ptr(db), ldb, -0.5, ptr(dc), ldc,
                           None, stream_ptr()), "gemm")
    got = from_device_colmajor(dc, M, N)
    ref = 1.5 * ((a.T if ta else a) @ (b.T if tb else b)) - 0.5 * c
    assert np.max(np.abs(got - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref))) * np.sqrt(K)


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("case", ["lowerA", "unitA", "strictB", "upperA_lowerC", "lowerB_upperC"])
def test_gemm_masks(dev, ta, tb, case):
    lib = _lib.load()
    M, N, K = 200, 190, 200
    rng = np.random.default_rng(5)
    a = rng.standard_normal((K, M) if ta else (M, K))
    b = rng.standard_normal((N, K) if tb else (K, N))
    c = rng.standard_normal((M, N))
    ma = mb = mc = None
    if case == "lowerA":
        ma = (None, 0, 0)
    elif case == "unitA":
        ma = (None, -1, 1)
    elif case == "strictB":
        mb = (None, -1, 0)
    elif case == "upperA_lowerC":
        ma, mc = (0, None, 0), (None, 0, 0)
    else:
        mb, mc = (None, 0, 0), (0, None, 0)
    am = _band(a, *ma) if ma else a
    bm = _band(b, *mb) if mb else b
    ref = 0.75 * ((am.T if ta else am) @ (bm.T if tb else bm)) + 2.0 * c
    if mc:
        ref = np.where(_band(np.ones_like(c), *mc) != 0, ref, c)
    da, lda = to_device_colmajor(a, dev)
    db, ldb = to_device_colmajor(b, dev)
    dc, ldc = to_device_colmajor(c, dev)
    check(lib.bse_gemm_dev(ta, tb, M, N, K, 0.75, ptr(da), lda, ptr(db), ldb, 2.0, ptr(dc), ldc,
                           mask_array(ma, mb, mc), stream_ptr()), "gemm")
    got = from_device_colmajor(dc, M, N)
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_cholesky_hand_expansion(dev):
    lib = _lib.load()
    a = np.array([[4.0, 2.0], [2.0, 5.0]])
    da, lda = to_device_colmajor(a, dev)
    info = _lib.BseInfo()
    check(lib.bse_potrf_dev(2, ptr(da), lda, stream_ptr(), C.byref(info)), "potrf")
    assert np.array_equal(from_device_colmajor(da, 2, 2), np.array([[2.0, 0.0], [1.0, 2.0]]))


def test_cholesky_indefinite_reports_pivot(dev):
    lib = _lib.load()
    da, lda = to_device_colmajor(np.array([[1.0, 2.0], [2.0, 1.0]]), dev)
    info = _lib.BseInfo()
    st = lib.bse_potrf_dev(2, ptr(da), lda, stream_ptr(), C.byref(info))
    assert st == _lib.BSE_NOT_POSITIVE_DEFINITE
    assert info.pivot_index == 1
    assert info.pivot_value == pytest.approx(-3.0)


@pytest.mark.parametrize("n", [1, 5, 64, 65, 127, 300, 1000, 2100])
def test_cholesky_random(dev, n):
    lib = _lib.load()
    s = random_spd_real(n, n)
    da, lda = to_device_colmajor(s, dev)
    info = _lib.BseInfo()
    check(lib.bse_potrf_dev(n, ptr(da), lda, stream_ptr(), C.byref(info)), "potrf")
    low = from_device_colmajor(da, n, n)
    assert np.array_equal(low, np.tril(low))
    assert np.linalg.norm(low @ low.T - s) <= 1e-14 * n * np.linalg.norm(s)
    ref = np.linalg.cholesky(s)
    assert np.max(np.abs(low - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_cholesky_late_pivot_failure(dev):
    lib = _lib.load()
    n = 300
    s = random_spd_real(n, 3)
    s[200, 200] = -1e6  # first failure at index 200
    da, lda = to_device_colmajor(s, dev)
    info = _lib.BseInfo()
    st = lib.bse_potrf_dev(n, ptr(da), lda, stream_ptr(), C.byref(info))
    assert st == _lib.BSE_NOT_POSITIVE_DEFINITE
    assert info.pivot_index == 200
    assert info.pivot_value < 0


@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("n,m", [(1, 3), (64, 64), (100, 37), (700, 333)])
def test_trsm(dev, kind, n, m):
    lib = _lib.load()
    low = np.linalg.cholesky(random_spd_real(n, 11))
    rng = np.random.default_rng(2)
    b = rng.standard_normal((m, n) if kind == 0 else (n, m))
    dl, ldl = to_device_colmajor(low, dev)
    db, ldb = to_device_colmajor(b, dev)
    check(lib.bse_trsm_dev(kind, n, ptr(dl), ldl, ptr(db), ldb, m, stream_ptr()), "trsm")
    got = from_device_colmajor(db, *b.shape)
    if kind == 0:
        ref = np.linalg.solve(low, b.T).T  # B L^{-T}
    elif kind == 1:
        ref = np.linalg.solve(low.T, b)
    else:
        ref = np.linalg.solve(low, b)
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
