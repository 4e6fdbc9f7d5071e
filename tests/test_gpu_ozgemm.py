"""Emulated FP64 GEMM on the INT8 tensor cores (csrc/ozgemm.cu: Ozaki scheme
II, tcgen05 kind::i8) against float64 references: every transpose, operand
and output masks (view-relative, like the DMMA engine), alpha/beta, column
chunking, ragged sizes, zero rows and rows spanning many binades."""
import numpy as np
import pytest

from paper_1501_03830_b200 import _lib
from paper_1501_03830_b200.device import (check, from_device_colmajor, mask_array, ptr,
                                          stream_ptr, to_device_colmajor)

from test_gpu_dense import _band

pytestmark = pytest.mark.gpu


def _oz(dev, ta, tb, a, b, c, alpha, beta, masks=None, chunk=0):
    lib = _lib.load()
    M, N = c.shape
    K = a.shape[0] if ta else a.shape[1]
    da, lda = to_device_colmajor(a, dev)
    db, ldb = to_device_colmajor(b, dev)
    dc, ldc = to_device_colmajor(c, dev)
    check(lib.bse_ozgemm_dev(ta, tb, M, N, K, alpha, ptr(da), lda, ptr(db), ldb, beta, ptr(dc),
                             ldc, masks, chunk, stream_ptr()), "ozgemm")
    return from_device_colmajor(dc, M, N)


def _bound(a_op, b_op):
    # per-entry truncation bound: 2^-52 (row max of A) sum|B| + sum|A| (col max of B)
    ra = np.max(np.abs(a_op), axis=1, keepdims=True)
    cb = np.max(np.abs(b_op), axis=0, keepdims=True)
    return 2.0 ** -51 * (ra * np.sum(np.abs(b_op), axis=0, keepdims=True)
                         + np.sum(np.abs(a_op), axis=1, keepdims=True) * cb)


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 5, 3), (130, 257, 77), (300, 129, 1000),
                                   (513, 511, 256), (1024, 1024, 4096)])
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_ozgemm_plain(dev, M, N, K, ta, tb):
    rng = np.random.default_rng(M * 7 + N * 3 + K + ta * 11 + tb * 13)
    a = rng.standard_normal((K, M) if ta else (M, K))
    b = rng.standard_normal((N, K) if tb else (K, N))
    c = rng.standard_normal((M, N))
    got = _oz(dev, ta, tb, a, b, c, 1.5, -0.5)
    ao, bo = (a.T if ta else a), (b.T if tb else b)
    ref = 1.5 * (ao @ bo) - 0.5 * c
    tol = 1.5 * _bound(ao, bo) + 1e-15 * (np.abs(ref) + 1) * np.sqrt(K)
    assert np.all(np.abs(got - ref) <= tol)
    # at least as accurate as the DMMA engine's test gate
    assert np.max(np.abs(got - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref))) * np.sqrt(K)


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("case", ["lowerA", "unitA", "strictB", "upperA_lowerC", "lowerB_upperC"])
def test_ozgemm_masks(dev, ta, tb, case):
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
    for chunk in (0, 64):  # chunked output columns shift the B / C masks
        got = _oz(dev, ta, tb, a, b, c, 0.75, 2.0, mask_array(ma, mb, mc), chunk)
        assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref))), chunk


def test_ozgemm_wide_dynamic_range_and_zero_rows(dev):
    rng = np.random.default_rng(11)
    M, N, K = 257, 300, 700
    a = rng.standard_normal((M, K)) * np.exp2(rng.integers(-300, 300, size=(M, 1)))
    a[::17] = 0.0
    a[5, :] *= np.exp2(rng.integers(-40, 0, size=K))  # one row spans 40 binades
    b = rng.standard_normal((K, N)) * np.exp2(rng.integers(-60, 60, size=(1, N)))
    got = _oz(dev, 0, 0, a, b, np.zeros((M, N)), 1.0, 0.0)
    ref = a @ b
    assert np.all(np.abs(got - ref) <= 1.5 * _bound(a, b) + 1e-300)
    assert np.all(got[::17] == 0.0)


def test_ozgemm_orthogonal_product_keeps_orthogonality(dev):
    # the solve uses it on orthogonal factors: Q^T Q must stay I to O(eps)
    rng = np.random.default_rng(3)
    n = 1536
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    got = _oz(dev, 1, 0, q, q, np.zeros((n, n)), 1.0, 0.0, chunk=512)
    assert np.max(np.abs(got - np.eye(n))) <= 5e-15 * np.sqrt(n)


@pytest.mark.parametrize("engine", [0, 1])
@pytest.mark.parametrize("M,N,K,chunk", [(1, 1, 1, 0), (33, 70, 17, 0), (300, 129, 1000, 0),
                                         (513, 700, 256, 256), (1024, 1500, 4100, 512),
                                         (2304, 2050, 640, 0)])
def test_tcgen05_kernel_bitwise_vs_library_kernel(dev, engine, M, N, K, chunk):
    """The 16 integer products are exact on either kernel, so the hand-written
    tcgen05 contraction (byte residues from its epilogue, csrc/i8mma.cu; CTA
    pairs = 0, single CTAs = 1) must reproduce the CUTLASS kernel + INT32
    planes (engine 2) bit for bit, including ragged tiles, K tails and column
    chunks."""
    lib = _lib.load()
    rng = np.random.default_rng(M + 3 * N + 7 * K)
    a = rng.standard_normal((M, K)) * np.exp(rng.uniform(-8, 8, (M, 1)))
    b = rng.standard_normal((K, N))
    c = rng.standard_normal((M, N))
    prev = lib.bse_oz_set_engine(2)
    try:
        ref = _oz(dev, 0, 0, a, b, c, 1.0, 0.25, chunk=chunk)
        lib.bse_oz_set_engine(engine)
        got = _oz(dev, 0, 0, a, b, c, 1.0, 0.25, chunk=chunk)
    finally:
        lib.bse_oz_set_engine(prev)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("engine", [0, 1])
def test_tcgen05_kernel_output_band(dev, engine):
    """Tiles entirely outside the output band are skipped by the kernel (the
    symmetric rank-k updates of the reduction only need the lower triangle)."""
    lib = _lib.load()
    M = N = 900
    K = 300
    rng = np.random.default_rng(11)
    a = rng.standard_normal((M, K))
    b = rng.standard_normal((K, N))
    c = rng.standard_normal((M, N))
    masks = mask_array(None, None, (None, 0, 0))
    prev = lib.bse_oz_set_engine(engine)
    try:
        got = _oz(dev, 0, 0, a, b, c, -1.0, 1.0, masks=masks)
    finally:
        lib.bse_oz_set_engine(prev)
    ref = np.where(np.tril(np.ones((M, N), bool)), c - a @ b, c)
    assert np.max(np.abs(got - ref)) <= 1e-12
    assert np.array_equal(np.triu(got, 1), np.triu(c, 1))


@pytest.mark.parametrize("engine", [0, 1])
def test_tcgen05_fp32_residue_path_extremes(dev, engine):
    """K <= 256 takes the epilogue's FP32 reduction: accumulators at the ends of
    its range (|c| = K * 2^14 when every residue is -128, i.e. constant rows
    whose scaled value is 128 mod m) must still reduce exactly -- compared bit
    for bit with the INT32-plane path."""
    lib = _lib.load()
    for K in (256, 255, 130, 64):
        M, N = 300, 260
        rng = np.random.default_rng(K)
        # rows of constants (every entry of a line equal to its maximum) and a
        # few random ones: constant lines hit the same residue in every slot
        a = np.repeat(rng.integers(1, 2 ** 20, (M, 1)).astype(float), K, axis=1)
        b = np.repeat(rng.integers(1, 2 ** 20, (1, N)).astype(float), K, axis=0)
        a[::7] = rng.standard_normal((a[::7].shape))
        b[:, ::5] = rng.standard_normal((b[:, ::5].shape))
        c = np.zeros((M, N))
        prev = lib.bse_oz_set_engine(2)
        try:
            ref = _oz(dev, 0, 0, a, b, c, 1.0, 0.0)
            lib.bse_oz_set_engine(engine)
            got = _oz(dev, 0, 0, a, b, c, 1.0, 0.0)
        finally:
            lib.bse_oz_set_engine(prev)
        assert np.array_equal(got, ref), K
        assert np.max(np.abs(got - a @ b)) <= 1e-12 * np.max(np.abs(a @ b))
