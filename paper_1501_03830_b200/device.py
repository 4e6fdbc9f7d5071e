"""Device plumbing: torch owns HBM allocations and streams; the C ABI does the
math.  Matrices live column-major: an (rows x cols) matrix with leading
dimension ld is a torch tensor of shape (cols, ld) whose row c is column c.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def _torch():
    import torch
    return torch


def require_cuda():
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1501_03830_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    return torch


def stream_ptr(device=None) -> int:
    torch = _torch()
    return torch.cuda.current_stream(device).cuda_stream


def colmajor_empty(rows: int, cols: int, device, ld: int | None = None, zero=False):
    """Column-major (rows x cols) FP64 buffer; returns (tensor, ld)."""
    torch = _torch()
    ld = max(1, rows if ld is None else ld)
    ld += ld & 1  # even leading dimension keeps 16-byte cp.async legal
    f = torch.zeros if zero else torch.empty
    return f((max(cols, 1), ld), dtype=torch.float64, device=device), ld


def to_device_colmajor(a: np.ndarray, device, ld: int | None = None):
    """Upload a 2-D float64 numpy array as a column-major device matrix."""
    torch = _torch()
    a = np.asarray(a, dtype=np.float64)
    rows, cols = a.shape
    t, ld = colmajor_empty(rows, cols, device, ld, zero=True)
    if rows and cols:
        # upload as stored, transpose on the device (a host transpose of a
        # multi-GB array costs seconds)
        src = np.ascontiguousarray(a)
        if not src.flags.writeable:
            src = src.copy()
        t[:cols, :rows].copy_(torch.from_numpy(src).to(t.device).T)
    return t, ld


def from_device_colmajor(t, rows: int, cols: int) -> np.ndarray:
    return t[:cols, :rows].T.cpu().numpy()


def view_colmajor(t, rows: int, cols: int):
    """Torch (rows x cols) view of a column-major buffer (no copy)."""
    return t[:cols, :rows].T


def ptr(t) -> int:
    return t.data_ptr()


def check(status: int, what: str):
    if status != _lib.BSE_OK:
        raise RuntimeError(f"{what} failed with status {status}: {_lib.last_error()}")


def mask_array(ma=None, mb=None, mc=None):
    big = 1 << 30
    out = []
    for m in (ma, mb, mc):
        if m is None:
            out += [-big, big, 0]
        else:
            lo, hi, unit = m
            out += [-big if lo is None else lo, big if hi is None else hi, unit]
    return (C.c_int32 * 9)(*out)


def upload_rowmajor(a: np.ndarray, device):
    """Device copy (same shape / dtype, C order) of a host array through the
    library's pinned staging ring (bse_memcpy2d_staged): the path for the
    multi-GB numpy blocks of the drop-in API."""
    torch = _torch()
    a = np.ascontiguousarray(a)
    t = torch.empty(a.shape, dtype=getattr(torch, a.dtype.name), device=device)
    if a.size:
        row = a.itemsize * (a.shape[-1] if a.ndim else 1)
        rows = a.size * a.itemsize // row
        st = _lib.load().bse_memcpy2d_staged(1, t.data_ptr(), row, a.ctypes.data, row, row, rows,
                                            torch.cuda.current_stream(device).cuda_stream)
        check(st, "bse_memcpy2d_staged")
    return t


def download_complex(t, rows: int, cols: int) -> np.ndarray:
    """numpy complex128 (rows x cols, C order) of the column-major real device
    matrix in ``t`` (imaginary part 0): transposed and widened on the device,
    then copied through the staging ring (bse_memcpy2d_staged)."""
    torch = _torch()
    out = np.empty((rows, cols), dtype=np.complex128)
    if rows and cols:
        dev = torch.zeros((rows, cols), dtype=torch.complex128, device=t.device)
        torch.view_as_real(dev)[..., 0].copy_(view_colmajor(t, rows, cols))
        st = _lib.load().bse_memcpy2d_staged(0, out.ctypes.data, 16 * cols, dev.data_ptr(),
                                            16 * cols, 16 * cols, rows,
                                            torch.cuda.current_stream(t.device).cuda_stream)
        check(st, "bse_memcpy2d_staged")
    return out
