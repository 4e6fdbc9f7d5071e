"""GPU probe: FP64 DMMA/DFMA peaks and GEMM / POTRF throughput (CUDA events)."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1501_03830_b200 import _lib  # noqa: E402
from paper_1501_03830_b200.device import check, ptr, stream_ptr  # noqa: E402

lib = _lib.load()
out = {}
for which, name in ((0, "dmma"), (1, "dfma")):
    f, ms = C.c_double(), C.c_double()
    for blocks in (148, 296, 592):
        check(lib.bse_peak_fp64(which, blocks, 20000, 5, C.byref(f), C.byref(ms)), "peak")
        out[f"{name}_tflops_b{blocks}"] = f.value / (ms.value * 1e-3) / 1e12

dev = torch.device("cuda:0")


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for n in (2048, 4096, 8192):
    A = torch.randn(n, n, dtype=torch.float64, device=dev)
    B = torch.randn(n, n, dtype=torch.float64, device=dev)
    Cm = torch.zeros(n, n, dtype=torch.float64, device=dev)
    for ta, tb in ((0, 0), (1, 0), (0, 1)):
        ms = timeit(lambda: check(lib.bse_gemm_dev(ta, tb, n, n, n, 1.0, ptr(A), n, ptr(B), n, 0.0,
                                                   ptr(Cm), n, None, stream_ptr()), "gemm"))
        out[f"gemm_{ta}{tb}_n{n}_tflops"] = 2 * n**3 / (ms * 1e-3) / 1e12
    ref = (B.T @ A.T)  # column-major C = A B  <=> row-major C^T = B^T A^T
    check(lib.bse_gemm_dev(0, 0, n, n, n, 1.0, ptr(A), n, ptr(B), n, 0.0, ptr(Cm), n, None,
                           stream_ptr()), "gemm")
    torch.cuda.synchronize()
    out[f"gemm_err_n{n}"] = float((Cm - ref).abs().max() / ref.abs().max())
    ms = timeit(lambda: torch.matmul(A, B))
    out[f"torch_dgemm_n{n}_tflops"] = 2 * n**3 / (ms * 1e-3) / 1e12
    S = A @ A.T + n * torch.eye(n, dtype=torch.float64, device=dev)
    W = torch.empty_like(S)
    info = _lib.BseInfo()

    def chol():
        W.copy_(S)
        check(lib.bse_potrf_dev(n, ptr(W), n, stream_ptr(), C.byref(info)), "potrf")
    ms = timeit(chol, reps=3)
    out[f"potrf_n{n}_tflops"] = n**3 / 3 / (ms * 1e-3) / 1e12
    out[f"potrf_n{n}_ms"] = ms
print(json.dumps(out, indent=1))
