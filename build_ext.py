"""Build the sm_100a shared library in-tree.

    python build_ext.py            # -> paper_1501_03830_b200/libbse_b200.so

Every .cu under paper_1501_03830_b200/csrc is compiled with
`-gencode arch=compute_100a,code=sm_100a -lineinfo` (objects in parallel,
cached by mtime under build/), then linked into one shared library exposing
the C ABI declared in include/bse_b200.h.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent
SRC = ROOT / "paper_1501_03830_b200" / "csrc"
OUT = ROOT / "paper_1501_03830_b200" / "libbse_b200.so"
OBJ = ROOT / "build" / "obj"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "--expt-relaxed-constexpr",
         "-I", str(ROOT / "include")]
# CuTe/CUTLASS headers (vendored in the image under flashinfer) for the
# tcgen05 int8 GEMM behind the emulated-FP64 engine (csrc/ozgemm.cu)
_CUTLASS = Path(sys.prefix) / "lib" / f"python{sys.version_info.major}.{sys.version_info.minor}" / \
    "site-packages" / "flashinfer" / "data" / "cutlass"
CUTLASS_FLAGS = ["-I", str(_CUTLASS / "include"), "-I", str(_CUTLASS / "tools" / "util" / "include"),
                 "-diag-suppress", "20012"]


def _compile(cu: Path) -> Path:
    obj = OBJ / (cu.stem + ".o")
    headers = list(SRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))
    newest = max([cu.stat().st_mtime] + [h.stat().st_mtime for h in headers])
    if obj.exists() and obj.stat().st_mtime >= newest:
        return obj
    extra = CUTLASS_FLAGS if cu.stem == "ozgemm" else []
    cmd = [NVCC, *FLAGS, *extra, "-c", str(cu), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed on {cu.name}")
    return obj


def build(verbose: bool = True) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    sources = sorted(SRC.glob("*.cu"))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(_compile, sources))
    if OUT.exists() and OUT.stat().st_mtime >= max(o.stat().st_mtime for o in objs):
        return OUT
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(OUT),
           *map(str, objs), "-lcudart", "-lcuda"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("link failed")
    if verbose:
        print(f"built {OUT.relative_to(ROOT)} from {len(objs)} objects")
    return OUT


if __name__ == "__main__":
    build()
