"""SB2ST per-step timing trace (BSE_SB2ST_TRACE=<sweep>): runs the values-only
eigensolver (SY2SB + SB2ST + bisection) on a random symmetric matrix and lets
sb2st.cu print the per-phase step breakdown of sweep <sweep>+1 against its
producer sweep (latewait / lateload / ABC / publish / bulk / period / handoff).

    BSE_SB2ST_TRACE=2000 python tools/sb2st_trace.py --n 16384
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_1501_03830_b200 import solvers
    from paper_1501_03830_b200.device import colmajor_empty
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    args = ap.parse_args()
    n = args.n
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    a = torch.randn(n, n, dtype=torch.float64, device=dev, generator=g)
    a = 0.5 * (a + a.T)
    At, lda = colmajor_empty(n, n, dev)
    At[:n, :n].copy_(a)
    del a
    w = solvers.syevd_values_device(At, lda, n)
    torch.cuda.synchronize()
    print("lambda range", float(w[0]), float(w[-1]))


if __name__ == "__main__":
    main()
