"""SB2ST stage time and a correctness check of the band -> tridiagonal stage.

Runs the values-only eigensolver (SY2SB + SB2ST + Sturm bisection) on a seeded
random symmetric matrix `reps` times with the stage profile on, prints the
`sb2st` stage time of every run, a hash of the eigenvalues (must not change
from run to run) and -- with --check -- the largest deviation from the trace
and Frobenius invariants (sum lam = tr A, sum lam^2 = |A|_F^2), which any lost
or stale hand-off value breaks.

    python tools/sb2st_time.py --n 16384 --reps 3 --check
"""
import argparse
import ctypes as C
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_1501_03830_b200 import _lib, solvers
    from paper_1501_03830_b200.device import colmajor_empty
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    n = args.n
    lib = _lib.load()
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    a = torch.randn(n, n, dtype=torch.float64, device=dev, generator=g)
    a = 0.5 * (a + a.T)
    tr, fro2 = float(torch.trace(a)), float((a * a).sum())
    At, lda = colmajor_empty(n, n, dev)
    hashes = []
    for rep in range(args.reps):
        At[:n, :n].copy_(a)
        torch.cuda.synchronize()
        lib.bse_profile_enable(1)
        w = solvers.syevd_values_device(At, lda, n)
        torch.cuda.synchronize()
        cnt = lib.bse_profile_count()
        ms = (C.c_double * max(cnt, 1))()
        names = C.create_string_buffer(32 * max(cnt, 1))
        got = lib.bse_profile_read(cnt, ms, names)
        lib.bse_profile_enable(0)
        st = {}
        for i in range(got):
            nm = names.raw[32 * i:32 * (i + 1)].split(b"\0")[0].decode()
            st[nm] = st.get(nm, 0.0) + ms[i]
        hashes.append(hashlib.sha1(w.cpu().numpy().tobytes()).hexdigest()[:12])
        line = (f"rep {rep}: sb2st {st.get('sb2st', float('nan')):.2f} ms  sy2sb panel "
                f"{st.get('sy2sb_panel', float('nan')):.2f} symm {st.get('sy2sb_symm', float('nan')):.2f} "
                f"small {st.get('sy2sb_small', float('nan')):.2f} syr2k {st.get('sy2sb_syr2k', float('nan')):.2f} ms"
                f"  hash {hashes[-1]}")
        if args.check:
            e1 = abs(float(w.sum()) - tr) / (abs(tr) + fro2 ** 0.5)
            e2 = abs(float((w * w).sum()) - fro2) / fro2
            line += f"  trace err {e1:.2e}  frob err {e2:.2e}"
        print(line, flush=True)
    print("deterministic", len(set(hashes)) == 1)


if __name__ == "__main__":
    main()
