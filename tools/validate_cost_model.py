"""Validate oracle/cost_model.py against complete oracle runs, phase by phase.

    python tools/validate_cost_model.py --n 256 512 1024 [--rounds 3] [--out FILE]

For each n (cfg2 recipe, seed 2) it runs the oracle's solve_complex
(the reference algorithm, solvers.py:29-77) to completion with a timer
around each phase, then the sampled full-size estimate (several rounds with
different stratum offsets), and reports both per phase.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import bse_oracle as orc  # noqa: E402
from oracle import cost_model as cm  # noqa: E402


def timed_solve_complex(a, b):
    """orc.solve_complex with per-phase wall times (same calls, same order)."""
    ph = {}
    n = a.shape[0]
    t = time.perf_counter()
    m = orc.build_m(a, b)
    ph["build_m"] = time.perf_counter() - t
    t = time.perf_counter()
    low = orc.cholesky(m, what="the definiteness embedding M")
    ph["cholesky"] = time.perf_counter() - t
    t = time.perf_counter()
    w = low.T @ np.vstack([low[n:], -low[:n]])
    w = 0.5 * (w - w.T)
    ph["congruence"] = time.perf_counter() - t
    t = time.perf_counter()
    _, sub, store, taus = orc.tridiagonalize(w, skew=True)
    ph["tridiagonalize"] = time.perf_counter() - t
    t = time.perf_counter()
    lam, vp = orc.tridiag_eig(np.zeros(2 * n), -sub, which="positive")
    ph["tridiag_eig"] = time.perf_counter() - t
    t = time.perf_counter()
    zr = np.zeros_like(vp)
    zi = np.zeros_like(vp)
    zr[0::4], zr[2::4] = vp[0::4], -vp[2::4]
    zi[1::4], zi[3::4] = vp[1::4], -vp[3::4]
    gr = low @ orc.apply_reflectors(store, taus, zr)
    gi = low @ orc.apply_reflectors(store, taus, zi)
    r2 = np.sqrt(2.0)
    top = ((gr[:n] + gi[n:]) + 1j * (gi[:n] - gr[n:])) / r2
    bot = ((gr[:n] - gi[n:]) + 1j * (gi[:n] + gr[n:])) / r2
    scale = 1.0 / np.sqrt(lam)
    _ = (top * scale, -bot * scale)
    ph["back_transform"] = time.perf_counter() - t
    return ph, lam


def main():
    from paper_1501_03830_b200 import configs
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[256, 512])
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--points", type=int, default=4)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    rows = []
    for n in args.n:
        a, b, _ = configs.config_operator(2, n=n, seed=2)
        full, lam = timed_solve_complex(a, b)
        sampler = cm.SolveComplexCost(a, b, (0.1, 100.0))
        ests, spent = [], []
        for u in cm.offsets(args.rounds):
            spent.append(sampler.round(points=args.points, u=u))
            ests.append(sampler.estimate())
        est = sampler.phases()
        row = {"n": n, "m": 2 * n, "full_s": sum(full.values()), "full_phases": full,
               "estimate_s": ests[-1], "estimate_after_each_round_s": ests,
               "estimate_phases": est,
               "measure_s_per_round": float(np.mean(spent)),
               "lam_range_actual": [float(lam.min()), float(lam.max())],
               "bisection_iterations_model": sampler.bisection_iterations(),
               "threads": os.environ.get("OPENBLAS_NUM_THREADS") or os.cpu_count()}
        mean = est
        row["ratio"] = row["estimate_s"] / row["full_s"]
        rows.append(row)
        print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in row.items()
                          if k not in ("full_phases", "estimate_phases")}), flush=True)
        for k in full:
            print(f"   {k:15s} full {full[k]:9.3f}  est {mean[k]:9.3f}", flush=True)
    if args.out:
        Path(args.out).parent.mkdir(parents=True, exist_ok=True)
        Path(args.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
