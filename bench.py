"""Benchmark: full BSE eigenpair time-to-solution on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--n 16384]

Workload (N=1): BASELINE config 2 -- real BSE, n = 16384, s, d log-uniform
on [0.1, 100], Haar U1, U2 -- the largest single-GPU configuration of the
metric's n = 16k-64k range.  One step = one complete solve through the C ABI
(bse_solve_spd_pair_dev): Cholesky of K, W = L^T M L, two-stage eigensolver
(SY2SB, SB2ST, D&C, Q2/Q1), recovery of X1/X2 (all eigenpairs).  Inputs are
2 GB each (> 126 MB L2) and resident in HBM when the timed region starts.

Multi-GPU (torchrun, N > 1): ONE solve spans the N GPUs ("scaling":
"strong"): the column-sharded path of bse_solve_spd_pair_dist_dev over an
NCCL communicator (congruence and eigenvector-side stages split by columns,
reduction and D&C replicated, column blocks broadcast from their owners;
DESIGN.md section 7).  Times are device (CUDA event) times, max over ranks.

--impl reference times the reference algorithm on the host cores: the numpy
restatement of the reference's solve_complex (oracle/bse_oracle.py; the
reference itself is pure Python and not installed on the GPU box), on a
bounded sample (cfg2 recipe at n = 256 and 512) extrapolated to the workload n
with the fitted power law.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CFG = 2
SEED = 2


def alg_flops(n: int) -> float:
    """Canonical one-stage-equivalent count F(N) = (20/3) N^3."""
    return 20.0 / 3.0 * n ** 3


STAGE_FLOPS = {  # per-stage algorithmic flops, N = n
    "potrf": lambda n: n ** 3 / 3.0,
    "congruence": lambda n: float(n) ** 3,
    "sy2sb": lambda n: 4.0 * n ** 3 / 3.0,
    "q2_apply": lambda n: 2.0 * n ** 3,
    "q1_apply": lambda n: 2.0 * n ** 3,
    "recover": lambda n: 2.0 * n ** 3,
}


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank timing over all ranks (the contract's job time)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# CPU baseline: the reference algorithm (numpy restatement) on host cores

def cpu_reference_sample(n_target: int, sizes=(256, 512)):
    import numpy as np
    from oracle import bse_oracle as orc
    from paper_1501_03830_b200 import configs
    times = []
    for n in sizes:
        a, b, _ = configs.config_operator(CFG, n=n, seed=SEED)
        t0 = time.perf_counter()
        orc.solve_complex(a, b)
        times.append(time.perf_counter() - t0)
    expo = float(np.log(times[-1] / times[0]) / np.log(sizes[-1] / sizes[0]))
    expo = min(max(expo, 2.5), 3.3)
    value = times[-1] * (n_target / sizes[-1]) ** expo
    threads = os.environ.get("OPENBLAS_NUM_THREADS") or os.environ.get("OMP_NUM_THREADS")
    cores = int(threads) if threads else (os.cpu_count() or 1)
    sample = (f"reference algorithm (oracle/bse_oracle.solve_complex: skew Householder "
              f"tridiagonalization + bisection/inverse iteration, numpy) on the cfg2 recipe at "
              f"n={sizes} took {[round(t, 2) for t in times]} s; extrapolated to n={n_target} "
              f"with fitted exponent {expo:.2f} (effectively single-core Python loops; "
              f"BLAS threads {cores})")
    return value, cores, sample, times


def run_reference(args):
    rank, _, world = env_rank()
    if rank != 0:
        return 0
    vals = []
    info = None
    for i in range(args.warmup + args.steps):
        v, cores, sample, _ = cpu_reference_sample(args.n)
        if i >= args.warmup:
            vals.append(v)
        info = (cores, sample)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": "full BSE eigenpair time-to-solution (s)", "value": value,
        "unit": "s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE cfg2 recipe)",
        "config": {"workload": f"cfg2 real BSE n={args.n}, log-uniform [0.1,100] spectra",
                   "n": args.n, "parallelism": "host cpu"},
        "cpu_baseline": {"value": value, "unit": "s", "cores": info[0], "kind": "port",
                         "sample": info[1]},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in out.strip().splitlines():
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s in sm if s > 300] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def run_ours_cfg1(args):
    """BASELINE config 1: complex Hermitian BSE n = 2048 (real embedding
    N = 4096), all eigenpairs incl. the complex extraction and the
    biorthogonality polish -- the solve_complex device path."""
    import numpy as np
    import torch

    import paper_1501_03830_b200 as bg
    from paper_1501_03830_b200 import configs, solvers
    from paper_1501_03830_b200.device import to_device_colmajor

    rank, local_rank, world = env_rank()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n = 2048
    a, b, _, a_vals = configs.complex_operator(n, seed=1 + rank)
    op = bg.make_operator(a, b, kind="complex")
    m, k = solvers.real_embedding(op)
    Mt, ldm = to_device_colmajor(m, dev)
    Kt, ldk = to_device_colmajor(k, dev)

    def step():
        lam2, X1, X2, ld = solvers.solve_pair_device(Mt, ldm, Kt, ldk, 2 * n)
        return solvers._select_and_polish(lam2, X1, X2, ld, n, dev)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        lam, X1c, X2c = step()
    ev1.record()
    torch.cuda.synchronize(dev)
    ms = ev0.elapsed_time(ev1) / args.steps
    ok = bool(np.all(lam > 0) and bg.dos_dominance(lam, a_vals))
    if rank == 0:
        print(json.dumps({
            "metric": "full BSE eigenpair time-to-solution (s)", "value": ms / 1e3, "unit": "s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE cfg1 recipe, numpy PCG64 seed 1)",
            "config": {"workload": "cfg1 complex BSE n=2048 (real embedding N=4096), all "
                                   "eigenpairs + complex extraction + biorthogonality polish",
                       "n": n, "parallelism": "single GPU"},
            "tflops_canonical": alg_flops(2 * n) / (ms / 1e3) / 1e12,
            "reference_measured_s": 366.0,
            "reference_note": "reference solve_complex at this config took 366 s on the survey "
                              "host (SURVEY 6, BASELINE.md 2)",
            "sanity_lambda_positive_tda": ok}), flush=True)
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1501_03830_b200 import _lib, configs
    from paper_1501_03830_b200.device import ptr

    rank, local_rank, world = env_rank()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = _lib.load(strict=True)
    n = args.n
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    comm = None
    if world > 1:
        from paper_1501_03830_b200.distributed import Communicator
        comm = Communicator.nccl()

    # inputs: M = A + B = S, K = A - B = D (symmetric: row-major == column-major)
    S, D, dip = configs.torch_real_operator(n, seed=SEED, spectrum="loguniform", lo=0.1,
                                            hi=100.0, device=dev)
    ld = n + (n & 1)
    Mt = torch.zeros((n, ld), dtype=torch.float64, device=dev)
    Kt = torch.zeros((n, ld), dtype=torch.float64, device=dev)
    Mt[:, :n].copy_(S)
    Kt[:, :n].copy_(D)
    del S, D
    X1 = torch.empty((n, ld), dtype=torch.float64, device=dev)
    X2 = torch.empty((n, ld), dtype=torch.float64, device=dev)
    lam = torch.empty(n, dtype=torch.float64, device=dev)
    wb = lib.bse_solve_workspace_bytes(n, 0)
    work = torch.empty(wb, dtype=torch.uint8, device=dev)
    info = _lib.BseInfo()
    if world > 1:
        # one solve over all ranks: every rank must hold rank 0's (M, K)
        dist.broadcast(Mt, src=0)
        dist.broadcast(Kt, src=0)
        torch.cuda.synchronize(dev)

    def step():
        if comm is None:
            st = lib.bse_solve_spd_pair_dev(n, ptr(Mt), ld, ptr(Kt), ld, ptr(lam), ptr(X1), ld,
                                            ptr(X2), ld, ptr(work), wb, 0, sp, C.byref(info))
        else:
            st = lib.bse_solve_spd_pair_dist_dev(comm.handle, n, ptr(Mt), ld, ptr(Kt), ld,
                                                 ptr(lam), ptr(X1), ld, ptr(X2), ld, ptr(work),
                                                 wb, 0, sp, C.byref(info))
        if st != 0:
            raise RuntimeError(f"solve failed ({st}): {_lib.last_error()}")

    # FP64 roofline denominator: measured DMMA peak on this GPU (no FP64 entry in
    # MEASURED_PEAKS.json)
    fl, ms = C.c_double(), C.c_double()
    lib.bse_peak_fp64(0, 296, 20000, 5, C.byref(fl), C.byref(ms))
    fp64_peak = fl.value / (ms.value * 1e-3) / 1e12

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # ---- timed region ----
    clocks = ClockSampler(local_rank)
    time.sleep(0.3)
    lib.bse_profile_enable(1)
    launches0 = lib.bse_launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = lib.bse_launch_count() - launches0
    clk = clocks.stop()
    total_ms = ev0.elapsed_time(ev1)
    msarr = (C.c_double * 4096)()
    names = C.create_string_buffer(32 * 4096)
    cnt = lib.bse_profile_read(4096, msarr, names)
    lib.bse_profile_enable(0)
    stages = {}
    for i in range(cnt):
        nm = names.raw[32 * i:32 * (i + 1)].split(b"\0")[0].decode()
        if nm == "end":
            continue
        stages[nm] = stages.get(nm, 0.0) + msarr[i] / args.steps
    ms_step = max_over_ranks(total_ms / args.steps, dist if world > 1 else None, dev)

    # sanity: eigenvalues positive, descending
    lam_h = lam.cpu().numpy()
    ok = bool(np.all(lam_h > 0) and np.all(np.diff(lam_h) <= 0))
    # size-independent verification of the last timed solve (outside the timed
    # region): per-pair residual / (lam_max ||x||) and ||X1^T X1 - X2^T X2 - I||_F
    verification = None
    if comm is None:
        # the single-GPU workspace is not needed after the timed region (the
        # host entry allocates its own): release it for the checks (n = 32768
        # needs 125 GB of workspace on a 178 GB device)
        del work
        torch.cuda.empty_cache()
    if not args.no_verify and rank == 0:
        from paper_1501_03830_b200.verify import pair_residuals_device
        res, xn, bio = pair_residuals_device(n, Mt, ld, Kt, ld, lam, X1, ld, X2, ld)
        verification = {"max_pair_residual": (res / (lam[0] * xn)).max().item(),
                        "biorthogonality_fro": bio.item(),
                        "gate": "<= 1e-13 n and <= 1e-12 n (SURVEY 8c(8))"}
        verification["pass"] = bool(verification["max_pair_residual"] <= 1e-13 * n and
                                    verification["biorthogonality_fro"] <= 1e-12 * n)
        del res, xn
        torch.cuda.empty_cache()

    # ---- e2e: public C-ABI host entry, pinned host buffers, copies inside ----
    e2e = None
    if args.e2e_steps > 0:
        Mh = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        Kh = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        Mh.copy_(Mt[:, :n])
        Kh.copy_(Kt[:, :n])
        if comm is None:
            # the host entry allocates its own device buffers
            del Mt, Kt, X1, X2
            torch.cuda.empty_cache()
        out_n = n if rank == 0 else 1  # only rank 0 reads the solution back
        lamh = torch.empty(out_n, dtype=torch.float64, pin_memory=True)
        X1h = torch.empty((out_n, out_n), dtype=torch.float64, pin_memory=True)
        X2h = torch.empty((out_n, out_n), dtype=torch.float64, pin_memory=True)
        torch.cuda.synchronize(dev)

        def e2e_step():
            if comm is None:
                st = lib.bse_solve_spd_pair_host(n, ptr(Mh), n, ptr(Kh), n, ptr(lamh), ptr(X1h),
                                                 n, ptr(X2h), n, 0, C.byref(info))
                if st != 0:
                    raise RuntimeError(f"host solve failed: {_lib.last_error()}")
                return
            # sharded: every rank uploads its host copy of (M, K), the solve
            # runs across the ranks, rank 0 reads the assembled solution back
            Mt[:, :n].copy_(Mh, non_blocking=True)
            Kt[:, :n].copy_(Kh, non_blocking=True)
            step()
            if rank == 0:
                lamh.copy_(lam, non_blocking=True)
                X1h.copy_(X1[:, :n], non_blocking=True)
                X2h.copy_(X2[:, :n], non_blocking=True)
            torch.cuda.synchronize(dev)
        e2e_step()  # warm the allocator pool
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        e2e_s = max_over_ranks((time.perf_counter() - t0) / args.e2e_steps,
                               dist if world > 1 else None, dev)
        e2e = {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": world * 2 * n * n * 8,
               "d2h_bytes_per_step": (2 * n * n + n) * 8,
               "path": ("bse_solve_spd_pair_host (pinned host M, K -> lam, X1, X2)" if comm is None
                        else "pinned host M, K -> every rank; bse_solve_spd_pair_dist_dev; "
                             "rank 0 lam, X1, X2 -> pinned host")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, sample, _ = cpu_reference_sample(n)
        cpu = {"value": v, "unit": "s", "cores": cores, "kind": "port", "sample": sample}

    if comm is not None:
        comm.close()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # roofline of the dominant FP64-tensor stage (algorithmic flops / live event time)
    tens = {k: v for k, v in stages.items() if k in STAGE_FLOPS}
    dom = max(tens, key=tens.get) if tens else None
    roof = None
    if dom:
        ach = STAGE_FLOPS[dom](n) / (tens[dom] * 1e-3) / 1e12
        traffic = None
        try:
            tr = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text()).get(dom)
            if tr and int(tr["n"]) == n:
                traffic = {"bytes": tr["dram_bytes"], "unit": "B", "source": tr["source"]}
        except (OSError, ValueError, KeyError):
            traffic = None
        roof = {"bound": "tensor", "kernel": dom, "achieved": ach, "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": ach / fp64_peak, "traffic": traffic,
                "peak_source": "measured in-run FP64 DMMA probe (mma.sync m8n8k4 f64); "
                               "MEASURED_PEAKS.json has no FP64 entry",
                "flops_per_launch": STAGE_FLOPS[dom](n)}
    solve_s = ms_step / 1e3
    line = {
        "metric": "full BSE eigenpair time-to-solution (s)", "value": solve_s, "unit": "s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": False, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE cfg2 recipe, torch Philox on GPU)",
        "config": {"workload": f"cfg2 real BSE n={n} (H {2 * n}x{2 * n}), log-uniform [0.1,100] "
                               f"spectra, all eigenpairs + X1/X2",
                   "n": n,
                   "parallelism": (f"column-sharded x{world} (NCCL; reduction + D&C replicated)"
                                   if world > 1 else "single GPU"),
                   "l2": f"inputs {n * n * 8 / 2**30:.0f} GiB each > 126 MB L2 (no flush needed)"},
        "tflops": alg_flops(n) / solve_s / 1e12,
        "fp64_peak_tflops": fp64_peak,
        "frac_of_fp64_peak": alg_flops(n) / solve_s / 1e12 / fp64_peak,
        "stages_ms": {k: round(v, 3) for k, v in stages.items()},
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk,
        "sanity_lambda_positive_desc": ok,
        "verification": verification,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--config", type=int, default=2, choices=[1, 2],
                    help="2 (default): real n=16384 headline; 1: complex n=2048 side line")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.impl == "reference":
        return run_reference(args)
    if args.config == 1:
        return run_ours_cfg1(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
