"""Text summary of one kernel in an ncu --set full report: key metrics, stall
reasons, hottest SASS instructions and CUDA source lines (for profiles/).

    python tools/ncu_summary.py gpurun_out/q2_v5.ncu-rep > profiles/r01/q2_apply_full.txt
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, val = raw[0], raw[2]
get = dict(zip(hdr, val))
keys = [
    "Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smsp__warps_active.avg.per_cycle_active", "smsp__inst_executed.sum",
]
units = dict(zip(hdr, raw[1]))
print("== metrics (ncu --set full --clock-control none)")
for k in keys:
    if k in get:
        print(f"{k:80s} {get[k]} {units.get(k, '')}")
stalls = {k.split("smsp__pcsamp_warps_issue_stalled_")[1]: float(v.replace(",", "") or 0)
          for k, v in get.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
tot = sum(stalls.values()) or 1.0
print("== stall reasons (pc sampling)")
for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]:
    print(f"  {k:32s} {100 * v / tot:5.1f}%")
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source=cuda,sass"))))
lines, sass, fname = {}, [], None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 5 or r[0] == "Line No":
        continue
    try:
        n = int(r[4])
    except ValueError:
        continue
    if r[0]:
        lines[(fname, r[0], r[1].strip()[:100])] = n
    else:
        sass.append((n, r[3].strip()[:90]))
tl = sum(lines.values()) or 1
print(f"== hottest source lines ({tl} samples)")
for (f, ln, src), n in sorted(lines.items(), key=lambda x: -x[1])[:top]:
    print(f"  {100 * n / tl:5.1f}%  {f}:{ln}  {src}")
print("== hottest SASS")
for n, ins in sorted(sass, key=lambda x: -x[0])[:top]:
    print(f"  {100 * n / tl:5.1f}%  {ins}")
