"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name.

    python tools/launch_summary.py gpurun_out/launches.csv [--last-fraction 0.5]
"""
import argparse
import collections
import csv
import re

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--last-fraction", type=float, default=1.0)
ap.add_argument("--top", type=int, default=30)
a = ap.parse_args()
lines = [ln for ln in open(a.csv) if not ln.startswith("==")]
rows = list(csv.DictReader(lines))
rows = [r for r in rows if "bse" in r["Kernel Name"] or "cutlass::device_kernel" in r["Kernel Name"]]
rows = rows[int(len(rows) * (1 - a.last_fraction)):]
tot = collections.defaultdict(float)
cnt = collections.Counter()
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
for r in rows:
    name = r["Kernel Name"]
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"bse::\(anonymous namespace\)::", "", name)
    name = re.sub(r"\(.*$", "", name)
    if name.startswith("cutlass::device_kernel"):
        name = "cutlass::device_kernel<int8 tcgen05 GEMM (emulated FP64)>"
    v = float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
    tot[name] += v
    cnt[name] += 1
s = sum(tot.values())
print(f"{'kernel':70s} {'launches':>8s} {'ms':>10s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:a.top]:
    print(f"{k[:70]:70s} {cnt[k]:8d} {v:10.2f} {100 * v / s:5.1f}%")
print(f"{'TOTAL':70s} {sum(cnt.values()):8d} {s:10.2f}")
