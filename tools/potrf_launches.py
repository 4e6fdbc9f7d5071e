"""Per-kernel summary of an ncu launch list (gpu__time_duration.sum,
launch__grid_size) taken over tools/bench_potrf.py --reps 1 (second half =
the timed call):  python tools/potrf_launches.py gpurun_out/potrf_launches.csv"""
import collections
import csv
import re
import sys

lines = [ln for ln in open(sys.argv[1]) if not ln.startswith("==")]
rows = list(csv.DictReader(lines))
k = {}
for r in rows:
    d = k.setdefault(r["ID"], {"name": r["Kernel Name"]})
    d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
ks = [k[i] for i in sorted(k, key=int)]
ks = ks[len(ks) // 2:]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for x in ks:
    m = re.search(r"(potf2_kernel|gemm_single_kernel<[^>]*>|gemm_grouped_kernel<[^>]*>|trtri_leaf|"
                  r"[a-z_0-9]+_kernel)", x["name"])
    nm = m.group(1) if m else x["name"][:60]
    g = int(x.get("launch__grid_size", 0))
    b = "g<=16" if g <= 16 else "g<=148" if g <= 148 else "g<=1024" if g <= 1024 else "big"
    t = x["gpu__time_duration.sum"] * 1e-6
    tot[(nm, b)] += t
    cnt[(nm, b)] += 1
print(f"total {sum(tot.values()):.2f} ms over {len(ks)} launches")
for n, v in sorted(tot.items(), key=lambda x: -x[1])[:15]:
    print(f"{v:8.2f} ms {cnt[n]:5d} {n}")
