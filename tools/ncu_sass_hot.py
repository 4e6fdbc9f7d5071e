"""Top SASS instructions by stall samples and shared-memory excess wavefronts
from an ncu report (--page source --print-source=sass).

    python tools/ncu_sass_hot.py gpurun_out/prof.ncu-rep [--top 25]
"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=25)
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
# multiple kernels may be present; parse each "Kernel Name" block
blocks, cur = [], []
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        if cur:
            blocks.append(cur)
        cur = [ln]
    else:
        cur.append(ln)
if cur:
    blocks.append(cur)
for blk in blocks[:1]:
    print(blk[0][:150])
    rows = list(csv.DictReader(io.StringIO("\n".join(blk[1:]))))
    def num(r, k):
        try:
            return float(r.get(k, "0").replace(",", ""))
        except ValueError:
            return 0.0
    tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in rows)
    exc = sum(num(r, "L1 Wavefronts Shared Excessive") for r in rows)
    print(f"samples {tot:.0f}  shared excessive wavefronts {exc:.3g}")
    stall_keys = [k for k in rows[0] if k.startswith("stall_") and "Not Issued" not in k]
    agg = {k: sum(num(r, k) for r in rows) for k in stall_keys}
    print("stalls:", ", ".join(f"{k[6:]} {100*v/max(tot,1):.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    print("-- hottest instructions")
    for r in sorted(rows, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:a.top]:
        print(f"{num(r,'Warp Stall Sampling (All Samples)'):8.0f} exc={num(r,'L1 Wavefronts Shared Excessive'):10.0f}  {r['Source'].strip()[:90]}")
    print("-- most excessive shared wavefronts")
    for r in sorted(rows, key=lambda r: -num(r, "L1 Wavefronts Shared Excessive"))[:8]:
        print(f"exc={num(r,'L1 Wavefronts Shared Excessive'):10.0f} ideal={num(r,'L1 Wavefronts Shared Ideal'):10.0f}  {r['Source'].strip()[:90]}")
