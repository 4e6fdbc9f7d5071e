set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out /tmp/dump
rm -f /tmp/dump/*
BSE_DEBUG_DUMP=/tmp/dump BSE_DEBUG_HASH=1 timeout 600 python tools/determinism_probe.py --n 4608 --procs 1 --reps 3 --values > gpurun_out/det_dump_ref.log 2>&1
mkdir -p /tmp/dump2
BSE_SB2ST_MODE=264 BSE_DEBUG_DUMP=/tmp/dump2 BSE_DEBUG_HASH=1 timeout 600 python tools/determinism_probe.py --n 4608 --procs 1 --reps 12 --values > gpurun_out/det_dump_264.log 2>&1
python - <<'PY' > gpurun_out/det_dump_analysis.log 2>&1
import glob, re, numpy as np
def key(f): return int(re.search(r"_(\d+)\.bin$", f).group(1))
ref = np.fromfile(sorted(glob.glob('/tmp/dump/d_*.bin'), key=key)[0])
refe = np.fromfile(sorted(glob.glob('/tmp/dump/e_*.bin'), key=key)[0])
ds = sorted(glob.glob('/tmp/dump2/d_*.bin'), key=key); es = sorted(glob.glob('/tmp/dump2/e_*.bin'), key=key)
for f, g in zip(ds, es):
    a = np.fromfile(f); e = np.fromfile(g)
    idx = np.nonzero(a != ref)[0]; idxe = np.nonzero(e != refe)[0]
    if len(idx) == 0:
        print(f, "equal"); continue
    print(f, "d first diff", idx[0], "count", len(idx), "last", idx[-1], "| e first diff", idxe[0] if len(idxe) else None,
          "count", len(idxe), "| max abs dd", np.max(np.abs(a - ref)), "rel at first", abs(a[idx[0]] - ref[idx[0]]) / abs(ref[idx[0]]))
PY
