set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out /tmp/dump
rm -f /tmp/dump/*
BSE_DEBUG_DUMP=/tmp/dump BSE_DEBUG_HASH=1 timeout 900 python tools/determinism_probe.py --n 4608 --procs 2 --reps 150 --values > gpurun_out/det_dump.log 2>&1
python - <<'PY' > gpurun_out/det_dump_analysis.log 2>&1
import glob, numpy as np, collections
files = sorted(glob.glob('/tmp/dump/d_*.bin'))
arrs = {f: np.fromfile(f) for f in files}
import hashlib
cnt = collections.Counter(hashlib.sha1(a.tobytes()).hexdigest() for a in arrs.values())
ref_h = cnt.most_common(1)[0][0]
ref = next(a for a in arrs.values() if hashlib.sha1(a.tobytes()).hexdigest() == ref_h)
print("runs", len(arrs), "distinct", len(cnt))
for f, a in arrs.items():
    if hashlib.sha1(a.tobytes()).hexdigest() != ref_h:
        idx = np.nonzero(a != ref)[0]
        e = np.fromfile(f.replace('/d_', '/e_'))
        print(f, "first diff index", idx[0], "count", len(idx), "last", idx[-1], "max abs", np.max(np.abs(a - ref)), "first vals", a[idx[0]], ref[idx[0]])
PY
