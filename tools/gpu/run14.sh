set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for e in 2 0 1; do
BSE_OZ_ENGINE=$e timeout 900 python tools/determinism_probe.py --n 4608 --procs 2 --reps 16 > gpurun_out/det_e$e.log 2>&1
done
