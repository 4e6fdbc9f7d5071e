set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in 0 1 2 3; do
BSE_SB2ST_MODE=$m BSE_DEBUG_HASH=1 timeout 900 python tools/determinism_probe.py --n 4608 --procs 2 --reps 120 --values > gpurun_out/det_sbmode$m.log 2>&1
done
