set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
BSE_DEBUG_HASH=1 BSE_BUILD_MODE=1 BSE_DC_MAIN=1 timeout 1500 python tools/determinism_probe.py --n 4608 --procs 2 --reps 100 --native > gpurun_out/det_hash.log 2>&1
