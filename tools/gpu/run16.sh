set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
BSE_BUILD_MODE=1 timeout 900 python tools/determinism_probe.py --n 4608 --procs 2 --reps 60 --native > gpurun_out/det_mode1.log 2>&1
BSE_BUILD_MODE=2 timeout 900 python tools/determinism_probe.py --n 4608 --procs 2 --reps 60 --native > gpurun_out/det_mode2.log 2>&1
