set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
BSE_BUILD_MODE=1 BSE_DC_MAIN=1 timeout 900 python tools/determinism_probe.py --n 4608 --procs 2 --reps 80 --native > gpurun_out/det_dcmain.log 2>&1
timeout 900 python tools/determinism_probe.py --n 4608 --procs 2 --reps 80 --stedc > gpurun_out/det_stedc_real.log 2>&1
