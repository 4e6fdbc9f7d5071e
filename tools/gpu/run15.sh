set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/determinism_probe.py --n 4608 --procs 2 --reps 40 --values > gpurun_out/det_values.log 2>&1
timeout 900 python tools/determinism_probe.py --n 4608 --procs 2 --reps 40 --stedc > gpurun_out/det_stedc.log 2>&1
timeout 900 python tools/determinism_probe.py --n 4608 --procs 2 --reps 40 --native > gpurun_out/det_native.log 2>&1
