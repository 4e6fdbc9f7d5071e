set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/determinism_probe.py --n 4608 --procs 2 --reps 6 > gpurun_out/det_4608_p2.log 2>&1
timeout 600 python tools/determinism_probe.py --n 4608 --procs 3 --reps 6 --native > gpurun_out/det_4608_p3_native.log 2>&1
timeout 600 python tools/determinism_probe.py --n 2300 --procs 4 --reps 8 > gpurun_out/det_2300_p4.log 2>&1
timeout 600 python tools/determinism_probe.py --n 4608 --procs 1 --reps 8 > gpurun_out/det_4608_p1.log 2>&1
