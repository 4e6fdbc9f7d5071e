set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/profile_solve.py --n 16384 --reps 1 > gpurun_out/plain_cfg2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_r02.csv python tools/profile_solve.py --n 16384 --reps 1 > gpurun_out/ncu_cfg2.log 2>&1
python tools/profile_solve.py --complex --n 16384 --reps 0 > gpurun_out/plain_cfg3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3_r02.csv python tools/profile_solve.py --complex --n 16384 --reps 0 > gpurun_out/ncu_cfg3.log 2>&1
python tools/profile_solve.py --n 16384 --reps 0 > gpurun_out/plain_q2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:q2_apply -c 1 -o gpurun_out/q2_apply_r02 python tools/profile_solve.py --n 16384 --reps 0 > gpurun_out/ncu_q2.log 2>&1
ls -la gpurun_out
