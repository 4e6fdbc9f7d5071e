set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_eig.py tests/test_gpu_solve.py -q > gpurun_out/pytest_eig29.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_eig29.log
timeout 1500 python bench.py > gpurun_out/bench_cfg2_final2.json 2> gpurun_out/bench_cfg2_final2.err
BSE_SB2ST_MODE=1 timeout 900 python bench.py --no-cpu-baseline --no-native --no-drop-in --e2e-steps 0 > gpurun_out/bench_cfg2_diagkernel.json 2> gpurun_out/bench_cfg2_diagkernel.err
