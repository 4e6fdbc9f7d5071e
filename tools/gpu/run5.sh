set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/diag_complex_biorth.py 512 > gpurun_out/diag_biorth5.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_complex.py tests/test_gpu_solve.py tests/test_gpu_errors.py -q > gpurun_out/pytest_new5.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_new5.log
timeout 900 python bench.py --config 3 --steps 2 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/bench_cfg3_r5.json 2> gpurun_out/bench_cfg3_r5.err
timeout 900 python bench.py --config 1 --steps 5 --warmup 3 --e2e-steps 3 > gpurun_out/bench_cfg1_r5.json 2> gpurun_out/bench_cfg1_r5.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_r5.json 2> gpurun_out/bench_cfg2_r5.err
