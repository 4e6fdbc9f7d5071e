set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_complex.py tests/test_gpu_cli.py tests/test_gpu_errors.py tests/test_gpu_parity.py -q > gpurun_out/pytest_new3.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_new3.log
timeout 900 python bench.py --config 3 --steps 2 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/bench_cfg3_r3.json 2> gpurun_out/bench_cfg3_r3.err
echo "rc=$?" >> gpurun_out/bench_cfg3_r3.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_r3.json 2> gpurun_out/bench_cfg2_r3.err
echo "rc=$?" >> gpurun_out/bench_cfg2_r3.err
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_all3.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_all3.log
