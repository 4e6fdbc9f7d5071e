set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py tests/test_gpu_errors.py tests/test_gpu_dense.py tests/test_gpu_complex.py tests/test_gpu_verify.py tests/test_gpu_ozgemm.py tests/test_gpu_bc.py -q > gpurun_out/pytest_thr.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_thr.log
timeout 1500 python bench.py > gpurun_out/bench_cfg2_final3.json 2> gpurun_out/bench_cfg2_final3.err
timeout 1500 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_cfg3_final3.json 2> gpurun_out/bench_cfg3_final3.err
