set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_bc.py tests/test_gpu_ozgemm.py tests/test_gpu_dist.py -q > gpurun_out/pytest_bc33.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_bc33.log
export NCCL_DEBUG=WARN
timeout 1800 python bench.py --bc --n 16384 --steps 2 --warmup 3 --transport nccl > gpurun_out/bench_bc_w1_n16384_oz.json 2> gpurun_out/bench_bc_w1_n16384_oz.err
echo "rc=$?" >> gpurun_out/bench_bc_w1_n16384_oz.err
timeout 2400 python bench.py --bc --n 32768 --nb 1024 --steps 1 --warmup 3 --transport nccl --e2e-steps 0 > gpurun_out/bench_bc_w1_n32768_oz.json 2> gpurun_out/bench_bc_w1_n32768_oz.err
echo "rc=$?" >> gpurun_out/bench_bc_w1_n32768_oz.err
timeout 900 python bench.py --no-cpu-baseline --no-native --no-drop-in > gpurun_out/bench_cfg2_ws.json 2>/dev/null
