set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python bench.py --bc --n 16384 --steps 2 --warmup 3 --transport nccl > gpurun_out/bench_bc_w1_n16384.json 2> gpurun_out/bench_bc_w1_n16384.err
echo "rc=$?" >> gpurun_out/bench_bc_w1_n16384.err
timeout 2400 python bench.py --bc --n 32768 --nb 1024 --steps 1 --warmup 3 --transport nccl --e2e-steps 0 > gpurun_out/bench_bc_w1_n32768.json 2> gpurun_out/bench_bc_w1_n32768.err
echo "rc=$?" >> gpurun_out/bench_bc_w1_n32768.err
