set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/pytest_final2.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_final2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final2.log 2>&1
echo "rc=$?" >> gpurun_out/smoke_final2.log
timeout 1500 python bench.py > gpurun_out/bench_cfg2_final4.json 2> gpurun_out/bench_cfg2_final4.err
for i in 1 2 3 4 5 6 7 8; do
timeout -k 20 400 python bench.py --no-cpu-baseline --no-native --no-drop-in > gpurun_out/loopb_$i.json 2> gpurun_out/loopb_$i.err
echo "rc=$?" >> gpurun_out/loopb_$i.err
done
timeout 1800 python bench.py --bc --n 16384 --steps 2 --warmup 3 --transport nccl > gpurun_out/bench_bc_w1_n16384_final.json 2> gpurun_out/bench_bc_w1_n16384_final.err
timeout 2400 python bench.py --bc --n 32768 --nb 1024 --steps 1 --warmup 3 --transport nccl --e2e-steps 0 > gpurun_out/bench_bc_w1_n32768_final.json 2> gpurun_out/bench_bc_w1_n32768_final.err
timeout 1500 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_cfg3_final4.json 2> gpurun_out/bench_cfg3_final4.err
