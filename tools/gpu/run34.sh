set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --no-native --no-drop-in --e2e-steps 0 --no-verify > gpurun_out/bench_ws_a.json 2> gpurun_out/bench_ws_a.err
echo "rc=$?" >> gpurun_out/bench_ws_a.err
timeout 600 python bench.py --no-cpu-baseline --no-native --no-drop-in --e2e-steps 0 > gpurun_out/bench_ws_b.json 2> gpurun_out/bench_ws_b.err
echo "rc=$?" >> gpurun_out/bench_ws_b.err
timeout 600 python bench.py --no-cpu-baseline --no-native --no-drop-in > gpurun_out/bench_ws_c.json 2> gpurun_out/bench_ws_c.err
echo "rc=$?" >> gpurun_out/bench_ws_c.err
