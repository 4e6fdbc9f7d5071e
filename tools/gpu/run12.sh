set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
BSE_OZ_ENGINE=2 timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_e2.json 2> gpurun_out/bench_e2.err
BSE_OZ_ENGINE=0 timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_e0.json 2> gpurun_out/bench_e0.err
BSE_OZ_ENGINE=1 timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_e1.json 2> gpurun_out/bench_e1.err
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_all12.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_all12.log
