set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all7.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_all7.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke7.log 2>&1
echo "rc=$?" >> gpurun_out/smoke7.log
/usr/bin/time -v timeout 1200 python bench.py > gpurun_out/bench_default7.json 2> gpurun_out/bench_default7.err
/usr/bin/time -v timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref7.json 2> gpurun_out/bench_ref7.err
