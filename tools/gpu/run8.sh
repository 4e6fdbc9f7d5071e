set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_all8.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_all8.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke8.log 2>&1
echo "rc=$?" >> gpurun_out/smoke8.log
timeout 1200 python bench.py > gpurun_out/bench_default8.json 2> gpurun_out/bench_default8.err
echo "rc=$?" >> gpurun_out/bench_default8.err
