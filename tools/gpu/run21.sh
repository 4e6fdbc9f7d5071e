set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/pytest_all21.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_all21.log
timeout 900 python -m pytest tests/test_gpu_bc.py tests/test_gpu_dist.py -q > gpurun_out/pytest_bc21b.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_bc21b.log
