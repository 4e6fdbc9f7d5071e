set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozgemm.py -x -q -k "tcgen05" > gpurun_out/pytest_i8mma.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_i8mma.log
timeout 300 python tools/bench_ozgemm.py --m 4096 --n 4096 --k 4096 --chunk 4096 > gpurun_out/oz_4096.log 2>&1
timeout 300 python tools/bench_ozgemm.py --m 16384 --n 4096 --k 16384 --chunk 4096 --no-dmma > gpurun_out/oz_16k.log 2>&1
timeout 300 python tools/bench_ozgemm.py --m 16384 --n 16384 --k 256 --chunk 4096 --tb 1 > gpurun_out/oz_k256.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_bc.py -q > gpurun_out/pytest_bc9.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_bc9.log
