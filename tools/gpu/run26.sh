set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozgemm.py -x -q -k "tcgen05" > gpurun_out/pytest_i8mma26.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_i8mma26.log
export BSE_OZ_TRACE=1
timeout 300 python tools/profile_oz.py --engine 0 --reps 3 > gpurun_out/t26_big.log 2>&1
timeout 300 python tools/profile_oz.py --engine 0 --reps 3 --m 16384 --n 16384 --k 256 --tb 1 > gpurun_out/t26_k256.log 2>&1
timeout 300 python tools/profile_oz.py --engine 0 --reps 3 --m 16384 --n 16384 --k 1024 --tb 1 > gpurun_out/t26_k1024.log 2>&1
timeout 300 python tools/profile_oz.py --engine 0 --reps 3 --m 16384 --n 16384 --k 512 --tb 1 > gpurun_out/t26_k512.log 2>&1
