set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export BSE_OZ_TRACE=1
for e in 2 1 0; do
timeout 300 python tools/profile_oz.py --engine $e --reps 3 > gpurun_out/t_big_e$e.log 2>&1
timeout 300 python tools/profile_oz.py --engine $e --reps 3 --m 16384 --n 16384 --k 256 --tb 1 > gpurun_out/t_k256_e$e.log 2>&1
timeout 300 python tools/profile_oz.py --engine $e --reps 3 --m 16384 --n 16384 --k 256 --tb 1 --lower > gpurun_out/t_k256l_e$e.log 2>&1
done
