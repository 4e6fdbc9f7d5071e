set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for e in 2 1 0; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_big_e$e.csv python tools/profile_oz.py --engine $e > gpurun_out/l_big_e$e.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_k256_e$e.csv python tools/profile_oz.py --engine $e --m 16384 --n 16384 --k 256 --tb 1 > gpurun_out/l_k256_e$e.log 2>&1
done
for e in 1 0; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:i8mma -s 1 -c 1 -o gpurun_out/i8mma_big_e$e python tools/profile_oz.py --engine $e > gpurun_out/f_big_e$e.log 2>&1
done
