set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export BSE_OZ_TRACE=1
for rep in 1 2; do
for epi in 1 2; do for sl in 0 1; do
echo "== epi $epi sleep $sl rep $rep"
BSE_I8_EPI=$epi BSE_I8_SLEEP=$sl timeout 300 python tools/profile_oz.py --engine 0 --reps 3 --m 16384 --n 16384 --k 256 --tb 1 2>&1 | grep "\[oz\]" | tail -1 | cut -c1-70
BSE_I8_EPI=$epi BSE_I8_SLEEP=$sl timeout 300 python tools/profile_oz.py --engine 0 --reps 3 2>&1 | grep "\[oz\]" | tail -1
done; done
echo "== cutlass rep $rep"
timeout 300 python tools/profile_oz.py --engine 2 --reps 3 2>&1 | grep "\[oz\]" | tail -1
done > gpurun_out/i8_ab27.log 2>&1
