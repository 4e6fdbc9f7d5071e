set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
F="--no-cpu-baseline --no-native --no-drop-in --e2e-steps 0 --steps 3"
BSE_POTRF_OZ_OLD=1 timeout 600 python bench.py $F > gpurun_out/thr_36_old.json 2>/dev/null
for w in 36 35 34 33; do
BSE_OZ_MIN_WORK_LOG2=$w timeout 600 python bench.py $F > gpurun_out/thr_$w.json 2>/dev/null
done
BSE_OZ_MIN_WORK_LOG2=34 BSE_DC_OZ_NODES=4 timeout 600 python bench.py $F > gpurun_out/thr_34_dc4.json 2>/dev/null
BSE_OZ_MIN_WORK_LOG2=33 BSE_DC_OZ_NODES=8 timeout 600 python bench.py $F > gpurun_out/thr_33_dc8.json 2>/dev/null
BSE_OZ_MIN_WORK_LOG2=36 timeout 600 python bench.py $F > gpurun_out/thr_36b.json 2>/dev/null
