set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do
timeout -s USR1 -k 20 400 python -c "
import faulthandler, signal, sys, runpy
faulthandler.register(signal.SIGUSR1, all_threads=True)
sys.argv=['bench.py','--no-cpu-baseline','--no-native','--no-drop-in']
runpy.run_path('bench.py', run_name='__main__')
" > gpurun_out/loop_$i.json 2> gpurun_out/loop_$i.err
echo "rc=$?" >> gpurun_out/loop_$i.err
done
