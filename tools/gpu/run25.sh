set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in 264 72 60; do
BSE_SB2ST_MODE=$m BSE_DEBUG_HASH=1 timeout 900 python tools/determinism_probe.py --n 4608 --procs 1 --reps 30 --values > gpurun_out/fix_delay$m.log 2>&1
done
BSE_DEBUG_HASH=1 BSE_BUILD_MODE=1 BSE_DC_MAIN=1 timeout 1500 python tools/determinism_probe.py --n 4608 --procs 2 --reps 150 --native > gpurun_out/fix_hash_p2.log 2>&1
timeout 900 python tools/determinism_probe.py --n 4608 --procs 3 --reps 60 > gpurun_out/fix_p3.log 2>&1
BSE_BENCH_N=4608 BSE_BENCH_TRANSPORT=host python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench_bc_host2.json 2> gpurun_out/bench_bc_host2.err
echo "rc=$?" >> gpurun_out/bench_bc_host2.err
