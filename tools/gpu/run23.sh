set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in 9 72 136 264; do
BSE_SB2ST_MODE=$m BSE_DEBUG_HASH=1 timeout 900 python tools/determinism_probe.py --n 4608 --procs 1 --reps 30 --values > gpurun_out/det_delay$m.log 2>&1
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --n=4608 --steps 2 --warmup 3 --transport host > gpurun_out/bench_bc_host2.json 2> gpurun_out/bench_bc_host2.err
echo "rc=$?" >> gpurun_out/bench_bc_host2.err
