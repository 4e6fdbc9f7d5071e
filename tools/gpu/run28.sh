set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/pytest_final.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1
echo "rc=$?" >> gpurun_out/smoke_final.log
timeout 1500 python bench.py > gpurun_out/bench_cfg2_final.json 2> gpurun_out/bench_cfg2_final.err
timeout 1500 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg2_steps20.json 2> gpurun_out/bench_cfg2_steps20.err
timeout 1800 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err
timeout 1500 python bench.py --config 3 > gpurun_out/bench_cfg3_final.json 2> gpurun_out/bench_cfg3_final.err
timeout 900 python bench.py --config 1 > gpurun_out/bench_cfg1_final.json 2> gpurun_out/bench_cfg1_final.err
python tools/profile_solve.py --n 16384 --reps 1 > gpurun_out/plain_cfg2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_final.csv python tools/profile_solve.py --n 16384 --reps 1 > gpurun_out/ncu_cfg2.log 2>&1
python tools/profile_oz.py --engine 0 > gpurun_out/plain_oz.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:i8mma -s 1 -c 1 -o gpurun_out/i8mma_final python tools/profile_oz.py --engine 0 > gpurun_out/ncu_i8mma.log 2>&1
