set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_complex.py tests/test_gpu_cli.py -x -q > gpurun_out/pytest_new.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_new.log
timeout 900 python bench.py --config 3 --steps 2 --warmup 3 --e2e-steps 2 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
echo "rc=$?" >> gpurun_out/bench_cfg3.err
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_all.log
timeout 1500 python tools/validate_cost_model.py --n 1024 2048 --rounds 3 --points 2 --out gpurun_out/cost_model_validation.json > gpurun_out/cost_val.log 2>&1
echo "rc=$?" >> gpurun_out/cost_val.log
