set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/diag_complex_biorth.py 512 > gpurun_out/diag_biorth.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_errors.py tests/test_gpu_complex.py tests/test_gpu_parity.py tests/test_gpu_cli.py -q > gpurun_out/pytest_new4.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_new4.log
BSE_SB2ST_TRACE=2000 timeout 300 python tools/sb2st_trace.py --n 16384 > gpurun_out/sb2st_trace.log 2>&1
