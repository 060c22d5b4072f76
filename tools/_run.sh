mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_coverage.py -m gpu -x -q > gpurun_out/pytest_rcp.log 2>&1; tail -1 gpurun_out/pytest_rcp.log
tools/sweep.sh > gpurun_out/sweep_v8.txt 2>&1
