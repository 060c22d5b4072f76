mkdir -p gpurun_out
python -m pytest tests/test_gpu_bench.py -x -q > gpurun_out/pytest_bench.log 2>&1; tail -3 gpurun_out/pytest_bench.log
