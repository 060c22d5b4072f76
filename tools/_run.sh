mkdir -p gpurun_out
python -m pytest tests/test_gpu_edge.py -q > gpurun_out/pytest_edge.log 2>&1; tail -15 gpurun_out/pytest_edge.log
