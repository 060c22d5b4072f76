mkdir -p gpurun_out
python -m pytest tests/test_gpu_coverage.py -q -k alternative > gpurun_out/pytest_alt.log 2>&1; tail -3 gpurun_out/pytest_alt.log
