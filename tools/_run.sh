mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_unr.log 2>&1; tail -1 gpurun_out/pytest_unr.log
tools/sweep_subset.sh C3-Q1 C4-quad-Q1 C4-quad-Q2 C4-hex-Q1 C5 > gpurun_out/sweep_unr.txt 2>&1
