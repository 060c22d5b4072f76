mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; tail -1 gpurun_out/pytest_all.log
tools/sweep_subset.sh C3-Q1 C3-Q2 C3-Q3 C3-Q4 C3-Q5 C3-Q6 > gpurun_out/sweep_c3.txt
