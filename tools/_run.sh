mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "solver or diagonal or cg" > gpurun_out/pytest_solver.log 2>&1; tail -3 gpurun_out/pytest_solver.log
