mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "C6 or tangent or neohookean or C5" > gpurun_out/pytest_tangent.log 2>&1; tail -3 gpurun_out/pytest_tangent.log
tools/sweep_subset.sh C5 C6 > gpurun_out/sweep_tangent.txt 2>&1; cut -c1-250 gpurun_out/sweep_tangent.txt
