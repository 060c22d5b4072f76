mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "C3-Q1 or hexahedron-1" > gpurun_out/pytest_hq1.log 2>&1; tail -2 gpurun_out/pytest_hq1.log
for m in 1 3 4; do echo "minb=$m $(FE_HEXQ1_MINB=$m python tools/profile_apply.py --config C3-Q1 --time --reps 20 2>&1 | tail -1)"; done > gpurun_out/sweep_hq1.txt
echo "qct $(FE_NO_HEXQ1=1 python tools/profile_apply.py --config C3-Q1 --time --reps 20 2>&1 | tail -1)" >> gpurun_out/sweep_hq1.txt
cut -c1-230 gpurun_out/sweep_hq1.txt
