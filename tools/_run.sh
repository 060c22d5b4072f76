mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "C3-Q1 or hexahedron-1" > gpurun_out/pytest_hw.log 2>&1; tail -1 gpurun_out/pytest_hw.log
for m in 3 4; do for w in 0 1 2; do
echo "minb=$m waves=$w $(FE_HEXQ1_MINB=$m FE_HEXQ1_WAVES=$w python tools/profile_apply.py --config C3-Q1 --time --reps 30 2>&1 | tail -1)"
done; done > gpurun_out/sweep_hq1_waves.txt 2>&1
cut -c1-200 gpurun_out/sweep_hq1_waves.txt
