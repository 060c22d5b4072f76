mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "C4-quad or quadrilateral-3 or quadrilateral-4" > gpurun_out/pytest_c2d.log 2>&1; tail -1 gpurun_out/pytest_c2d.log
for c in C4-quad-Q3 C4-quad-Q4; do
echo "cell2d $(python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
echo "pair $(FE_NO_CELL2D=1 python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
done > gpurun_out/sweep_cell2d.txt 2>&1
cut -c1-200 gpurun_out/sweep_cell2d.txt
