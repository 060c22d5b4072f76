mkdir -p gpurun_out
FE_WARPCELL=1 python -m pytest tests -m gpu -x -q -k "C3-Q4 or C3-Q5 or C3-Q6 or laplacian_scalar-hexahedron" > gpurun_out/pytest_wc.log 2>&1; tail -1 gpurun_out/pytest_wc.log
for c in C3-Q4 C3-Q5 C3-Q6; do
echo "warpcell $(FE_WARPCELL=1 python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
echo "current $(python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
done > gpurun_out/sweep_wc.txt 2>&1
cut -c1-200 gpurun_out/sweep_wc.txt
