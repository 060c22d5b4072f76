mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "C2 or slab or range or macro or accumulate or tetrahedron" > gpurun_out/pytest_macro.log 2>&1; tail -3 gpurun_out/pytest_macro.log
for i in 1 2; do
echo "macro $(python tools/profile_apply.py --config C2-P1 --time --reps 20 2>&1 | tail -1)"
echo "nomacro $(FE_NO_MACRO=1 python tools/profile_apply.py --config C2-P1 --time --reps 20 2>&1 | tail -1)"
done > gpurun_out/sweep_macro.txt 2>&1
cut -c1-250 gpurun_out/sweep_macro.txt
