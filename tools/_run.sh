mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "C2-P1 or macro or range or slab" > gpurun_out/pytest_mw.log 2>&1; tail -1 gpurun_out/pytest_mw.log
for w in 0 1 2 4; do
echo "waves=$w $(FE_MACRO_WAVES=$w python tools/profile_apply.py --config C2-P1 --time --reps 30 2>&1 | tail -1)"
done > gpurun_out/sweep_macro_waves.txt 2>&1
cut -c1-200 gpurun_out/sweep_macro_waves.txt
