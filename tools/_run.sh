mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "C1 or golden or triangle or range" > gpurun_out/pytest_c1m.log 2>&1; tail -1 gpurun_out/pytest_c1m.log
for i in 1 2; do
echo "macro $(python tools/profile_apply.py --config C1 --time --reps 30 2>&1 | tail -1)"
echo "nomacro $(FE_NO_MACRO=1 python tools/profile_apply.py --config C1 --time --reps 30 2>&1 | tail -1)"
done > gpurun_out/sweep_c1macro.txt 2>&1
cut -c1-200 gpurun_out/sweep_c1macro.txt
