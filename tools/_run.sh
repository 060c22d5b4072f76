mkdir -p gpurun_out
export FE_LIB_PATH=paper_1903_08243_b200/libfeb200_plq56.so
python -m pytest tests -m gpu -x -q -k "C3-Q5 or C3-Q6" > gpurun_out/pytest_plq56.log 2>&1; tail -1 gpurun_out/pytest_plq56.log
for c in C3-Q5 C3-Q6; do
echo "plane $(python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
echo "team $(FE_NO_PLANE=1 python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
done > gpurun_out/sweep_plq56.txt 2>&1
cut -c1-200 gpurun_out/sweep_plq56.txt
