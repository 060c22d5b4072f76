mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "elasticity or C4 or golden" > gpurun_out/pytest_el.log 2>&1; tail -1 gpurun_out/pytest_el.log
for c in C4-quad-Q1 C4-quad-Q2 C4-hex-Q1 C4-hex-Q2 C4-hex-Q3; do
echo "new $(python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
echo "old $(FE_LIB_PATH=paper_1903_08243_b200/libfeb200_old.so python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
done > gpurun_out/sweep_el.txt 2>&1
cut -c1-160 gpurun_out/sweep_el.txt
