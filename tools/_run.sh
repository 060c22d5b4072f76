mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "C1 or C2 or golden or alternative or tetrahedron or triangle" > gpurun_out/pytest_etc.log 2>&1; tail -1 gpurun_out/pytest_etc.log
for c in C1 C2-P3 C2-P4; do
echo "new $(python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
echo "old $(FE_LIB_PATH=paper_1903_08243_b200/libfeb200_old.so python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
done > gpurun_out/sweep_etc.txt 2>&1
cut -c1-170 gpurun_out/sweep_etc.txt
