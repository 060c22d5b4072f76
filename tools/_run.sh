mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "neohookean or C5 or C6 or tangent or diagonal" > gpurun_out/pytest_nh.log 2>&1; tail -1 gpurun_out/pytest_nh.log
for c in C5 C6; do
echo "new $(python tools/profile_apply.py --config $c --time --reps 10 2>&1 | tail -1)"
echo "old $(FE_LIB_PATH=paper_1903_08243_b200/libfeb200_old.so python tools/profile_apply.py --config $c --time --reps 10 2>&1 | tail -1)"
done > gpurun_out/sweep_nh.txt 2>&1
cut -c1-200 gpurun_out/sweep_nh.txt
