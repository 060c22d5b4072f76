mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "C1 or golden or mass" > gpurun_out/pytest_c1d.log 2>&1; tail -1 gpurun_out/pytest_c1d.log
for i in 1 2 3; do
echo "new $(python tools/profile_apply.py --config C1 --time --reps 30 2>&1 | tail -1)"
echo "old $(FE_LIB_PATH=paper_1903_08243_b200/libfeb200_old.so python tools/profile_apply.py --config C1 --time --reps 30 2>&1 | tail -1)"
done > gpurun_out/sweep_c1det.txt 2>&1
cut -c1-140 gpurun_out/sweep_c1det.txt
