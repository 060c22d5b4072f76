mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "C6 or tangent" > gpurun_out/pytest_c6s.log 2>&1; tail -1 gpurun_out/pytest_c6s.log
echo "new $(python tools/profile_apply.py --config C6 --time --reps 10 2>&1 | tail -1)" > gpurun_out/sweep_c6s.txt
echo "old $(FE_LIB_PATH=paper_1903_08243_b200/libfeb200_old.so python tools/profile_apply.py --config C6 --time --reps 10 2>&1 | tail -1)" >> gpurun_out/sweep_c6s.txt
cut -c1-170 gpurun_out/sweep_c6s.txt
