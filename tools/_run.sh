mkdir -p gpurun_out
FE_LIB_PATH=paper_1903_08243_b200/libfeb200_ncx2.so python -m pytest tests -m gpu -x -q -k "C2-P1 or macro or range" > gpurun_out/pytest_ncx2.log 2>&1; tail -1 gpurun_out/pytest_ncx2.log
for i in 1 2; do
echo "ncx1 $(python tools/profile_apply.py --config C2-P1 --time --reps 30 2>&1 | tail -1)"
echo "ncx2 $(FE_LIB_PATH=paper_1903_08243_b200/libfeb200_ncx2.so python tools/profile_apply.py --config C2-P1 --time --reps 30 2>&1 | tail -1)"
done >> gpurun_out/sweep_p1const.txt 2>&1
tail -4 gpurun_out/sweep_p1const.txt | cut -c1-200
