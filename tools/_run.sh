mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "C3-Q1 or hexahedron-1 or laplacian_scalar-hexahedron" > gpurun_out/pytest_hq1b.log 2>&1; tail -1 gpurun_out/pytest_hq1b.log
for m in 3 1 4; do
echo "new minb=$m $(FE_HEXQ1_MINB=$m python tools/profile_apply.py --config C3-Q1 --time --reps 30 2>&1 | tail -1)"
done > gpurun_out/sweep_hq1b.txt 2>&1
echo "old $(FE_LIB_PATH=paper_1903_08243_b200/libfeb200_old.so python tools/profile_apply.py --config C3-Q1 --time --reps 30 2>&1 | tail -1)" >> gpurun_out/sweep_hq1b.txt
cut -c1-200 gpurun_out/sweep_hq1b.txt
