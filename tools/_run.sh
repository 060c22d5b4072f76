mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "C4-quad-Q1 or C4-quad-Q2 or C4-hex-Q1 or quadrilateral-1 or quadrilateral-2 or hexahedron-1" > gpurun_out/pytest_qadj.log 2>&1; tail -1 gpurun_out/pytest_qadj.log
for i in 1 2; do for c in C4-quad-Q1 C4-quad-Q2 C4-hex-Q1; do
echo "adj $(python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
echo "inv $(FE_LIB_PATH=paper_1903_08243_b200/libfeb200_noadj.so python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
done; done > gpurun_out/sweep_qadj.txt 2>&1
cut -c1-170 gpurun_out/sweep_qadj.txt
