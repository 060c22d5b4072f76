mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "C3-Q5 or C3-Q6 or C4-hex-Q2 or C4-hex-Q3 or hexahedron or quadrilateral" > gpurun_out/pytest_tadj.log 2>&1; tail -1 gpurun_out/pytest_tadj.log
for c in C3-Q5 C3-Q6 C4-hex-Q2 C4-hex-Q3; do
echo "adj $(python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
echo "inv $(FE_LIB_PATH=paper_1903_08243_b200/libfeb200_noadj.so python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
done > gpurun_out/sweep_tadj.txt 2>&1
cut -c1-170 gpurun_out/sweep_tadj.txt
