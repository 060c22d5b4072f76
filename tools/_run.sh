mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "C2-P1 or C2-P2 or macro or tetrahedron-1 or tetrahedron-2" > gpurun_out/pytest_split2.log 2>&1; tail -1 gpurun_out/pytest_split2.log
for lib in libfeb200 libfeb200_slowrcp libfeb200_base; do for c in C2-P1 C2-P2; do
echo "$lib $(FE_LIB_PATH=paper_1903_08243_b200/$lib.so python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
done; done > gpurun_out/sweep_split2.txt 2>&1
cut -c1-200 gpurun_out/sweep_split2.txt
