mkdir -p gpurun_out
FE_LIB_PATH=paper_1903_08243_b200/libfeb200_etadj.so python -m pytest tests -m gpu -x -q -k "C2-P3 or C2-P4 or C1 or alternative" 2>&1 | tail -1
for i in 1 2; do for c in C2-P3 C2-P4; do
echo "base $(python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
echo "adj $(FE_LIB_PATH=paper_1903_08243_b200/libfeb200_etadj.so python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
done; done > gpurun_out/sweep_etadj.txt 2>&1
cut -c1-150 gpurun_out/sweep_etadj.txt
