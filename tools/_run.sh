mkdir -p gpurun_out
for c in C2-P3 C2-P4; do
echo "base $(python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
echo "nogeom $(FE_LIB_PATH=paper_1903_08243_b200/libfeb200_ablg.so python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
done > gpurun_out/sweep_ablg.txt 2>&1
cut -c1-140 gpurun_out/sweep_ablg.txt
