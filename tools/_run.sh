mkdir -p gpurun_out
for lib in libfeb200 libfeb200_mm4 libfeb200_mm5 libfeb200_mm6; do
echo "$lib $(FE_LIB_PATH=paper_1903_08243_b200/$lib.so python tools/profile_apply.py --config C2-P1 --time --reps 30 2>&1 | tail -1)"
done > gpurun_out/sweep_macro_minb.txt 2>&1
cut -c1-190 gpurun_out/sweep_macro_minb.txt
