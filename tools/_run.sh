mkdir -p gpurun_out
for lib in libfeb200 libfeb200_u1 libfeb200_u2; do
echo "$lib $(FE_LIB_PATH=paper_1903_08243_b200/$lib.so python tools/profile_apply.py --config C5 --time --reps 10 2>&1 | tail -1)"
done > gpurun_out/sweep_c5unr.txt 2>&1
cut -c1-150 gpurun_out/sweep_c5unr.txt
