mkdir -p gpurun_out
for i in 1 2; do for lib in libfeb200 libfeb200_p1m3 libfeb200_p1m4; do
echo "$lib $(FE_LIB_PATH=paper_1903_08243_b200/$lib.so python tools/profile_apply.py --config C3-Q2 --time --reps 20 2>&1 | tail -1)"
done; done > gpurun_out/sweep_p1minb.txt 2>&1
cut -c1-170 gpurun_out/sweep_p1minb.txt
