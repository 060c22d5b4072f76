mkdir -p gpurun_out
for i in 1 2; do for lib in libfeb200 libfeb200_pf libfeb200_pf2; do
echo "$lib $(FE_LIB_PATH=paper_1903_08243_b200/$lib.so python tools/profile_apply.py --config C2-P1 --time --reps 30 2>&1 | tail -1)"
done; done > gpurun_out/sweep_l2pf.txt 2>&1
cut -c1-175 gpurun_out/sweep_l2pf.txt
