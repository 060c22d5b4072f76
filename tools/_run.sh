mkdir -p gpurun_out
for lib in libfeb200 libfeb200_xs33 libfeb200_xs36 libfeb200_xs40; do for c in C3-Q3 C3-Q4; do
echo "$lib $(FE_LIB_PATH=paper_1903_08243_b200/$lib.so python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
done; done > gpurun_out/sweep_xs.txt 2>&1
cut -c1-175 gpurun_out/sweep_xs.txt
FE_LIB_PATH=paper_1903_08243_b200/libfeb200_xs33.so python -m pytest tests -m gpu -x -q -k "C3-Q3 or C3-Q4" 2>&1 | tail -1
