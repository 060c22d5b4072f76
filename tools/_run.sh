mkdir -p gpurun_out
for lib in libfeb200 libfeb200_g3; do
 export FE_LIB_PATH=$PWD/paper_1903_08243_b200/$lib.so
 echo "== $lib"
 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -x -q 2>&1 | tail -1
 tools/sweep_subset.sh C2-P1 C2-P1 C1
done > gpurun_out/sweep_group2.txt 2>&1
