mkdir -p gpurun_out
for v in w1 w2 w3; do echo "== $v"; FE_LIB_PATH=$PWD/paper_1903_08243_b200/libfeb200_$v.so tools/sweep_subset.sh C3-Q3 C3-Q4 C4-quad-Q3 C4-quad-Q4; done > gpurun_out/sweep_warps.txt 2>&1
echo "== default" >> gpurun_out/sweep_warps.txt; tools/sweep_subset.sh C3-Q3 C3-Q4 C4-quad-Q3 C4-quad-Q4 >> gpurun_out/sweep_warps.txt 2>&1
