mkdir -p gpurun_out
tools/sweep.sh > gpurun_out/sweep_v10.txt 2>&1
for v in cu2 cu5; do echo "== $v"; FE_LIB_PATH=$PWD/paper_1903_08243_b200/libfeb200_$v.so tools/sweep_subset.sh C3-Q3 C3-Q4; done >> gpurun_out/sweep_v10.txt 2>&1
