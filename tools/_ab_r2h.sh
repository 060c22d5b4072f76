python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2h_c3_new.log 2>&1
FE_LIB_PATH=paper_1903_08243_b200/libfeb200_vtx_u3m1.so python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2h_c3_old.log 2>&1
python bench.py --config C4 --steps 10 --warmup 3 > gpurun_out/r2h_c4_new.log 2>&1
FE_LIB_PATH=paper_1903_08243_b200/libfeb200_vtx_u3m1.so python bench.py --config C4 --steps 10 --warmup 3 > gpurun_out/r2h_c4_old.log 2>&1
FE_LIB_PATH=paper_1903_08243_b200/libfeb200_tkstrict.so python bench.py --config C4 --steps 10 --warmup 3 > gpurun_out/r2h_c4_strict.log 2>&1
python bench.py --config C2 --steps 10 --warmup 3 > gpurun_out/r2h_c2_new.log 2>&1
FE_LIB_PATH=paper_1903_08243_b200/libfeb200_macro3.so python bench.py --config C2 --steps 10 --warmup 3 > gpurun_out/r2h_c2_m3.log 2>&1
FE_LIB_PATH=paper_1903_08243_b200/libfeb200_macro4.so python bench.py --config C2 --steps 10 --warmup 3 > gpurun_out/r2h_c2_m4.log 2>&1
for c in C5 C3-Q6 C3-Q5 C4-hex-Q3; do mkdir -p /tmp/prof; done
