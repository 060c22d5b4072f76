python -m pytest tests/test_gpu_coverage.py -q -m gpu -x -k "c3_rule" > gpurun_out/r2af_pytest.log 2>&1
tail -3 gpurun_out/r2af_pytest.log
python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2af_c3_direct.log 2>&1
FE_TK_COLLOC56=1 python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2af_c3_colloc.log 2>&1
FE_TK_COLLOC56=1 FE_LIB_PATH=paper_1903_08243_b200/libfeb200_c1.so python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2af_c3_colloc_c1.log 2>&1
FE_TK_COLLOC56=1 FE_LIB_PATH=paper_1903_08243_b200/libfeb200_c2.so python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2af_c3_colloc_c2.log 2>&1
python tools/bench_table.py gpurun_out/r2af_c3_direct.log gpurun_out/r2af_c3_colloc.log gpurun_out/r2af_c3_colloc_c1.log gpurun_out/r2af_c3_colloc_c2.log
