python -m pytest tests -q -m gpu -x -k "C3 or hex or edge or coverage or fullsize" > gpurun_out/r2p_pytest.log 2>&1
tail -3 gpurun_out/r2p_pytest.log
python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2p_c3.log 2>&1
FE_LIB_PATH=paper_1903_08243_b200/libfeb200_prcp.so python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2p_c3_prcp.log 2>&1
FE_NO_HEXQ2=1 python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2p_c3_noq2.log 2>&1
python tools/bench_table.py gpurun_out/r2p_c3.log gpurun_out/r2p_c3_prcp.log gpurun_out/r2p_c3_noq2.log
