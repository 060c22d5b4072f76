FE_LIB_PATH=paper_1903_08243_b200/libfeb200_rcp3.so python -m pytest tests -q -m gpu -x -k "parity or edge or coverage" > gpurun_out/r2au_pytest.log 2>&1
tail -2 gpurun_out/r2au_pytest.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r2au_base.log 2>&1
FE_LIB_PATH=paper_1903_08243_b200/libfeb200_rcp3.so python bench.py --steps 10 --warmup 3 > gpurun_out/r2au_rcp3.log 2>&1
python tools/bench_table.py gpurun_out/r2au_base.log gpurun_out/r2au_rcp3.log
