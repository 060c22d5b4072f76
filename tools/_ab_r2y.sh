python -m pytest tests -q -m gpu -x -k "C2 or tet or helmholtz or coverage or edge or fullsize" > gpurun_out/r2y_pytest.log 2>&1
tail -2 gpurun_out/r2y_pytest.log
python bench.py --config C2 --steps 20 --warmup 5 > gpurun_out/r2y_c2_pipe.log 2>&1
FE_NO_MACRO_PIPE=1 python bench.py --config C2 --steps 20 --warmup 5 > gpurun_out/r2y_c2_nopipe.log 2>&1
FE_MACRO_WAVES=2 python bench.py --config C2 --steps 20 --warmup 5 > gpurun_out/r2y_c2_pipe_w2.log 2>&1
python tools/bench_table.py gpurun_out/r2y_c2_pipe.log gpurun_out/r2y_c2_nopipe.log gpurun_out/r2y_c2_pipe_w2.log
