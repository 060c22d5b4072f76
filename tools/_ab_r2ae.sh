python -m pytest tests/test_gpu_coverage.py -q -m gpu -x -k "c3_rule" > gpurun_out/r2ae_pytest.log 2>&1
tail -3 gpurun_out/r2ae_pytest.log
python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2ae_c3_base.log 2>&1
FE_HEXLP=1 python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2ae_c3_lp.log 2>&1
python tools/bench_table.py gpurun_out/r2ae_c3_base.log gpurun_out/r2ae_c3_lp.log
