FE_PAIR_CFG=2 python -m pytest tests -q -m gpu -x -k "quad or elasticity or C4" > gpurun_out/r2az_pytest.log 2>&1
tail -2 gpurun_out/r2az_pytest.log
python bench.py --config C4 --steps 20 --warmup 3 > gpurun_out/r2az_c4_base.log 2>&1
FE_PAIR_CFG=2 python bench.py --config C4 --steps 20 --warmup 3 > gpurun_out/r2az_c4_eo.log 2>&1
python tools/bench_table.py gpurun_out/r2az_c4_base.log gpurun_out/r2az_c4_eo.log
