python -m pytest tests -q -m gpu -x -k "quad or elasticity or C4 or edge" > gpurun_out/r2aq_pytest.log 2>&1
tail -2 gpurun_out/r2aq_pytest.log
python bench.py --config C4 --steps 20 --warmup 3 > gpurun_out/r2aq_c4.log 2>&1
python tools/bench_table.py gpurun_out/r2aq_c4.log
