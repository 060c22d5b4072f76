timeout 1500 python -m pytest tests -q -m gpu -x -k "parity or edge or abi or fullsize or slabs or solver or bench" > gpurun_out/r2ar_pytest.log 2>&1
tail -2 gpurun_out/r2ar_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2ar_prio.log 2>&1
FE_FILL_PRIO_MB=0 timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2ar_noprio.log 2>&1
FE_FILL_PRIO_MB=8 timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2ar_prio8.log 2>&1
python tools/bench_table.py gpurun_out/r2ar_prio.log gpurun_out/r2ar_noprio.log gpurun_out/r2ar_prio8.log
