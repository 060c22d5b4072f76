python -m pytest tests -q -m gpu -x -k "parity or edge or abi or fullsize or slabs or solver" > gpurun_out/r2ao_pytest.log 2>&1
tail -2 gpurun_out/r2ao_pytest.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r2ao_2phase.log 2>&1
FE_FILL_2PHASE_MB=0 python bench.py --steps 10 --warmup 3 > gpurun_out/r2ao_1phase.log 2>&1
FE_FILL_2PHASE_MB=8 python bench.py --steps 10 --warmup 3 > gpurun_out/r2ao_2phase8.log 2>&1
python tools/bench_table.py gpurun_out/r2ao_2phase.log gpurun_out/r2ao_1phase.log gpurun_out/r2ao_2phase8.log
