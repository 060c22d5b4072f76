python -m pytest tests -q -m gpu > gpurun_out/r2k_pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/r2k_bench.log 2>&1
FE_E2E_THREADS=1 python bench.py --steps 5 --warmup 3 > gpurun_out/r2k_bench_e2e1.log 2>&1
FE_E2E_THREADS=8 python bench.py --steps 5 --warmup 3 > gpurun_out/r2k_bench_e2e8.log 2>&1
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2k_bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2k_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/r2k_ncu_bench.log 2>&1
