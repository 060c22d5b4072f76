python -m pytest tests -q -m gpu > gpurun_out/r2n_pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n_smoke.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/r2n_bench.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2n_bench_ref.log 2>&1
tail -3 gpurun_out/r2n_pytest_gpu.log; tail -2 gpurun_out/r2n_smoke.log
