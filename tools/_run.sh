mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v13.log 2>&1; tail -1 gpurun_out/pytest_v13.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v13.log 2>&1; tail -2 gpurun_out/smoke_v13.log
python bench.py > gpurun_out/bench_v13.log 2>&1; tail -1 gpurun_out/bench_v13.log | cut -c1-600
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v13.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_bench_v13.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_v13.log 2>&1; tail -1 gpurun_out/bench_ref_v13.log | cut -c1-300
