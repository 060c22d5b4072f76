mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v11.log 2>&1; tail -1 gpurun_out/pytest_v11.log
tools/sweep.sh > gpurun_out/sweep_v11.txt 2>&1
python bench.py > gpurun_out/bench_v11.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v11.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_bench_v11.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v11.log 2>&1; tail -3 gpurun_out/smoke_v11.log
