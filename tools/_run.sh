mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_v16.log 2>&1; tail -1 gpurun_out/pytest_v16.log
tools/sweep.sh > gpurun_out/sweep_v16.txt 2>&1
python tools/fmt_sweep.py gpurun_out/sweep_v16.txt
python bench.py > gpurun_out/bench_v16.log 2>&1; tail -1 gpurun_out/bench_v16.log | cut -c1-300
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v16.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_bench_v16.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_v16.log 2>&1; tail -1 gpurun_out/bench_ref_v16.log | cut -c1-200
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v16.log 2>&1; tail -2 gpurun_out/smoke_v16.log
