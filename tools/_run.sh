mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v14.log 2>&1; tail -1 gpurun_out/pytest_v14.log
tools/sweep.sh > gpurun_out/sweep_v14.txt 2>&1
python tools/fmt_sweep.py gpurun_out/sweep_v14.txt
python bench.py > gpurun_out/bench_v14.log 2>&1; tail -1 gpurun_out/bench_v14.log | cut -c1-300
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v14.log 2>&1; tail -1 gpurun_out/smoke_v14.log
