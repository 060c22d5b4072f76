mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_v17.log 2>&1; tail -1 gpurun_out/pytest_v17.log
tools/sweep.sh > gpurun_out/sweep_v17.txt 2>&1
python tools/fmt_sweep.py gpurun_out/sweep_v17.txt
python bench.py > gpurun_out/bench_v17.log 2>&1; tail -1 gpurun_out/bench_v17.log | cut -c1-200
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v17.log 2>&1; tail -1 gpurun_out/smoke_v17.log
