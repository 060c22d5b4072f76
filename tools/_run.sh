mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_final2.log 2>&1; tail -1 gpurun_out/pytest_final2.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final2.log 2>&1; tail -2 gpurun_out/smoke_final2.log
