mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_coverage.py -m gpu -x -q -k "C3 or laplacian_scalar or hex" > gpurun_out/pytest_plane.log 2>&1; tail -3 gpurun_out/pytest_plane.log
tools/sweep_subset.sh C3-Q1 C3-Q2 C3-Q3 > gpurun_out/plane_on.jsonl
FE_NO_QCT=1 tools/sweep_subset.sh C3-Q1 >> gpurun_out/plane_on.jsonl
FE_NO_PLANE=1 tools/sweep_subset.sh C3-Q2 C3-Q3 > gpurun_out/plane_off.jsonl
cat gpurun_out/plane_on.jsonl gpurun_out/plane_off.jsonl
