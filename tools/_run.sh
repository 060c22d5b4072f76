mkdir -p gpurun_out
python -m pytest tests/test_gpu_edge.py -q -rs -k "hyperelastic" 2>&1 | tail -3
FE_LIB_PATH=paper_1903_08243_b200/libfeb200_old.so python -m pytest tests/test_gpu_edge.py -q -rs -k "hyperelastic" 2>&1 | tail -2
