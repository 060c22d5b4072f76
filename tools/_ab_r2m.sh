for v in "" q6a q6b; do
  lib=""; [ -n "$v" ] && lib="FE_LIB_PATH=paper_1903_08243_b200/libfeb200_$v.so"
  env $lib python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2m_c3_${v:-base}.log 2>&1
done
python bench.py --steps 20 --warmup 5 > gpurun_out/r2m_bench.log 2>&1
python -m pytest tests -q -m gpu -x -k "C3 or coverage or fullsize_parity" > gpurun_out/r2m_pytest.log 2>&1
