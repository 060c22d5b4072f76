for v in "" full full4; do
  lib=""; [ -n "$v" ] && lib="FE_LIB_PATH=paper_1903_08243_b200/libfeb200_$v.so"
  env $lib python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2aj_c3_${v:-base}.log 2>&1
done
python tools/bench_table.py gpurun_out/r2aj_c3_base.log gpurun_out/r2aj_c3_full.log gpurun_out/r2aj_c3_full4.log
FE_LIB_PATH=paper_1903_08243_b200/libfeb200_full.so python -m pytest tests -q -m gpu -x -k "C3 or c3_rule or hex" > gpurun_out/r2aj_pytest.log 2>&1
tail -2 gpurun_out/r2aj_pytest.log
