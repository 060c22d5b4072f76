FE_LIB_PATH=paper_1903_08243_b200/libfeb200_eo.so python -m pytest tests -q -m gpu -x -k "C3 or c3_rule or hex or edge" > gpurun_out/r2aw_pytest.log 2>&1
tail -2 gpurun_out/r2aw_pytest.log
for v in head "" eo; do
  lib=""; [ -n "$v" ] && lib="FE_LIB_PATH=paper_1903_08243_b200/libfeb200_$v.so"
  env $lib python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2aw_c3_${v:-new}.log 2>&1
done
python tools/bench_table.py gpurun_out/r2aw_c3_head.log gpurun_out/r2aw_c3_new.log gpurun_out/r2aw_c3_eo.log
