for v in "" nr b128 b96; do
  lib=""; [ -n "$v" ] && lib="FE_LIB_PATH=paper_1903_08243_b200/libfeb200_$v.so"
  env $lib python bench.py --config C4 --steps 20 --warmup 3 > gpurun_out/r2as_c4_${v:-base}.log 2>&1
done
python tools/bench_table.py gpurun_out/r2as_c4_base.log gpurun_out/r2as_c4_nr.log gpurun_out/r2as_c4_b128.log gpurun_out/r2as_c4_b96.log
