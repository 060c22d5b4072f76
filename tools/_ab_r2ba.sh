for v in "" sx ra sxra; do
  lib=""; [ -n "$v" ] && lib="FE_LIB_PATH=paper_1903_08243_b200/libfeb200_$v.so"
  env $lib python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2ba_c3_${v:-base}.log 2>&1
done
python tools/bench_table.py gpurun_out/r2ba_c3_base.log gpurun_out/r2ba_c3_sx.log gpurun_out/r2ba_c3_ra.log gpurun_out/r2ba_c3_sxra.log
