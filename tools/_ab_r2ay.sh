for v in "" q5a q5b q5c q5d; do
  lib=""; [ -n "$v" ] && lib="FE_LIB_PATH=paper_1903_08243_b200/libfeb200_$v.so"
  env $lib python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2ay_c3_${v:-base}.log 2>&1
done
python tools/bench_table.py gpurun_out/r2ay_c3_base.log gpurun_out/r2ay_c3_q5a.log gpurun_out/r2ay_c3_q5b.log gpurun_out/r2ay_c3_q5c.log gpurun_out/r2ay_c3_q5d.log
