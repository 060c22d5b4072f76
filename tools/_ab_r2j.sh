for v in "" tkA tkB tkC; do
  lib=""; [ -n "$v" ] && lib="FE_LIB_PATH=paper_1903_08243_b200/libfeb200_$v.so"
  env $lib python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2j_c3_${v:-base}.log 2>&1
  env $lib python bench.py --config C4 --steps 10 --warmup 3 > gpurun_out/r2j_c4_${v:-base}.log 2>&1
done
