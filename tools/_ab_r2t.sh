for v in "" pr8 pr12 pm12; do
  lib=""; [ -n "$v" ] && lib="FE_LIB_PATH=paper_1903_08243_b200/libfeb200_$v.so"
  env $lib python bench.py --config C4 --steps 10 --warmup 3 > gpurun_out/r2t_c4_${v:-base}.log 2>&1
done
python tools/bench_table.py gpurun_out/r2t_c4_base.log gpurun_out/r2t_c4_pr8.log gpurun_out/r2t_c4_pr12.log gpurun_out/r2t_c4_pm12.log
for b in 128 64 32; do
  FE_HEXQ1_BLOCK=$b python bench.py --config C3 --steps 20 --warmup 3 > gpurun_out/r2t_c3_b$b.log 2>&1
done
FE_HEXQ1_BLOCK=64 FE_HEXQ1_MINB=3 python bench.py --config C3 --steps 20 --warmup 3 > gpurun_out/r2t_c3_b64m3.log 2>&1
python tools/bench_table.py gpurun_out/r2t_c3_b128.log gpurun_out/r2t_c3_b64.log gpurun_out/r2t_c3_b32.log gpurun_out/r2t_c3_b64m3.log
