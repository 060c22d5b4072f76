for n in 4 2 8 1; do
  FE_FILL_CTAS=$n python bench.py --config C4 --steps 20 --warmup 3 > gpurun_out/r2ap_c4_f$n.log 2>&1
done
python tools/bench_table.py gpurun_out/r2ap_c4_f4.log gpurun_out/r2ap_c4_f2.log gpurun_out/r2ap_c4_f8.log gpurun_out/r2ap_c4_f1.log
