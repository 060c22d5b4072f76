for v in "" t0; do
  lib=""; [ -n "$v" ] && lib="FE_LIB_PATH=paper_1903_08243_b200/libfeb200_$v.so"
  env $lib python bench.py --config C4 --steps 20 --warmup 3 > gpurun_out/r2at_c4_${v:-base}.log 2>&1
done
python tools/bench_table.py gpurun_out/r2at_c4_base.log gpurun_out/r2at_c4_t0.log
FE_LIB_PATH=paper_1903_08243_b200/libfeb200_t0.so python -m pytest tests -q -m gpu -x -k "quad and (C4 or elasticity or coverage)" 2>&1 | tail -2
