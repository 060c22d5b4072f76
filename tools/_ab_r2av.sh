for v in "" elt; do
  lib=""; [ -n "$v" ] && lib="FE_LIB_PATH=paper_1903_08243_b200/libfeb200_$v.so"
  env $lib python bench.py --config C4 --steps 20 --warmup 3 > gpurun_out/r2av_c4_${v:-base}.log 2>&1
done
python tools/bench_table.py gpurun_out/r2av_c4_base.log gpurun_out/r2av_c4_elt.log
FE_LIB_PATH=paper_1903_08243_b200/libfeb200_elt.so python -m pytest tests -q -m gpu -x -k "elasticity or C4" 2>&1 | tail -2
