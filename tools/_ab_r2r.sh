python -m pytest tests -q -m gpu -x -k "C3 or C4 or hex or quad or coverage or edge" > gpurun_out/r2r_pytest.log 2>&1
tail -2 gpurun_out/r2r_pytest.log
for v in "" nosym sym7; do
  lib=""; [ -n "$v" ] && lib="FE_LIB_PATH=paper_1903_08243_b200/libfeb200_$v.so"
  env $lib python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2r_c3_${v:-base}.log 2>&1
  env $lib python bench.py --config C4 --steps 10 --warmup 3 > gpurun_out/r2r_c4_${v:-base}.log 2>&1
done
python tools/bench_table.py gpurun_out/r2r_c3_base.log gpurun_out/r2r_c3_nosym.log gpurun_out/r2r_c3_sym7.log
python tools/bench_table.py gpurun_out/r2r_c4_base.log gpurun_out/r2r_c4_nosym.log gpurun_out/r2r_c4_sym7.log
