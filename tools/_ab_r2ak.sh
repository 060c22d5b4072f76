python -m pytest tests -q -m gpu -x -k "quad or elasticity or C4 or edge" > gpurun_out/r2ak_pytest.log 2>&1
tail -2 gpurun_out/r2ak_pytest.log
for v in "" sel; do
  lib=""; [ -n "$v" ] && lib="FE_LIB_PATH=paper_1903_08243_b200/libfeb200_$v.so"
  env $lib python bench.py --config C4 --steps 10 --warmup 3 > gpurun_out/r2ak_c4_${v:-base}.log 2>&1
done
python tools/bench_table.py gpurun_out/r2ak_c4_base.log gpurun_out/r2ak_c4_sel.log
