python -m pytest tests -q -m gpu -x -k "C2 or tet or coverage or edge or hex" > gpurun_out/r2s_pytest.log 2>&1
tail -2 gpurun_out/r2s_pytest.log
for v in "" nosplit; do
  lib=""; [ -n "$v" ] && lib="FE_LIB_PATH=paper_1903_08243_b200/libfeb200_$v.so"
  env $lib python bench.py --config C2 --steps 20 --warmup 3 > gpurun_out/r2s_c2_${v:-base}.log 2>&1
done
python tools/bench_table.py gpurun_out/r2s_c2_base.log gpurun_out/r2s_c2_nosplit.log
python bench.py --config C4 --steps 10 --warmup 3 > gpurun_out/r2s_c4.log 2>&1
python tools/bench_table.py gpurun_out/r2s_c4.log
