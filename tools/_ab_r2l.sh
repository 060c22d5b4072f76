for v in "" tkasync; do
  lib=""; [ -n "$v" ] && lib="FE_LIB_PATH=paper_1903_08243_b200/libfeb200_$v.so"
  env $lib python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2l_c3_${v:-base}.log 2>&1
  env $lib python bench.py --config C4 --steps 10 --warmup 3 > gpurun_out/r2l_c4_${v:-base}.log 2>&1
done
FE_LIB_PATH=paper_1903_08243_b200/libfeb200_tkasync.so python -m pytest tests -q -m gpu -x -k "coverage or parity or edge or slabs" > gpurun_out/r2l_pytest_async.log 2>&1
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2l_bench_ref.log 2>&1
