mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "golden or device_path or accumulate or range or fault or config or C6 or cli" > gpurun_out/pytest_e2e2.log 2>&1; tail -1 gpurun_out/pytest_e2e2.log
for lib in libfeb200 libfeb200_old libfeb200; do
FE_LIB_PATH=paper_1903_08243_b200/$lib.so python bench.py --steps 10 > gpurun_out/bench_e2e2_$lib.log 2>&1
echo "$lib $(tail -1 gpurun_out/bench_e2e2_$lib.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["e2e"]["value"], d["value"], d["ms_per_step"])')"
done
