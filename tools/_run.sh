mkdir -p gpurun_out
tools/sweep.sh > gpurun_out/sweep_v9.txt 2>&1
python bench.py > gpurun_out/bench_v9.log 2>&1; tail -1 gpurun_out/bench_v9.log | cut -c1-600
