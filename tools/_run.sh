mkdir -p gpurun_out
for w in C3 C4 C5 C6; do
timeout 600 python bench.py --config $w --steps 3 --warmup 3 > gpurun_out/bench_$w.log 2>&1; echo "$w rc=$? $(tail -1 gpurun_out/bench_$w.log | cut -c1-220)"
done
