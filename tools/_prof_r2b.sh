mkdir -p /tmp/prof
for spec in "C3-Q5:tensor_kernel" "C3-Q6:tensor_kernel" "C4-hex-Q3:tensor_kernel" "C4-hex-Q2:tensor_kernel" "C4-quad-Q4:pair_kernel" "C2-P3:dmma_modal" "C3-Q4:plane_kernel"; do
  c=${spec%%:*}; k=${spec##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -f -o /tmp/prof/$c python tools/profile_apply.py --config $c --reps 2 > /tmp/prof/$c.log 2>&1
  python tools/ncu_hot.py /tmp/prof/$c.ncu-rep --top 40 > gpurun_out/ncu_r2_${c}_hot.txt 2>&1
done
python bench.py --steps 20 --warmup 3 > gpurun_out/r2i_bench_all.log 2>&1
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r2i_bench_ref.log 2>&1
