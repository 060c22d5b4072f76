# round-2 final validation: full GPU suite, smoke, bench (both arms), launch list, ncu summaries, e2e repeat
python -m pytest tests -q -m gpu > gpurun_out/r2z_pytest_gpu.log 2>&1
tail -2 gpurun_out/r2z_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z_smoke.log 2>&1
tail -1 gpurun_out/r2z_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2z_bench.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2z_bench_ref.log 2>&1
python bench.py --config C6 --steps 10 --warmup 3 > gpurun_out/r2z_bench_c6.log 2>&1
python bench.py --config C2 --steps 20 --warmup 5 > gpurun_out/r2z_bench_c2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2z_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/r2z_ncu_bench.log 2>&1
mkdir -p /tmp/prof
for spec in "C5:quad_vtx" "C2-P3:dmma_modal" "C2-P4:dmma_modal" "C3-Q2:hexq2" "C3-Q3:plane_kernel" "C3-Q4:plane_kernel" "C3-Q5:tensor_kernel" "C3-Q6:tensor_kernel" "C4-hex-Q2:tensor_kernel" "C4-hex-Q3:tensor_kernel" "C4-quad-Q4:pair_" "C2-P1:macro_split" "C3-Q1:hexq1" "C1:affine_et"; do
  c=${spec%%:*}; k=${spec##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -f -o /tmp/prof/$c python tools/profile_apply.py --config $c --reps 2 > /tmp/prof/$c.log 2>&1
  python tools/ncu_summary.py /tmp/prof/$c.ncu-rep > gpurun_out/ncu_r2z_$c.txt 2>&1
  python tools/ncu_hot.py /tmp/prof/$c.ncu-rep >> gpurun_out/ncu_r2z_$c.txt 2>&1
done
du -sm gpurun_out
