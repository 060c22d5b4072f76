# ncu captures of the hot kernels: text summaries into gpurun_out/, reports
# kept in /tmp on the box (gpurun_out is capped at 64 MiB); the C5 report is
# copied back when small
mkdir -p /tmp/prof
for spec in "C5:quad_vtx" "C3-Q5:tensor_kernel" "C3-Q6:tensor_kernel" "C4-hex-Q3:tensor_kernel" "C4-quad-Q4:pair_kernel" "C2-P3:dmma_modal" "C2-P4:dmma_modal" "C2-P1:macro_split" "C3-Q3:plane_kernel"; do
  c=${spec%%:*}; k=${spec##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -f -o /tmp/prof/$c python tools/profile_apply.py --config $c --reps 2 > /tmp/prof/$c.log 2>&1
  python tools/ncu_summary.py /tmp/prof/$c.ncu-rep > gpurun_out/ncu_r2_$c.txt 2>&1
  python tools/ncu_hot.py /tmp/prof/$c.ncu-rep >> gpurun_out/ncu_r2_$c.txt 2>&1
  ls -la /tmp/prof/$c.ncu-rep >> gpurun_out/ncu_r2_sizes.txt
done
cp /tmp/prof/C5.ncu-rep gpurun_out/prof_r2_C5.ncu-rep 2>/dev/null
du -sm gpurun_out
