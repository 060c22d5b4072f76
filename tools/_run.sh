mkdir -p gpurun_out /tmp/prof
for c in C5 C6 C2-P1 C3-Q1 C2-P2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'^(?!k_|spin|vectorized).*' -c 1 -o /tmp/prof/prof17_$c python tools/profile_apply.py --config $c --reps 1 > /tmp/prof/ncu17_$c.log 2>&1
  python tools/ncu_summary.py /tmp/prof/prof17_$c.ncu-rep >> gpurun_out/ncu17_summaries.txt 2>&1
done
cp /tmp/prof/prof17_C5.ncu-rep /tmp/prof/prof17_C2-P1.ncu-rep gpurun_out/
du -sh gpurun_out
