python -m pytest tests -q -m gpu -x -k "coverage" > gpurun_out/r2q_pytest.log 2>&1
tail -2 gpurun_out/r2q_pytest.log
for v in "" pw2 pw8 pm2; do
  lib=""; [ -n "$v" ] && lib="FE_LIB_PATH=paper_1903_08243_b200/libfeb200_$v.so"
  env $lib python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2q_c3_${v:-base}.log 2>&1
done
python tools/bench_table.py gpurun_out/r2q_c3_base.log gpurun_out/r2q_c3_pw2.log gpurun_out/r2q_c3_pw8.log gpurun_out/r2q_c3_pm2.log
mkdir -p /tmp/prof
prof() { # config kernel-regex env
  c=$1; k=$2; shift 2
  env "$@" timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -f -o /tmp/prof/$c python tools/profile_apply.py --config $c --reps 2 > /tmp/prof/$c.log 2>&1
  python tools/ncu_summary.py /tmp/prof/$c.ncu-rep > gpurun_out/ncu_r2q_$c.txt 2>&1
  python tools/ncu_hot.py /tmp/prof/$c.ncu-rep >> gpurun_out/ncu_r2q_$c.txt 2>&1
}
prof C3-Q2 hexq2 X=1
prof C4-quad-Q4 pair_pipe FE_PAIR_CFG=1
mv gpurun_out/ncu_r2q_C4-quad-Q4.txt gpurun_out/ncu_r2q_C4-quad-Q4_pipe.txt
prof C4-quad-Q3 pair_kernel X=1
