for c in C4-quad-Q3 C4-quad-Q4 C3-Q4 C3-Q5 C3-Q6 C4-hex-Q2 C4-hex-Q3 C3-Q1 C2-P1 C2-P4; do
  python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1 | python -c "
import sys, json
d=json.loads(sys.stdin.read()); print(d['config'], 'acc %.4f ms  with-fill %.4f ms  (+%.1f%%)  frac %.3f -> %.3f' % (d['best_ms'], d['best_ms_with_zero_fill'], 100*(d['best_ms_with_zero_fill']/d['best_ms']-1), d['roofline_frac'], d['roofline_frac_with_zero_fill']))"
done
