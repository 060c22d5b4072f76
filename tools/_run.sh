mkdir -p gpurun_out
for lib in libfeb200 libfeb200_qa libfeb200_qb libfeb200_qc; do for c in C4-hex-Q1 C4-quad-Q1 C4-quad-Q2; do
echo "$lib $(FE_LIB_PATH=paper_1903_08243_b200/$lib.so python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
done; done > gpurun_out/sweep_qct_retune.txt 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/sweep_qct_retune.txt'):
    lib, js = l.split(' ', 1)
    try:
        d = json.loads(js); print(lib, d['config'], round(d['best_ms']*1e3, 1), round(d['roofline_frac'], 3))
    except Exception as e: print(lib, 'ERR', js[:100])
PY
