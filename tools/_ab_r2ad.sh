python -m pytest tests -q -m gpu -x -k "abi or host or edge or bench or cli" > gpurun_out/r2ad_pytest.log 2>&1
tail -3 gpurun_out/r2ad_pytest.log
python tools/e2e_percall.py > gpurun_out/r2ad_percall.txt 2>&1; tail -21 gpurun_out/r2ad_percall.txt
run() { # tag env...
  tag=$1; shift
  env "$@" python bench.py --steps 8 --warmup 3 > gpurun_out/r2ad_$tag.log 2>&1
  python - <<PY
import json
d=json.loads(open('gpurun_out/r2ad_$tag.log').read().strip().splitlines()[-1])
e=d['e2e']; fl=d['value']*d['ms_per_step']*1e-3
print('$tag', 'e2e', e['value'], 'ms/step', round(fl/e['value']*1e3,1))
PY
}
run t4 X=1
run t4_s4 FE_HOST_SCAN_THREADS=4
run t6_s3 FE_E2E_THREADS=6 FE_HOST_SCAN_THREADS=3
run t3_s5 FE_E2E_THREADS=3 FE_HOST_SCAN_THREADS=5
run t2_s8 FE_E2E_THREADS=2 FE_HOST_SCAN_THREADS=8
