run() { # tag env...
  tag=$1; shift
  env "$@" python bench.py --steps 5 --warmup 3 > gpurun_out/r2v_$tag.log 2>&1
  python - <<PY
import json
d=json.loads(open('gpurun_out/r2v_$tag.log').read().strip().splitlines()[-1])
print('$tag', 'e2e', d['e2e']['value'], 'value', d['value'])
PY
}
run cfg_t4 FE_E2E_ORDER=config FE_E2E_THREADS=4
run size_t4 FE_E2E_THREADS=4
run size_t3 FE_E2E_THREADS=3
run size_t6 FE_E2E_THREADS=6
run size_t8 FE_E2E_THREADS=8
run size_t4_s2 FE_E2E_THREADS=4 FE_HOST_SCAN_THREADS=2
run size_t4_b FE_E2E_THREADS=4
