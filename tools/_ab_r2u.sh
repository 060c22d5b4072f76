nproc; python - <<'PY'
import os; print("affinity", len(os.sched_getaffinity(0)))
PY
run() { # tag env...
  tag=$1; shift
  env "$@" python bench.py --steps 5 --warmup 3 > gpurun_out/r2u_$tag.log 2>&1
  python - <<PY
import json
d=json.loads(open('gpurun_out/r2u_$tag.log').read().strip().splitlines()[-1])
print('$tag', 'e2e', d['e2e']['value'], 'value', d['value'])
PY
}
run base X=1
run zero FE_HOST_ASSUME_ZERO=1
run scan2 FE_HOST_SCAN_THREADS=2
run scan4 FE_HOST_SCAN_THREADS=4
run zero_t1 FE_HOST_ASSUME_ZERO=1 FE_E2E_THREADS=1
run zero_t4 FE_HOST_ASSUME_ZERO=1 FE_E2E_THREADS=4
run zero_t16 FE_HOST_ASSUME_ZERO=1 FE_E2E_THREADS=16
