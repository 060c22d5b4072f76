run() { # tag env...
  tag=$1; shift
  env "$@" python bench.py --steps 8 --warmup 3 > gpurun_out/r2aa_$tag.log 2>&1
  python - <<PY
import json
d=json.loads(open('gpurun_out/r2aa_$tag.log').read().strip().splitlines()[-1])
e=d['e2e']; fl=d['value']*d['ms_per_step']*1e-3
print('$tag', 'e2e', e['value'], 'ms/step', round(fl/e['value']*1e3,1))
PY
}
run base X=1
run noapply_zero FE_HOST_NOAPPLY=1 FE_HOST_ASSUME_ZERO=1
run noapply_zero_t1 FE_HOST_NOAPPLY=1 FE_HOST_ASSUME_ZERO=1 FE_E2E_THREADS=1
run noapply_zero_t8 FE_HOST_NOAPPLY=1 FE_HOST_ASSUME_ZERO=1 FE_E2E_THREADS=8
run zero_passive FE_HOST_ASSUME_ZERO=1 OMP_WAIT_POLICY=passive
run passive_s2 OMP_WAIT_POLICY=passive FE_HOST_SCAN_THREADS=2
