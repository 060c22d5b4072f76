# monomial trilinear geometry (plane, plane_t, team kernels) + pair pipe with symmetric tables
python -m pytest tests -q -m gpu -x -k "C3 or C4 or hex or quad or edge or coverage" > gpurun_out/r2o_pytest.log 2>&1
tail -3 gpurun_out/r2o_pytest.log
python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r2o_c3.log 2>&1
for cfg in 0 1; do
  FE_PAIR_CFG=$cfg python bench.py --config C4 --steps 10 --warmup 3 > gpurun_out/r2o_c4_cfg$cfg.log 2>&1
done
python tools/bench_table.py gpurun_out/r2o_c3.log
python tools/bench_table.py gpurun_out/r2o_c4_cfg0.log gpurun_out/r2o_c4_cfg1.log
