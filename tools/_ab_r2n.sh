# pair kernel: round-1 (0) vs pipelined persistent at 2/3/4 CTAs per SM
FE_PAIR_CFG=1 python -m pytest tests -q -m gpu -x -k "C4-quad or quad or edge or coverage" > gpurun_out/r2n_pair_pytest.log 2>&1
tail -3 gpurun_out/r2n_pair_pytest.log
for cfg in 0 1 2 3; do
  FE_PAIR_CFG=$cfg python bench.py --config C4 --steps 10 --warmup 3 > gpurun_out/r2n_pair_cfg$cfg.log 2>&1
done
python tools/bench_table.py gpurun_out/r2n_pair_cfg0.log gpurun_out/r2n_pair_cfg1.log gpurun_out/r2n_pair_cfg2.log gpurun_out/r2n_pair_cfg3.log
