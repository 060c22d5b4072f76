mkdir -p gpurun_out
for c in C2-P1 C2-P2; do
  for cfg in 0 1 2 3; do
    echo "dmma cfg=$cfg $(FE_NO_SPLIT=1 FE_DMMA_CFG=$cfg python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
  done
  echo "split $(python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
  echo "split-g2 $(FE_LIB_PATH=paper_1903_08243_b200/libfeb200_g2.so python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
done > gpurun_out/sweep_modal2.txt 2>&1
cut -c1-200 gpurun_out/sweep_modal2.txt
