mkdir -p gpurun_out
for c in C2-P3 C2-P4; do for cfg in 1 4 5 6; do
echo "cfg=$cfg $(FE_DMMA_CFG=$cfg python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
done; done > gpurun_out/sweep_modal_occ.txt 2>&1
cut -c1-200 gpurun_out/sweep_modal_occ.txt
FE_DMMA_CFG=4 python -m pytest tests -m gpu -x -q -k "C2-P3 or alternative" 2>&1 | tail -1
