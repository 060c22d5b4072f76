mkdir -p gpurun_out
FE_MACRO_P2=1 python -m pytest tests -m gpu -x -q -k "C2-P2 or range" > gpurun_out/pytest_p2m.log 2>&1; tail -1 gpurun_out/pytest_p2m.log
for i in 1 2; do
echo "macro $(FE_MACRO_P2=1 python tools/profile_apply.py --config C2-P2 --time --reps 20 2>&1 | tail -1)"
echo "split $(python tools/profile_apply.py --config C2-P2 --time --reps 20 2>&1 | tail -1)"
done > gpurun_out/sweep_p2macro.txt 2>&1
cut -c1-200 gpurun_out/sweep_p2macro.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v15.log 2>&1; tail -13 gpurun_out/smoke_v15.log
