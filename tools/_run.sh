mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "C5 or neohookean or hyperelastic" 2>&1 | tail -1
python tools/profile_apply.py --config C5 --time --reps 10 2>&1 | tail -1 > gpurun_out/c5_final.txt; cut -c1-400 gpurun_out/c5_final.txt
