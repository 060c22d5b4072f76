mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "C3-Q5 or C3-Q6 or C4-hex-Q2 or C4-hex-Q3 or hexahedron-5 or hexahedron-6 or elasticity_lame-hexahedron or slab" > gpurun_out/pytest_pre.log 2>&1; tail -1 gpurun_out/pytest_pre.log
for c in C3-Q5 C3-Q6 C4-hex-Q2 C4-hex-Q3; do
echo "pre $(python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
echo "team $(FE_NO_PREGEO=1 python tools/profile_apply.py --config $c --time --reps 20 2>&1 | tail -1)"
done > gpurun_out/sweep_pre.txt 2>&1
cut -c1-220 gpurun_out/sweep_pre.txt
