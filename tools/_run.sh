mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "C6 or tangent or C5" > gpurun_out/pytest_vtx2.log 2>&1; tail -1 gpurun_out/pytest_vtx2.log
echo "vtx1 $(python tools/profile_apply.py --config C6 --time --reps 10 2>&1 | tail -1)" > gpurun_out/sweep_vtx2.txt
echo "vtx3 $(FE_LIB_PATH=paper_1903_08243_b200/libfeb200_t3.so python tools/profile_apply.py --config C6 --time --reps 10 2>&1 | tail -1)" >> gpurun_out/sweep_vtx2.txt
echo "qc $(FE_NO_VTX=1 python tools/profile_apply.py --config C6 --time --reps 10 2>&1 | tail -1)" >> gpurun_out/sweep_vtx2.txt
echo "c5 $(python tools/profile_apply.py --config C5 --time --reps 10 2>&1 | tail -1)" >> gpurun_out/sweep_vtx2.txt
cut -c1-200 gpurun_out/sweep_vtx2.txt
