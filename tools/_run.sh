mkdir -p gpurun_out
python tools/c1_floor.py > gpurun_out/c1_floor2.txt 2>&1; cat gpurun_out/c1_floor2.txt | tail -3
