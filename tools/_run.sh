mkdir -p gpurun_out
python tools/pcie_bw.py
for i in 1 2 3; do for lib in libfeb200 libfeb200_y16; do
FE_LIB_PATH=paper_1903_08243_b200/$lib.so python bench.py --steps 10 > gpurun_out/b.log 2>&1
echo "$lib $(tail -1 gpurun_out/b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["e2e"]["value"])')"
done; done > gpurun_out/ych.txt
cat gpurun_out/ych.txt
