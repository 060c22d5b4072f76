mkdir -p gpurun_out
python tools/pcie_bw.py > gpurun_out/pcie_bw.txt 2>&1; cat gpurun_out/pcie_bw.txt
