mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "cli" > gpurun_out/pytest_cli.log 2>&1; tail -3 gpurun_out/pytest_cli.log
python -m paper_1903_08243_b200 verify --n 4 > gpurun_out/cli_verify.txt 2>&1; tail -25 gpurun_out/cli_verify.txt
