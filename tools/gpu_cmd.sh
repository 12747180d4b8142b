timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; echo "rc $?" >> gpurun_out/pytest_gpu3.log
bash tools/ab_bench.sh split > gpurun_out/ab.txt 2>&1
bash tools/ab_bench.sh nosplit COMBO_SPLIT_SWEEP=0 >> gpurun_out/ab.txt 2>&1
