timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu4.log 2>&1; echo "rc $?" >> gpurun_out/pytest_gpu4.log
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_e2e.log 2>&1
