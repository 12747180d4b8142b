timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r1d.log 2>&1; echo "rc $?" >> gpurun_out/pytest_gpu_r1d.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1d.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke_r1d.log
