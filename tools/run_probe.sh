mkdir -p gpurun_out
timeout 1500 python tools/gpu_fullsize_probe.py C2 C3 C4 C5 --max-ls 0 > gpurun_out/fullsize_probe.log 2>&1; echo "rc $?" >> gpurun_out/fullsize_probe.log
