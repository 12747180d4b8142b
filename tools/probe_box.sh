# Box facts for DESIGN.md (host cores / RAM for the CPU arm) + the GPU suite.
mkdir -p gpurun_out
{ nproc; lscpu | head -25; free -g; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; df -h /tmp | tail -1; } > gpurun_out/box_info.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_probe.log 2>&1; echo "rc $?" >> gpurun_out/pytest_gpu_probe.log
