# Round-end GPU pass (run on the box from the repo root): bash tools/gpu_round.sh <tag>
tag=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$tag.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke_$tag.log
timeout 1200 python bench.py > gpurun_out/bench_$tag.log 2>&1; echo "bench rc $?" >> gpurun_out/bench_$tag.log
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_$tag.log 2>&1
timeout 2400 bash tools/profile_round.sh $tag > gpurun_out/profile_$tag.log 2>&1
