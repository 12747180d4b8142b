# GPU session: tests (gpu marker), a short bench, projection A/B of knobs.
#   gpurun -- 'bash tools/gpu_session.sh <tag> [knob sets...]'
tag=${1:-s}; shift
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "rc $?" >> gpurun_out/pytest_gpu_$tag.log
for kv in "COMBO_XTMA=1" "$@"; do
  echo "== $kv"; env $kv timeout 300 python tools/bench_proj.py 512 5 2>&1 | tail -1
done > gpurun_out/proj_ab_$tag.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_$tag.log 2>&1; echo "rc $?" >> gpurun_out/bench_$tag.log
