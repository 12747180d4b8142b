# One gpurun call of GPU-side steps, each logged with its exit code:
#   gpurun -- 'bash tools/session_gpu.sh <tag> "<cmd>" ...'
tag=$1; shift
mkdir -p gpurun_out
for s in "$@"; do
  echo "== $s"; bash -c "$s"; echo "rc $?"
done > gpurun_out/session_$tag.log 2>&1
tail -5 gpurun_out/session_$tag.log | cut -c1-400
