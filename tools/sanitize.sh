# compute-sanitizer over the small-grid driver (tools/sanitize_case.py); logs -> gpurun_out/sanitizer_<tool>_<tag>.log
tag=${1:-x}; n=${2:-16}
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py $n > gpurun_out/sanitizer_${tool}_$tag.log 2>&1
  echo "rc $?" >> gpurun_out/sanitizer_${tool}_$tag.log
done
