# One gpurun call: an oracle fixture on the host cores (background, cores 0-13)
# while the GPU side (cores 14-15) runs tests / profiles with small host memory.
#   gpurun --timeout 3600 -- 'bash tools/session_fix.sh <case> <tag> <budget_s> <gpu script...>'
case=$1; tag=$2; budget=${3:-3300}; shift 3
mkdir -p gpurun_out/golden
make -s -C oracle
( export OMP_NUM_THREADS=14 OMP_PROC_BIND=close ORACLE_LEAN_TANGENTS=1
  for c in $case; do
    taskset -c 0-13 timeout $budget python tools/fullsize_fixtures.py $c --out gpurun_out/golden $FIXTURE_ARGS > gpurun_out/golden/log_$c.txt 2>&1
    echo "rc $?" >> gpurun_out/golden/log_$c.txt
  done ) &
FIX=$!
export OMP_NUM_THREADS=2
{ nproc; lscpu | head -25; free -g; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; } > gpurun_out/box_info.txt 2>&1
for s in "$@"; do
  echo "== $s"; taskset -c 14,15 bash -c "$s"; echo "rc $?"
done > gpurun_out/session_$tag.log 2>&1
wait $FIX
tail -3 gpurun_out/golden/log_*.txt
