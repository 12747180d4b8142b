# Round profiling recipe (run on the GPU box from the repo root):
#   bash tools/profile_round.sh <tag>
# 1. launch list of the bench command (gpu__time_duration per launch), summarized
#    per kernel; 2. one `ncu --set full` capture of the LS kernels of a bounded
#    solve (tools/prof_ls.py), exported to raw/source CSV summaries. Only small
#    text files are left in gpurun_out/ (the .ncu-rep stays in /tmp).
set -e
tag=${1:-r1}
out=gpurun_out
mkdir -p $out
BENCH="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e"
$BENCH > $out/plain_bench_$tag.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches_$tag.csv $BENCH \
  > /tmp/ncu_bench_$tag.log 2>&1
python tools/launch_summary.py /tmp/launches_$tag.csv > $out/launches_$tag.txt
gzip -c /tmp/launches_$tag.csv > $out/launches_$tag.csv.gz
python tools/prof_ls.py --ls 4 > $out/plain_ls_$tag.log 2>&1
ncu --set full --clock-control none --import-source on \
  -k "regex:k_matvec|zfwd|ypass|xgamma|zinv|k_cg_update|k_sweep|k_comp_tangent" -c 20 \
  -o /tmp/ls_$tag python tools/prof_ls.py --ls 4 > /tmp/ncu_ls_$tag.log 2>&1
python tools/ncu_summary.py /tmp/ls_$tag.ncu-rep > $out/ncu_full_$tag.txt
ncu -i /tmp/ls_$tag.ncu-rep --page raw --csv > /tmp/raw_$tag.csv
gzip -c /tmp/raw_$tag.csv > $out/ncu_raw_$tag.csv.gz
ls -la $out
