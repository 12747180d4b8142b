# one ncu --set full capture of the LS kernels of a bounded solve (tools/prof_ls.py)
# usage: bash tools/ncu_ls.sh <tag> [kernel regex] [count]
tag=${1:-x}; rx=${2:-"k_matvec|zfwd|ypass|xgamma|zinv|k_cg_update|k_sweep|k_comp_tangent"}; cnt=${3:-20}
mkdir -p gpurun_out
python tools/prof_ls.py --ls 4 > gpurun_out/plain_ls_$tag.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k "regex:$rx" -c $cnt \
  -o /tmp/ls_$tag python tools/prof_ls.py --ls 4 > /tmp/ncu_ls_$tag.log 2>&1
tail -3 /tmp/ncu_ls_$tag.log > gpurun_out/ncu_ls_$tag.tail
python tools/ncu_summary.py /tmp/ls_$tag.ncu-rep > gpurun_out/ncu_full_$tag.txt
ncu -i /tmp/ls_$tag.ncu-rep --page raw --csv > /tmp/raw_$tag.csv
gzip -c /tmp/raw_$tag.csv > gpurun_out/ncu_raw_$tag.csv.gz
ncu -i /tmp/ls_$tag.ncu-rep --page source --csv --print-source sass > /tmp/src_$tag.csv 2>/dev/null
gzip -c /tmp/src_$tag.csv > gpurun_out/ncu_src_$tag.csv.gz
