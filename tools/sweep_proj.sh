# projection microbenchmark sweep over the FFT tuning knobs (tools/bench_proj.py)
python -m pytest tests/test_gpu_parity.py -q -x -k "project or green or continuous" 2>&1 | tail -2
COMBO_XV=4 COMBO_XMINB=3 python -m pytest tests/test_gpu_parity.py -q -x -k "project or green" 2>&1 | tail -2
for kv in "COMBO_XV=3" "COMBO_XV=4" "COMBO_XV=4 COMBO_XMINB=3" "COMBO_XV=4 COMBO_XW=2" "COMBO_XV=4 COMBO_XW=2 COMBO_XMINB=3"; do
  echo "$kv"; env $kv python tools/bench_proj.py 512 5 2>&1 | tail -1
done
for k in continuous staggered; do python tools/bench_proj.py 512 3 $k 2>&1 | tail -1; done
