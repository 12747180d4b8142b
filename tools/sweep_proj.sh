# projection microbenchmark sweep over the FFT tuning knobs (tools/bench_proj.py)
for kv in "COMBO_XV=2" "COMBO_XV=3" "COMBO_XV=4 COMBO_XW=8" "COMBO_XV=3 COMBO_YW=4" "COMBO_XV=3 COMBO_ZLINES=1"; do
  env $kv python tools/bench_proj.py 512 5 2>&1 | tail -1
done
for k in continuous staggered; do COMBO_XV=3 python tools/bench_proj.py 512 3 $k 2>&1 | tail -1; done
python -m pytest tests/test_gpu_parity.py -q -x -k "project or green or continuous" 2>&1 | tail -2
