# projection microbenchmark sweep over the FFT tuning knobs (tools/bench_proj.py)
python -m pytest tests/test_gpu_parity.py -q -x -k "fft or project or green" 2>&1 | tail -2
for kv in "COMBO_SWAP=0 COMBO_YW=8" "COMBO_SWAP=0 COMBO_YW=4" "COMBO_SWAP=1 COMBO_YW=8" "COMBO_SWAP=1 COMBO_YW=16" "COMBO_SWAP=0 COMBO_YW=16"; do
  echo "$kv"; env $kv python tools/bench_proj.py 512 3 2>&1 | tail -1
done
