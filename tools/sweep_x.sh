# x+Gamma pass variants at 512^3 (tools/bench_proj.py): tile width, kernel
# variant, launch bound, carveout. Output: gpurun_out/sweep_x.log
mkdir -p gpurun_out
for kv in "COMBO_XV=4" "COMBO_XV=4 COMBO_XMINB=3" "COMBO_XV=4 COMBO_XW=2" "COMBO_XV=4 COMBO_XW=2 COMBO_XMINB=3" \
          "COMBO_XV=4 COMBO_XW=8" "COMBO_XV=3" "COMBO_XV=3 COMBO_XW=2" "COMBO_XV=5" "COMBO_XV=0" "COMBO_PIPE_X=1" \
          "COMBO_XV=4 COMBO_CARVEOUT=100" "COMBO_SWAP=0"; do
  echo "== $kv"; env $kv timeout 120 python tools/bench_proj.py 512 5 2>&1 | tail -1
done > gpurun_out/sweep_x.log 2>&1
