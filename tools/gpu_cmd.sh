timeout 600 bash tools/ab_bench.sh fused_imaj COMBO_SWAP=0 > gpurun_out/ab.txt 2>&1
timeout 600 bash tools/ab_bench.sh fused_imaj_w4 COMBO_SWAP=0 COMBO_FUSE_WY=4 >> gpurun_out/ab.txt 2>&1
timeout 600 bash tools/ab_bench.sh fused_imaj_nodisc COMBO_SWAP=0 COMBO_FUSE_DISCARD=0 >> gpurun_out/ab.txt 2>&1
COMBO_SWAP=0 timeout 900 bash tools/ncu_ls.sh fz2 "fused" 2 > /dev/null 2>&1
