bash tools/ab_bench.sh base > gpurun_out/ab2.txt 2>&1
bash tools/ab_bench.sh xw8 COMBO_XW=8 >> gpurun_out/ab2.txt 2>&1
bash tools/ab_bench.sh xw2 COMBO_XW=2 >> gpurun_out/ab2.txt 2>&1
bash tools/ab_bench.sh yw8 COMBO_YW=8 >> gpurun_out/ab2.txt 2>&1
bash tools/ab_bench.sh yw2 COMBO_YW=2 >> gpurun_out/ab2.txt 2>&1
bash tools/ab_bench.sh zl2 COMBO_ZLINES=2 >> gpurun_out/ab2.txt 2>&1
