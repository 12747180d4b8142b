# Full-size oracle fixtures on the B200 box's host cores (16 cores, 196 GB):
#   gpurun -- 'bash tools/run_fixtures_box.sh C5 C4'
mkdir -p gpurun_out/golden
export OMP_NUM_THREADS=$(nproc) OMP_PROC_BIND=close ORACLE_LEAN_TANGENTS=1
make -s -C oracle
for c in "$@"; do
  python tools/fullsize_fixtures.py $c --out gpurun_out/golden > gpurun_out/golden/log_$c.txt 2>&1
  echo "rc $?" >> gpurun_out/golden/log_$c.txt
done
