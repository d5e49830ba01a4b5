mkdir -p gpurun_out/s2
o=gpurun_out/s2/cols.log; : > $o
for m in 0 1 2; do timeout 120 python scripts/pc_time.py $m >> $o 2>&1; done
CPDDG_BWD_LAYOUT=rows timeout 120 python scripts/pc_time.py 2 >> $o 2>&1
CPDDG_SOLVE_SHAPE=big timeout 120 python scripts/pc_time.py 0 >> $o 2>&1
timeout 300 python scripts/quick_headline.py >> $o 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s2/parity_cols.log 2>&1
