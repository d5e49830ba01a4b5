mkdir -p gpurun_out/s2
o=gpurun_out/s2/tma.log; : > $o
timeout 120 python scripts/pc_time.py 1 >> $o 2>&1 || { echo "mode1 failed $?" >> $o; exit 1; }
for m in 2 0; do timeout 120 python scripts/pc_time.py $m >> $o 2>&1; done
CPDDG_TMA=0 timeout 120 python scripts/pc_time.py 0 >> $o 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s2/parity_tma.log 2>&1
timeout 300 python scripts/quick_headline.py >> $o 2>&1
