mkdir -p gpurun_out/s2
o=gpurun_out/s2/mgs.log; : > $o
timeout 300 python scripts/mgs_compare.py >> $o 2>&1
timeout 300 python scripts/quick_headline.py >> $o 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s2/parity_mgs.log 2>&1
