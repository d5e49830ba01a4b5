mkdir -p gpurun_out/s2
o=gpurun_out/s2/pre.log; : > $o
for m in 0 1 2; do timeout 120 python scripts/pc_time.py $m >> $o 2>&1; done
for m in 0 2; do CPDDG_BWD_LAYOUT=rows timeout 120 python scripts/pc_time.py $m >> $o 2>&1; done
CPDDG_SOLVE_DEBUG=256 timeout 120 python scripts/pc_time.py 1 >> $o 2>&1
CPDDG_SOLVE_DEBUG=4 timeout 120 python scripts/pc_time.py 1 >> $o 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s2/parity_pre.log 2>&1
