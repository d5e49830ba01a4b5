mkdir -p gpurun_out/s2
o=gpurun_out/s2/sloan.log; : > $o
for ord in rcm sloan; do CPDDG_ORDER=$ord CPDDG_VERBOSE=1 timeout 120 python scripts/pc_time.py 0 >> $o 2>&1; done
CPDDG_ORDER=sloan timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s2/parity_sloan.log 2>&1
