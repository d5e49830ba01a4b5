mkdir -p gpurun_out/s2
o=gpurun_out/s2/tmab.log; : > $o
for m in 0 1 2; do timeout 60 python scripts/pc_time.py $m >> $o 2>&1; done
for m in 1; do CPDDG_SOLVE_DEBUG=16 timeout 60 python scripts/trace_tma_steps.py $m >> $o 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s2/parity_tma.log 2>&1
