mkdir -p gpurun_out/s2
o=gpurun_out/s2/lpt.log; : > $o
timeout 60 python scripts/pc_time.py 0 >> $o 2>&1
CPDDG_SOLVE_DEBUG=32 timeout 60 python scripts/trace_tma_ctas.py >> $o 2>&1
