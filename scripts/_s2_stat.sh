mkdir -p gpurun_out/s2
CPDDG_VERBOSE=1 timeout 120 python scripts/pc_time.py 0 > gpurun_out/s2/stat.log 2>&1
CPDDG_SOLVE_DEBUG=32 timeout 300 python scripts/trace_ctas.py 2 >> gpurun_out/s2/stat.log 2>&1
