mkdir -p gpurun_out/s2
o=gpurun_out/s2/knobs.log; : > $o
for d in 0 4 256 512; do CPDDG_SOLVE_DEBUG=$d timeout 120 python scripts/pc_time.py 0 >> $o 2>&1; done
CPDDG_SOLVE_SHAPE=small timeout 120 python scripts/pc_time.py 0 >> $o 2>&1
CPDDG_SOLVE_SHAPE=small CPDDG_BLOCKINV=0 timeout 120 python scripts/pc_time.py 0 >> $o 2>&1
CPDDG_BWD_PREFETCH=2 timeout 120 python scripts/pc_time.py 2 >> $o 2>&1
timeout 120 python scripts/pc_time.py 2 >> $o 2>&1
timeout 120 python scripts/pc_time.py 1 >> $o 2>&1
