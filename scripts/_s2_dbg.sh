mkdir -p gpurun_out/s2
o=gpurun_out/s2/dbg.log; : > $o
for d in 0 1 2 3 4 7; do CPDDG_SOLVE_DEBUG=$d timeout 120 python scripts/pc_time.py 1 >> $o 2>&1; done
