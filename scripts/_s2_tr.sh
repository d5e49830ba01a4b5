mkdir -p gpurun_out/s2
o=gpurun_out/s2/tr.log; : > $o
for d in 0 4 8; do CPDDG_SOLVE_DEBUG=$d timeout 120 python scripts/pc_time.py 1 >> $o 2>&1; done
for d in 16 20 $((16 + (100<<16))) $((20 + (100<<16))) $((16 + (200<<16))); do CPDDG_SOLVE_DEBUG=$d timeout 120 python scripts/trace_rec.py >> $o 2>&1; done
