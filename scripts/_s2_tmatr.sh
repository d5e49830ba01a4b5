mkdir -p gpurun_out/s2
o=gpurun_out/s2/tmatr.log; : > $o
for m in 1 0 2; do CPDDG_SOLVE_DEBUG=16 timeout 120 python scripts/trace_tma_steps.py $m >> $o 2>&1; done
CPDDG_SOLVE_DEBUG=$((16 + (60<<16))) timeout 120 python scripts/trace_tma_steps.py 0 >> $o 2>&1
