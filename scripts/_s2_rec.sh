mkdir -p gpurun_out/s2
o=gpurun_out/s2/rec.log; : > $o
for m in 1 2 0; do timeout 120 python scripts/pc_time.py $m >> $o 2>&1; done
for m in 2 0; do CPDDG_BWD_LAYOUT=rows timeout 120 python scripts/pc_time.py $m >> $o 2>&1; done
CPDDG_SOLVE_SHAPE=mid timeout 120 python scripts/pc_time.py 0 >> $o 2>&1
CPDDG_SOLVE_DEBUG=4 timeout 120 python scripts/pc_time.py 1 >> $o 2>&1
for d in 16 $((16 + (100<<16))); do CPDDG_SOLVE_DEBUG=$d timeout 120 python scripts/trace_rec.py >> $o 2>&1; done
CPDDG_SOLVE_DEBUG=32 timeout 300 python scripts/trace_ctas.py 1 >> $o 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s2/parity_rec.log 2>&1
