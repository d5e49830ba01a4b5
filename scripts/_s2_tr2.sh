mkdir -p gpurun_out/s2
o=gpurun_out/s2/tr2.log; : > $o
for m in 1 2 0; do timeout 120 python scripts/pc_time.py $m >> $o 2>&1; done
CPDDG_SOLVE_DEBUG=4 timeout 120 python scripts/pc_time.py 1 >> $o 2>&1
for d in 16 $((16 + (100<<16))); do CPDDG_SOLVE_DEBUG=$d timeout 120 python scripts/trace_rec.py >> $o 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s2/parity_tr2.log 2>&1
