mkdir -p gpurun_out/s2
timeout 300 python scripts/ab_env.py CPDDG_BLOCKINV 0 1 > gpurun_out/s2/ab_inv.log 2>&1
timeout 300 python scripts/quick_headline.py > gpurun_out/s2/quick_inv.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s2/parity_inv.log 2>&1
