for d in 0 256 4; do CPDDG_SOLVE_DEBUG=$d python scripts/pc_time.py 0; done
