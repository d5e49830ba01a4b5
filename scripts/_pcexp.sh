CPDDG_SOLVE_DEBUG=16 CPDDG_SOLVE_LIMIT=1 python scripts/trace_solve.py 1 | head -3
CPDDG_SOLVE_DEBUG=16 CPDDG_SOLVE_LIMIT=1 python scripts/trace_solve.py 2 | head -3
for m in 1 2 0; do python scripts/pc_time.py $m; done
python scripts/spec_compare.py
