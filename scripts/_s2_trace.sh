mkdir -p gpurun_out/s2
for inv in 1 0; do
CPDDG_BLOCKINV=$inv CPDDG_SOLVE_DEBUG=32 timeout 300 python scripts/trace_ctas.py 0 > gpurun_out/s2/ctas_inv$inv.log 2>&1
CPDDG_BLOCKINV=$inv CPDDG_SOLVE_DEBUG=16 timeout 300 python scripts/trace_solve.py 1 > gpurun_out/s2/trace_inv$inv.log 2>&1
done
