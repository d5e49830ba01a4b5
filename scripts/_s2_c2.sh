mkdir -p gpurun_out/s2
o=gpurun_out/s2/c2.log; : > $o
for sh in auto rec; do
  if [ $sh = auto ]; then timeout 120 python scripts/pc_time.py 0 0.05 64 >> $o 2>&1; else CPDDG_SOLVE_SHAPE=rec timeout 120 python scripts/pc_time.py 0 0.05 64 >> $o 2>&1; fi
done
