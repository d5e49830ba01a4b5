for i in 1 2; do
python scripts/pc_time.py 0
CPDDG_ENVELOPE=sym python scripts/pc_time.py 0
done
ncu --set full --import-source on --clock-control none -k regex:k_solve -s 2 -c 1 -o gpurun_out/r01b_k_solve python scripts/profile_pc_mode.py 0 > gpurun_out/r01b_ncu_solve.log 2>&1
tail -2 gpurun_out/r01b_ncu_solve.log
