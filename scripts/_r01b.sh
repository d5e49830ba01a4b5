set -x
python bench.py > gpurun_out/r01b_bench.json 2> gpurun_out/r01b_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 1500 --csv --log-file gpurun_out/r01b_launches.csv python bench.py --steps 1 --warmup 3 --cpu-baseline off > gpurun_out/r01b_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_solve -s 20 -c 1 -o gpurun_out/r01b_k_solve python scripts/profile_pc_mode.py 0 > gpurun_out/r01b_ncu_solve.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_extend_staged -s 3 -c 1 -o gpurun_out/r01b_k_extend python scripts/ext_compare.py 0.0125 > gpurun_out/r01b_ncu_ext.log 2>&1
tail -1 gpurun_out/r01b_bench.json
