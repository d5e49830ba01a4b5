set -x
mkdir -p gpurun_out/final
python bench.py > gpurun_out/final/bench_headline.json 2> gpurun_out/final/bench_headline.err || exit 1
python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 1500 --csv --log-file gpurun_out/final/launches.csv python bench.py --steps 1 --warmup 3 --cpu-baseline off > gpurun_out/final/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_solve -s 2 -c 1 -o gpurun_out/final/k_solve python scripts/profile_pc_mode.py 0 > gpurun_out/final/ncu_solve.log 2>&1
