set -x
mkdir -p gpurun_out/s2/prof
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "streamed or layouts or dense" > gpurun_out/s2/prof/newtest.log 2>&1
python bench.py > gpurun_out/s2/prof/bench_headline.json 2> gpurun_out/s2/prof/bench_headline.err || exit 1
python bench.py --impl reference > gpurun_out/s2/prof/bench_ref.json 2> gpurun_out/s2/prof/bench_ref.err
python bench.py --steps 1 --warmup 3 --cpu-baseline off > gpurun_out/s2/prof/plain_launch.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 1500 --csv --log-file gpurun_out/s2/prof/launches.csv python bench.py --steps 1 --warmup 3 --cpu-baseline off > gpurun_out/s2/prof/ncu_launch.log 2>&1
python scripts/profile_pc_mode.py 0 > gpurun_out/s2/prof/plain_pc.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:k_solve_tma -s 2 -c 1 -o gpurun_out/s2/prof/k_solve_tma python scripts/profile_pc_mode.py 0 > gpurun_out/s2/prof/ncu_solve.log 2>&1
