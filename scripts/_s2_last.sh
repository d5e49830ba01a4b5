set -x
mkdir -p gpurun_out/s2l
# (pytest run separately)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2l/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/s2l/smoke.log
python bench.py > gpurun_out/s2l/bench_headline.json 2> gpurun_out/s2l/bench_headline.err
python bench.py --impl reference > gpurun_out/s2l/bench_ref.json 2> gpurun_out/s2l/bench_ref.err
python bench.py --steps 1 --warmup 3 --cpu-baseline off > gpurun_out/s2l/plain_launch.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 1500 --csv --log-file gpurun_out/s2l/launches.csv python bench.py --steps 1 --warmup 3 --cpu-baseline off > gpurun_out/s2l/ncu_launch.log 2>&1
