mkdir -p gpurun_out/s2
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s2/pytest_c2.log 2>&1; echo "exit $?" >> gpurun_out/s2/pytest_c2.log
for c in sphere05 circle headline; do timeout 900 python bench.py --config $c --cpu-baseline off > gpurun_out/s2/bench_c2_$c.json 2>> gpurun_out/s2/bench_c2.err; done
