mkdir -p gpurun_out/s2
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/s2/pytest_full.log 2>&1; echo "pytest exit $?" >> gpurun_out/s2/pytest_full.log
timeout 600 python bench.py --cpu-baseline off > gpurun_out/s2/bench2.json 2> gpurun_out/s2/bench2.err
for c in torus trimesh sphere05 circle; do timeout 900 python bench.py --config $c --cpu-baseline off > gpurun_out/s2/bench_$c.json 2>> gpurun_out/s2/bench2.err; done
