mkdir -p gpurun_out/s2l
for c in torus headline; do timeout 900 python bench.py --config $c --cpu-baseline off > gpurun_out/s2l/bench2_$c.json 2> gpurun_out/s2l/bench2_$c.err; done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/s2l/parity_mgs.log 2>&1
