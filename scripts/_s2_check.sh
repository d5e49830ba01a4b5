mkdir -p gpurun_out/s2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/s2/pytest_gpu.log
timeout 600 python bench.py --cpu-baseline off > gpurun_out/s2/bench.json 2> gpurun_out/s2/bench.err
