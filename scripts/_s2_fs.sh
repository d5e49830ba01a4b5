mkdir -p gpurun_out/s2
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/s2/pytest_fs.log 2>&1; echo "exit $?" >> gpurun_out/s2/pytest_fs.log
