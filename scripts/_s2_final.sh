set -x
mkdir -p gpurun_out/s2f
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/s2f/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/s2f/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2f/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/s2f/smoke.log
python bench.py > gpurun_out/s2f/bench_headline.json 2> gpurun_out/s2f/bench_headline.err
for c in circle sphere05 torus trimesh; do timeout 900 python bench.py --config $c > gpurun_out/s2f/bench_$c.json 2> gpurun_out/s2f/bench_$c.err; done
python bench.py --impl reference > gpurun_out/s2f/bench_ref.json 2> gpurun_out/s2f/bench_ref.err
