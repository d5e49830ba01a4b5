mkdir -p gpurun_out/s2l
for c in circle sphere05 torus trimesh; do timeout 900 python bench.py --config $c > gpurun_out/s2l/bench_$c.json 2> gpurun_out/s2l/bench_$c.err; done
