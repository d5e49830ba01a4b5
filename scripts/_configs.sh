mkdir -p gpurun_out/cfg
for c in circle sphere05 torus trimesh; do
  python bench.py --config $c > gpurun_out/cfg/bench_$c.json 2> gpurun_out/cfg/bench_$c.err || echo "FAIL $c"
done
python bench.py --impl reference > gpurun_out/cfg/bench_ref.json 2> gpurun_out/cfg/bench_ref.err || echo "FAIL ref"
for c in circle sphere05 torus trimesh ref; do python -c "
import json;d=json.load(open('gpurun_out/cfg/bench_$c.json'));print('$c', d.get('value'), d.get('ms_per_step'), d.get('config',{}).get('gmres_iterations'))"; done
