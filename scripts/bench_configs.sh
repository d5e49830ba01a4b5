#!/usr/bin/env bash
# Bench lines of the other BASELINE configs and the scale points (run under gpurun):
#   bash scripts/bench_configs.sh TAG   ->  gpurun_out/TAG_configs/bench_<config>.json
set -u
TAG=${1:-r02}
OUT=gpurun_out/${TAG}_configs
mkdir -p $OUT
for c in circle sphere05 torus trimesh headline_r17 sphere2p6m; do
    timeout 900 python bench.py --config $c --warmup 3 --cpu-baseline off > $OUT/bench_$c.json 2> $OUT/bench_$c.err
    echo "$c rc=$?"
done
