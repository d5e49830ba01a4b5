#!/usr/bin/env bash
# Regenerates the committed profiles of a round on a B200 (run under gpurun):
#   bash scripts/profile_round.sh TAG
# 1. the headline bench line (no profiler), 2. the ncu launch list of the same
# command, 3. ncu --set full captures of the preconditioner apply (k_solve_win),
# the operator (k_extend_union + k_helm_pdl) and the factorisation (k_factor2).
# Outputs under gpurun_out/TAG_*.
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --steps 1 --warmup 3 --cpu-baseline off --host-loop > $OUT/${TAG}_ncu_bench.log 2>&1
echo "launch list rc=$?"
# the timed region only (bench.py's NVTX range "timed": one complete solve).  --host-loop: the same
# kernels launched one by one from the host; ncu does not list the kernels inside the
# while-conditional graph nodes of the default device-driven cycles
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $OUT/${TAG}_launches_step.csv \
    python bench.py --steps 1 --warmup 3 --cpu-baseline off --host-loop > $OUT/${TAG}_ncu_bench_step.log 2>&1
echo "step launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve_win -s 2 -c 1 \
    -o $OUT/${TAG}_k_solve_win -f python scripts/profile_pc_mode.py 0 > $OUT/${TAG}_ncu_pc.log 2>&1
echo "pc capture rc=$?"
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on \
    -k regex:"k_extend_union|k_helm_pdl" -s 2 -c 2 -o $OUT/${TAG}_op -f python scripts/profile_kernels.py > $OUT/${TAG}_ncu_op.log 2>&1
echo "op capture rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_factor2" -c 1 \
    -o $OUT/${TAG}_k_factor2 -f python scripts/profile_kernels.py > $OUT/${TAG}_ncu_factor.log 2>&1
echo "factor capture rc=$?"
