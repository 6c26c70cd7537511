#!/bin/bash
# Round evidence on the GPU box: bench line, ncu launch list, one --set full capture of a step.
# usage (via gpurun): bash tools/capture_round.sh <tag>
set -x
TAG=$1
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --quick --no-graph --steps 2 --warmup 3 > gpurun_out/ncu_launches_$TAG.log 2>&1
timeout 1800 ncu --set full --import-source on --clock-control none \
    -k 'regex:project_kernel|bin_coop|bucket_emit|render_fwd2|zero_sgrad|valid_count|render_bwd|gaussian_bwd' \
    -s 40 -c 8 -o gpurun_out/prof_$TAG python bench.py --quick --no-graph --steps 2 --warmup 3 \
    > gpurun_out/ncu_full_$TAG.log 2>&1
tail -1 gpurun_out/bench_$TAG.log
