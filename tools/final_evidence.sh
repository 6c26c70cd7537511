#!/bin/bash
# Round evidence (GPU box): headline bench line, the other configs' lines, the reference arm, the
# pose sweep, and the ncu launch list + --set full capture. usage: bash tools/final_evidence.sh <tag>
set -x
TAG=$1
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_$TAG.log 2>&1
timeout 600 python bench.py --config 1 --no-cpu-baseline > gpurun_out/cfg1_$TAG.log 2>&1
timeout 600 python bench.py --config 3 --steps 5 > gpurun_out/cfg3_$TAG.log 2>&1
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 > gpurun_out/cfg4_$TAG.log 2>&1
timeout 600 python bench.py --config 4 --frame --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/cfg4frame_$TAG.log 2>&1
timeout 600 python bench.py --sh 1 --no-cpu-baseline --no-e2e > gpurun_out/sh1_$TAG.log 2>&1
timeout 1500 python tools/pose_sweep.py gpurun_out/pose_sweep_$TAG.json > gpurun_out/pose_sweep_$TAG.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --quick --no-graph --steps 2 --warmup 3 > gpurun_out/ncu_launches_$TAG.log 2>&1
timeout 1800 ncu --set full --import-source on --clock-control none \
    -k 'regex:project_kernel|bin_coop|bucket_emit|render_fwd2|zero_sgrad|render_bwd|gaussian_bwd' \
    -s 40 -c 7 -o gpurun_out/prof_$TAG python bench.py --quick --no-graph --steps 2 --warmup 3 \
    > gpurun_out/ncu_full_$TAG.log 2>&1
tail -c 400 gpurun_out/bench_$TAG.log
