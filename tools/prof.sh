#!/bin/bash
# ncu evidence for a bench workload (one GPU). Usage: bash tools/prof.sh <tag> [bench args...]
tag=$1; shift
NCU=/usr/local/cuda/bin/ncu
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu "$@" > gpurun_out/launches_${tag}.json 2> gpurun_out/launches_${tag}.log
$NCU --set full --clock-control none --import-source on -k regex:k_match -s 1 -c 1 -o gpurun_out/prof_${tag} -f \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu "$@" > gpurun_out/prof_${tag}.json 2> gpurun_out/prof_${tag}.log
